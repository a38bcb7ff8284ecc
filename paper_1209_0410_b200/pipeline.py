"""Host-to-host serving pipeline: query batches in pinned host memory, results
back to pinned host memory, with the copies overlapped with the search.

Three CUDA streams and two device slots: H2D of batch b+1 runs while batch b
is searched, and the D2H of batch b runs while batch b+1 is searched.  Events
order slot reuse (a slot's queries are not overwritten before its search read
them; its outputs are not overwritten before they were copied out).  This is
the double buffer of the reference's GPU path (PAPER.md:1024-1031,
SPEC.md:436) with both directions of the PCIe copy hidden.
"""
from __future__ import annotations


class HostPipeline:
    def __init__(self, search_fn, k: int, max_batch: int, d_full: int = 128, device: int = 0, slots: int = 2):
        """search_fn(queries_cuda, (ids, sqdist, len)) runs on the current stream; it may return
        the (lo, hi) rows it produced (a routed sharded aggregate), only those are read back."""
        import torch
        self.torch = torch
        self.search_fn = search_fn
        dev = torch.device("cuda", device)
        self.dev = dev
        self.h2d = torch.cuda.Stream(device=dev)
        self.comp = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        self.slots = slots
        self.dq = [torch.empty((max_batch, d_full), dtype=torch.uint8, device=dev) for _ in range(slots)]
        self.out = [(torch.empty((max_batch, k), dtype=torch.uint64, device=dev),
                     torch.empty((max_batch, k), dtype=torch.uint32, device=dev),
                     torch.empty((max_batch,), dtype=torch.uint32, device=dev)) for _ in range(slots)]

    def run(self, host_batches, host_outs, start_event=None, end_event=None):
        """Search every pinned host batch into the matching pinned host outputs.

        start_event / end_event (optional CUDA timing events) bracket the whole
        run on the device: start before the first H2D, end after the last D2H."""
        torch = self.torch
        ev_read = [None] * self.slots    # search of the slot's last batch has read its queries
        ev_copied = [None] * self.slots  # the slot's last results are on the host
        if start_event is not None:
            start_event.record(self.h2d)
        for b, hq in enumerate(host_batches):
            s = b % self.slots
            n = int(hq.shape[0])
            with torch.cuda.stream(self.h2d):
                if ev_read[s] is not None:
                    self.h2d.wait_event(ev_read[s])
                self.dq[s][:n].copy_(hq, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(self.h2d)
            with torch.cuda.stream(self.comp):
                self.comp.wait_event(loaded)
                if ev_copied[s] is not None:
                    self.comp.wait_event(ev_copied[s])
                outs = tuple(o[:n] for o in self.out[s])
                rows = self.search_fn(self.dq[s][:n], outs)
                routed = isinstance(rows, tuple) and len(rows) == 2 and all(isinstance(x, int) for x in rows)
                lo, hi = rows if routed else (0, n)
                done = torch.cuda.Event()
                done.record(self.comp)
                ev_read[s] = done
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(done)
                for h, d in zip(host_outs[b], outs):
                    h[lo:hi].copy_(d[lo:hi], non_blocking=True)
                copied = torch.cuda.Event()
                copied.record(self.d2h)
                ev_copied[s] = copied
        if end_event is not None:
            end_event.record(self.d2h)
        self.d2h.synchronize()
