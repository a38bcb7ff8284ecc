"""NCCL sharded search on >= 2 GPUs against the sharded CPU oracle (skipped on
a 1-GPU box; the host-side protocol is covered on CPU by test_sharded_gloo)."""
import os
import subprocess
import sys

import pytest

from hcg_testutil import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or _ngpus() < 2, reason="needs >= 2 GPUs")
def test_sharded_search_two_gpus():
    g = min(_ngpus(), 4)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
                          "--master-addr", "127.0.0.1", "--master-port", "29533",
                          os.path.join(ROOT, "tools", "sharded_check.py")],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "sharded ok" in out.stdout
