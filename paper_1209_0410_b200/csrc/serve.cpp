// serve.cpp -- the GPU batch-size controller: the reference's DTAHE scheduler
// (Alg. 3) re-targeted at a GPU-only
// search path, in the host C++ layer behind the C ABI.
//
// DTAHE moves each arriving query either to a CPU core (lines 3-4) or into the
// current GPU buffer, and queues the buffer on the device when "ready < CC and
// the GPU is idle, or the buffer is full" (lines 9-10), with at most two
// buffers alive (double buffering).  The north star has no CPU
// branch (CC = 0), which leaves the buffer rule:
//
//   with a slot free (at most `slots` batches in flight), launch
//   min(waiting, max_batch) queries when the device is idle (DTAHE "GPU
//   idle"), or the queue holds >= min_batch queries ("buffer full"), or the
//   oldest waiting query has waited max_wait;  otherwise keep buffering.
//
// Batch size follows the load: one query per batch when lightly loaded,
// growing towards max_batch near saturation.  Queries are served FIFO (no
// reordering), each exactly once (work conservation, :491).
//
// A batch is H2D (pinned / registered host queries -> the slot's device
// buffer, copy stream) -> search (compute stream; one index, or a shard group:
// per-GPU search + exchange + merge) -> D2H (results -> host, copy
// stream); events order slot reuse, so batch b+1's upload and batch b-1's
// download overlap batch b's search.  A query's response time runs from its
// arrival to the moment its results are in host memory (the CUDA event after
// the D2H, read on the device clock aligned with the host clock at start).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hcg_host.hpp"

namespace hcg {
namespace {

#define SV_CUDA(call)                                                                                   \
    do {                                                                                                \
        const cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return set_error(HCG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

using Clock = std::chrono::steady_clock;

// Batches up to this size may run side by side (launch): the one-CTA-per-query
// search path's range (search.cu kSmallBatch).
constexpr uint32_t kServeSmallBatch = 512;
constexpr uint32_t kSideSlots = 8;  // slots beyond pol.slots for side batches

double seconds_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

struct Slot {
    uint8_t* dq = nullptr;     // device queries, max_batch x d_full
    uint64_t* dids = nullptr;  // device results
    uint32_t* dsq = nullptr;
    uint32_t* dlen = nullptr;
    cudaEvent_t loaded = nullptr, searched = nullptr, copied = nullptr;  // copied: timing event
    cudaStream_t own = nullptr;  // the whole batch when it runs beside others (see launch)
    bool side = false;           // launched on `own`
    uint32_t cap = 0;            // queries it holds
    bool busy = false;
    uint64_t first = 0;  // sequence number of the batch's first query
    uint32_t count = 0;
};

}  // namespace
}  // namespace hcg

using namespace hcg;

struct hcg_server {
    const hcg_index* ix = nullptr;
    hcg_shard_group* group = nullptr;
    int device = 0;
    uint32_t d_full = 0, k = 0, depth = 0;
    uint32_t sms = 0;  // SM count: the budget for batches that run side by side
    hcg_server_policy pol{};
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    std::vector<Slot> slots;
    cudaEvent_t start = nullptr;  // device-clock origin
    Clock::time_point t0;         // host-clock origin (aligned with `start`)
    std::mutex run_mu;            // one replay / online session at a time
    // online mode
    std::thread worker;
    std::mutex mu;
    std::condition_variable cv_in, cv_out;
    bool stop = false;
    uint8_t* in_ring = nullptr;   // pinned: capacity x d_full
    uint64_t* out_ids = nullptr;  // pinned: capacity x k
    uint32_t* out_sq = nullptr;
    uint32_t* out_len = nullptr;
    double* arrive = nullptr;     // capacity
    double* finish = nullptr;     // capacity (< 0: pending)
    uint64_t capacity = 0;
    uint64_t submitted = 0;       // sequence numbers handed out
    uint64_t reclaimed = 0;       // ring entries below this may be reused
    std::deque<std::pair<uint64_t, uint32_t>> open_tickets;  // (first, count) not yet waited
    hcg_status worker_rc = HCG_OK;
};

namespace {

hcg_status engine_init(hcg_server* s) {
    SV_CUDA(cudaSetDevice(s->device));
    int sms = 0;
    SV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    s->sms = uint32_t(sms);
    SV_CUDA(cudaStreamCreateWithFlags(&s->h2d, cudaStreamNonBlocking));
    SV_CUDA(cudaStreamCreateWithFlags(&s->comp, cudaStreamNonBlocking));
    SV_CUDA(cudaStreamCreateWithFlags(&s->d2h, cudaStreamNonBlocking));
    SV_CUDA(cudaEventCreate(&s->start));
    s->slots.resize(s->pol.slots + (s->pol.slots >= 2 ? kSideSlots : 0));
    for (size_t i = 0; i < s->slots.size(); ++i) {
        Slot& sl = s->slots[i];
        // the pipeline's slots hold max_batch queries, the extra ones a side batch
        sl.cap = i < s->pol.slots ? s->pol.max_batch : std::min(s->pol.max_batch, kServeSmallBatch);
        const size_t B = sl.cap;
        SV_CUDA(cudaMalloc(&sl.dq, B * s->d_full));
        SV_CUDA(cudaMalloc(&sl.dids, B * s->k * 8));
        SV_CUDA(cudaMalloc(&sl.dsq, B * s->k * 4));
        SV_CUDA(cudaMalloc(&sl.dlen, B * 4));
        SV_CUDA(cudaEventCreateWithFlags(&sl.loaded, cudaEventDisableTiming));
        SV_CUDA(cudaEventCreateWithFlags(&sl.searched, cudaEventDisableTiming));
        SV_CUDA(cudaEventCreate(&sl.copied));
        SV_CUDA(cudaStreamCreateWithFlags(&sl.own, cudaStreamNonBlocking));
    }
    return HCG_OK;
}

void engine_free(hcg_server* s) {
    cudaSetDevice(s->device);
    if (s->comp) cudaStreamSynchronize(s->comp);
    if (s->d2h) cudaStreamSynchronize(s->d2h);
    for (auto& sl : s->slots) {
        cudaFree(sl.dq);
        cudaFree(sl.dids);
        cudaFree(sl.dsq);
        cudaFree(sl.dlen);
        if (sl.loaded) cudaEventDestroy(sl.loaded);
        if (sl.searched) cudaEventDestroy(sl.searched);
        if (sl.copied) cudaEventDestroy(sl.copied);
        if (sl.own) {
            cudaStreamSynchronize(sl.own);
            cudaStreamDestroy(sl.own);
        }
    }
    if (s->start) cudaEventDestroy(s->start);
    for (cudaStream_t st : {s->h2d, s->comp, s->d2h})
        if (st) cudaStreamDestroy(st);
    cudaFreeHost(s->in_ring);
    cudaFreeHost(s->out_ids);
    cudaFreeHost(s->out_sq);
    cudaFreeHost(s->out_len);
    delete[] s->arrive;
    delete[] s->finish;
}

// Align the device clock (event `start`) with the host clock t0.
hcg_status clock_sync(hcg_server* s) {
    SV_CUDA(cudaStreamSynchronize(s->comp));
    SV_CUDA(cudaEventRecord(s->start, s->comp));
    SV_CUDA(cudaEventSynchronize(s->start));
    s->t0 = Clock::now();
    return HCG_OK;
}

// Enqueue one batch: `count` queries from host memory q (pinned or registered)
// into slot `si`; results to host memory (ids / sq / len, count rows).  A side
// batch (pick) runs H2D -> search -> D2H on the slot's own stream; any other
// runs on s->comp after the side batches in flight, its copies overlapped on
// s->h2d / s->d2h.  The slot's events order its reuse either way.
hcg_status launch(hcg_server* s, uint32_t si, bool side, const uint8_t* q, uint32_t count, uint64_t* ids,
                  uint32_t* sq, uint32_t* len) {
    Slot& sl = s->slots[si];
    const size_t k = s->k;
    cudaStream_t up = side ? sl.own : s->h2d, cs = side ? sl.own : s->comp, down = side ? sl.own : s->d2h;
    if (!side)
        for (const auto& o : s->slots)
            if (o.busy && o.side) SV_CUDA(cudaStreamWaitEvent(cs, o.searched, 0));
    // upload (after this slot's previous search read its queries)
    SV_CUDA(cudaStreamWaitEvent(up, sl.searched, 0));
    SV_CUDA(cudaMemcpyAsync(sl.dq, q, size_t(count) * s->d_full, cudaMemcpyHostToDevice, up));
    SV_CUDA(cudaEventRecord(sl.loaded, up));
    // search (after the upload, and after this slot's previous results left)
    if (cs != up) SV_CUDA(cudaStreamWaitEvent(cs, sl.loaded, 0));
    SV_CUDA(cudaStreamWaitEvent(cs, sl.copied, 0));
    if (s->group)
        HCG_RET_IF(hcg_shard_group_search(s->group, sl.dq, count, s->k, s->depth, sl.dids, sl.dsq, sl.dlen, cs));
    else
        HCG_RET_IF(hcg_search(s->ix, sl.dq, count, s->k, s->depth, sl.dids, sl.dsq, sl.dlen, cs));
    SV_CUDA(cudaEventRecord(sl.searched, cs));
    // download; the copy event is the batch's completion
    if (down != cs) SV_CUDA(cudaStreamWaitEvent(down, sl.searched, 0));
    SV_CUDA(cudaMemcpyAsync(ids, sl.dids, count * k * 8, cudaMemcpyDeviceToHost, down));
    SV_CUDA(cudaMemcpyAsync(sq, sl.dsq, count * k * 4, cudaMemcpyDeviceToHost, down));
    SV_CUDA(cudaMemcpyAsync(len, sl.dlen, size_t(count) * 4, cudaMemcpyDeviceToHost, down));
    SV_CUDA(cudaEventRecord(sl.copied, down));
    sl.busy = true;
    sl.side = side;
    sl.count = count;
    return HCG_OK;
}

// Completed? -> *t = completion time in seconds since t0 (device clock).
hcg_status poll(hcg_server* s, uint32_t si, bool* done, double* t) {
    Slot& sl = s->slots[si];
    *done = false;
    const cudaError_t e = cudaEventQuery(sl.copied);
    if (e == cudaErrorNotReady) return HCG_OK;
    if (e != cudaSuccess) return set_error(HCG_ECUDA, std::string("batch: ") + cudaGetErrorString(e));
    float ms = 0.0f;
    SV_CUDA(cudaEventElapsedTime(&ms, s->start, sl.copied));
    *t = double(ms) * 1e-3;
    *done = true;
    sl.busy = false;
    return HCG_OK;
}

bool any_busy(const hcg_server* s) {
    for (const auto& sl : s->slots)
        if (sl.busy) return true;
    return false;
}

// Slot for a batch of `count` queries, or -1 (keep buffering).  The paper's
// pipeline keeps pol.slots batches in flight, one after another on the device.
// At light load a batch is small and its search takes one SM per query: such
// a batch runs beside the other small ones in flight (*side) while their
// queries fit one CTA per SM and no large batch is in flight; the side
// batches together count as one stage of the pipeline.
int pick(const hcg_server* s, uint32_t count, bool* side) {
    uint32_t side_q = 0, stages = 0;
    bool any_side = false;
    int free_full = -1, free_side = -1;  // a free pipeline slot / a free extra slot
    for (size_t i = 0; i < s->slots.size(); ++i) {
        const Slot& o = s->slots[i];
        if (!o.busy) {
            int& f = i < s->pol.slots ? free_full : free_side;
            if (f < 0) f = int(i);
        } else if (o.side) {
            side_q += o.count;
            any_side = true;
        } else {
            ++stages;
        }
    }
    *side = !s->group && s->pol.slots >= 2 && stages == 0 && count <= kServeSmallBatch && side_q + count <= s->sms;
    if (*side) return free_side >= 0 ? free_side : free_full;
    return stages + (any_side ? 1 : 0) < s->pol.slots ? free_full : -1;
}

// The dispatch rule (Alg. 3 lines 9-10 with CC = 0, plus max_wait).
bool should_launch(const hcg_server* s, uint64_t waiting, double oldest_wait) {
    return waiting > 0 && (!any_busy(s) || waiting >= s->pol.min_batch || oldest_wait >= s->pol.max_wait_s);
}

// Pin a caller buffer for async copies for the duration of a call.
struct HostPin {
    void* p = nullptr;
    explicit HostPin(const void* ptr, size_t bytes) {
        if (!ptr || !bytes) return;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type != cudaMemoryTypeUnregistered) return;
        cudaGetLastError();
        if (cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault) == cudaSuccess)
            p = const_cast<void*>(ptr);
        else
            cudaGetLastError();  // pageable copies still work (synchronously staged by the driver)
    }
    ~HostPin() {
        if (p) cudaHostUnregister(p);
    }
};

// ----------------------------------------------------------------- online ----
void worker_loop(hcg_server* s) {
    cudaSetDevice(s->device);
    uint64_t head = 0;  // first query not yet dispatched
    while (true) {
        // retire finished batches
        for (uint32_t si = 0; si < s->slots.size(); ++si) {
            Slot& sl = s->slots[si];
            if (!sl.busy) continue;
            bool done = false;
            double t = 0;
            if (poll(s, si, &done, &t) != HCG_OK) {
                std::lock_guard<std::mutex> g(s->mu);
                s->worker_rc = HCG_ECUDA;
                s->cv_out.notify_all();
                return;
            }
            if (done) {
                std::lock_guard<std::mutex> g(s->mu);
                for (uint64_t i = sl.first; i < sl.first + sl.count; ++i) s->finish[i % s->capacity] = t;
                s->cv_out.notify_all();
                s->cv_in.notify_all();
            }
        }
        std::unique_lock<std::mutex> lk(s->mu);
        if (s->stop && head == s->submitted && !any_busy(s)) return;
        const uint64_t waiting = s->submitted - head;
        const double now = seconds_since(s->t0);
        const double oldest = waiting ? now - s->arrive[head % s->capacity] : 0.0;
        // a batch never wraps the ring: it ends at the ring's end at the latest
        const uint64_t ring_off = head % s->capacity;
        const uint32_t count = uint32_t(std::min<uint64_t>({waiting, s->pol.max_batch, s->capacity - ring_off}));
        bool side = false;
        const int si = should_launch(s, waiting, oldest) ? pick(s, count, &side) : -1;
        if (si >= 0) {
            lk.unlock();
            Slot& sl = s->slots[si];
            sl.first = head;
            const hcg_status rc = launch(s, uint32_t(si), side, s->in_ring + ring_off * s->d_full, count,
                                         s->out_ids + ring_off * s->k, s->out_sq + ring_off * s->k,
                                         s->out_len + ring_off);
            if (rc != HCG_OK) {
                std::lock_guard<std::mutex> g(s->mu);
                s->worker_rc = rc;
                s->cv_out.notify_all();
                return;
            }
            head += count;
            continue;
        }
        if (waiting == 0 && !any_busy(s)) {
            s->cv_in.wait_for(lk, std::chrono::milliseconds(2));  // idle: sleep until a submit
            continue;
        }
        lk.unlock();
        std::this_thread::yield();  // batches finish in 0.05 - 10 ms: poll
    }
}

}  // namespace

extern "C" {

hcg_status hcg_server_create(const hcg_index* index, hcg_shard_group* group, uint32_t k, uint32_t depth,
                             const hcg_server_policy* policy, hcg_server** out) {
    if (!out) return set_error(HCG_EINVAL, "null output handle");
    *out = nullptr;
    if ((index == nullptr) == (group == nullptr)) return set_error(HCG_EINVAL, "serve exactly one index or shard group");
    if (group && hcg_shard_group_local_shards(group) != hcg_shard_group_shards(group))
        return set_error(HCG_EINVAL, "the server drives a one-process shard group (a per-rank group's searches are collective)");
    if (k < 1 || depth < 1) return set_error(HCG_EINVAL, "k and probe_depth must be >= 1");
    if (k > HCG_MAX_K) return set_error(HCG_ECAPACITY, "k exceeds HCG_MAX_K");
    hcg_server_policy p{8192, 1, 0.0, 2};
    if (policy) p = *policy;
    if (p.max_batch < 1 || p.slots < 1 || p.slots > 8 || p.min_batch < 1 || !(p.max_wait_s >= 0.0))
        return set_error(HCG_EINVAL, "policy: max_batch >= 1, 1 <= slots <= 8, min_batch >= 1, max_wait >= 0");
    auto* s = new hcg_server;
    s->ix = index;
    s->group = group;
    s->k = k;
    s->depth = depth;
    s->pol = p;
    hcg_scheme sc;
    uint32_t alen = 0;
    hcg_status rc = HCG_OK;
    if (index) {
        rc = hcg_describe(index, &sc, nullptr, nullptr, &alen);
        if (rc == HCG_OK && sc.dtype != HCG_U8) rc = set_error(HCG_EINVAL, "the server serves u8 indexes");
        s->device = hcg_index_device(index);
        s->d_full = sc.d_full;
    } else {
        s->device = hcg_shard_group_device(group);
        s->d_full = hcg_shard_group_dims(group);
    }
    if (rc == HCG_OK) rc = engine_init(s);
    if (rc != HCG_OK) {
        engine_free(s);
        delete s;
        return rc;
    }
    *out = s;
    return HCG_OK;
}

hcg_status hcg_server_free(hcg_server* s) {
    if (!s) return HCG_OK;
    if (s->worker.joinable()) {
        {
            std::lock_guard<std::mutex> g(s->mu);
            s->stop = true;
        }
        s->cv_in.notify_all();
        s->worker.join();
    }
    engine_free(s);
    delete s;
    return HCG_OK;
}

hcg_status hcg_server_replay(hcg_server* s, const uint8_t* queries, uint32_t nq, const double* arrival_s,
                             uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, double* latency_s,
                             uint32_t* batch_sizes, uint32_t* n_batches) {
    if (!s) return set_error(HCG_EINVAL, "null server");
    if (nq == 0) {
        if (n_batches) *n_batches = 0;
        return HCG_OK;
    }
    if (!queries || !arrival_s || !out_ids || !out_sqdist || !out_len || !latency_s)
        return set_error(HCG_EINVAL, "null buffer");
    for (uint32_t i = 1; i < nq; ++i)
        if (!(arrival_s[i] >= arrival_s[i - 1])) return set_error(HCG_EINVAL, "arrivals must be non-decreasing");
    std::unique_lock<std::mutex> session(s->run_mu, std::try_to_lock);
    if (!session.owns_lock() || s->worker.joinable()) return set_error(HCG_EINVAL, "server busy (online session)");
    SV_CUDA(cudaSetDevice(s->device));
    const size_t k = s->k;
    HostPin pq(queries, size_t(nq) * s->d_full), pi(out_ids, size_t(nq) * k * 8), ps(out_sqdist, size_t(nq) * k * 4),
        pl(out_len, size_t(nq) * 4);
    std::vector<double> finish(nq, -1.0);
    std::vector<uint32_t> sizes;
    HCG_RET_IF(clock_sync(s));
    uint64_t head = 0, arrived = 0, done = 0;
    while (done < nq) {
        const double now = seconds_since(s->t0);
        while (arrived < nq && arrival_s[arrived] <= now) ++arrived;
        for (uint32_t si = 0; si < s->slots.size(); ++si) {
            Slot& sl = s->slots[si];
            if (!sl.busy) continue;
            bool fin = false;
            double t = 0;
            HCG_RET_IF(poll(s, si, &fin, &t));
            if (fin) {
                for (uint64_t i = sl.first; i < sl.first + sl.count; ++i) finish[i] = t;
                done += sl.count;
            }
        }
        const uint64_t waiting = arrived - head;
        const uint32_t count = uint32_t(std::min<uint64_t>(waiting, s->pol.max_batch));
        bool side = false;
        const int si = should_launch(s, waiting, waiting ? now - arrival_s[head] : 0.0) ? pick(s, count, &side) : -1;
        if (si >= 0) {
            s->slots[si].first = head;
            HCG_RET_IF(launch(s, uint32_t(si), side, queries + head * s->d_full, count, out_ids + head * k,
                              out_sqdist + head * k, out_len + head));
            sizes.push_back(count);
            head += count;
            continue;
        }
        // nothing to launch: sleep until the next arrival when the device is idle, else poll
        if (!any_busy(s) && arrived < nq) {
            const double dt = arrival_s[arrived] - seconds_since(s->t0);
            if (dt > 300e-6) std::this_thread::sleep_for(std::chrono::duration<double>(dt - 200e-6));
        } else {
            std::this_thread::yield();
        }
    }
    for (uint32_t i = 0; i < nq; ++i) latency_s[i] = finish[i] - arrival_s[i];
    if (n_batches) *n_batches = uint32_t(sizes.size());
    if (batch_sizes) std::memcpy(batch_sizes, sizes.data(), sizes.size() * 4);
    return HCG_OK;
}

hcg_status hcg_server_start(hcg_server* s, uint64_t capacity) {
    if (!s) return set_error(HCG_EINVAL, "null server");
    if (capacity < s->pol.max_batch) return set_error(HCG_EINVAL, "capacity must be >= max_batch");
    std::lock_guard<std::mutex> g(s->mu);
    if (s->worker.joinable()) return set_error(HCG_EINVAL, "server already started");
    SV_CUDA(cudaSetDevice(s->device));
    s->capacity = capacity;
    SV_CUDA(cudaMallocHost(&s->in_ring, capacity * s->d_full));
    SV_CUDA(cudaMallocHost(&s->out_ids, capacity * s->k * 8));
    SV_CUDA(cudaMallocHost(&s->out_sq, capacity * s->k * 4));
    SV_CUDA(cudaMallocHost(&s->out_len, capacity * 4));
    s->arrive = new double[capacity];
    s->finish = new double[capacity];
    HCG_RET_IF(clock_sync(s));
    s->stop = false;
    s->worker = std::thread(worker_loop, s);
    return HCG_OK;
}

hcg_status hcg_server_submit(hcg_server* s, const uint8_t* queries, uint32_t nq, uint64_t* ticket) {
    if (!s || !ticket) return set_error(HCG_EINVAL, "null argument");
    if (nq == 0 || !queries) return set_error(HCG_EINVAL, "empty submission");
    std::unique_lock<std::mutex> lk(s->mu);
    if (!s->worker.joinable()) return set_error(HCG_EINVAL, "server not started (hcg_server_start)");
    if (nq > s->capacity) return set_error(HCG_ECAPACITY, "submission larger than the server's ring");
    // block while the ring is full of queries nobody collected yet
    s->cv_out.wait(lk, [&] { return s->worker_rc != HCG_OK || s->submitted + nq - s->reclaimed <= s->capacity; });
    if (s->worker_rc != HCG_OK) return set_error(s->worker_rc, "server worker failed");
    const uint64_t first = s->submitted;
    const double now = seconds_since(s->t0);
    for (uint32_t i = 0; i < nq; ++i) {
        const uint64_t r = (first + i) % s->capacity;
        std::memcpy(s->in_ring + r * s->d_full, queries + size_t(i) * s->d_full, s->d_full);
        s->arrive[r] = now;
        s->finish[r] = -1.0;
    }
    s->submitted += nq;
    s->open_tickets.emplace_back(first, nq);
    *ticket = first;
    s->cv_in.notify_all();
    return HCG_OK;
}

hcg_status hcg_server_wait(hcg_server* s, uint64_t ticket, uint64_t* out_ids, uint32_t* out_sqdist,
                           uint32_t* out_len, double* latency_s) {
    if (!s) return set_error(HCG_EINVAL, "null server");
    std::unique_lock<std::mutex> lk(s->mu);
    auto it = std::find_if(s->open_tickets.begin(), s->open_tickets.end(),
                           [&](const std::pair<uint64_t, uint32_t>& t) { return t.first == ticket; });
    if (it == s->open_tickets.end()) return set_error(HCG_EINVAL, "unknown or already collected ticket");
    const uint32_t nq = it->second;
    auto ready = [&] {
        if (s->worker_rc != HCG_OK) return true;
        for (uint32_t i = 0; i < nq; ++i)
            if (s->finish[(ticket + i) % s->capacity] < 0) return false;
        return true;
    };
    s->cv_out.wait(lk, ready);
    if (s->worker_rc != HCG_OK) return set_error(s->worker_rc, "server worker failed");
    const size_t k = s->k;
    for (uint32_t i = 0; i < nq; ++i) {
        const uint64_t r = (ticket + i) % s->capacity;
        if (out_ids) std::memcpy(out_ids + i * k, s->out_ids + r * k, k * 8);
        if (out_sqdist) std::memcpy(out_sqdist + i * k, s->out_sq + r * k, k * 4);
        if (out_len) out_len[i] = s->out_len[r];
        if (latency_s) latency_s[i] = s->finish[r] - s->arrive[r];
    }
    s->open_tickets.erase(it);
    // reclaim the ring up to the oldest ticket still open
    s->reclaimed = s->open_tickets.empty() ? s->submitted : s->open_tickets.front().first;
    for (const auto& t : s->open_tickets) s->reclaimed = std::min(s->reclaimed, t.first);
    s->cv_out.notify_all();
    return HCG_OK;
}

}  // extern "C"
