// shard.cu -- the hypershard partition / aggregate behind
// the C ABI: a shard group holds G Multicurves shards (global id i on shard
// i mod G, local slot i / G) and one NCCL communicator per shard.  A search
// broadcasts the query batch, runs the per-shard search at the per-shard
// probe depth on every GPU (hcg_search_packed: packed (sqdist << 32 | gid)
// top-k), all-gathers the packed lists over NVLink (ncclAllGather, B x k x 8
// bytes per shard) and merges them by (distance, id) with K4 (k_merge),
// truncated to k.
//
// Two ways to drive it:
//   * one process, G GPUs (hcg_shard_group_build / _adopt): one stream per
//     GPU, the merged result on the first GPU; with NVLink peer access the
//     exchange is fused into the search: every shard's kernel stores its
//     packed top-k straight into the first GPU's gathered buffer (no
//     collective, no copy); otherwise ncclCommInitAll + ncclAllGather;
//   * one process per GPU (hcg_shard_group_join): ncclCommInitRank from an id
//     the caller distributed (hcg_nccl_unique_id); every rank gets the result.
//
// NCCL is resolved at run time (dlopen) rather than linked: a process that
// already loaded libnccl.so.2 (PyTorch does, at import) shares that copy, and
// libhcg.so loads on machines without NCCL as long as no group is created.
#include <dlfcn.h>
#include <nccl.h>  // types only

#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "hcg_host.hpp"

namespace hcg {
namespace {

struct NcclApi {
    bool loaded = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // an already-loaded copy first (PyTorch's), then $HCG_NCCL_LIB, then the system one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = getenv("HCG_NCCL_LIB");
        if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn) ok = false;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.AllGather, "ncclAllGather");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GetVersion, "ncclGetVersion");
        if (!ok) {
            api.err = "libnccl.so.2 lacks a required symbol";
            return;
        }
        api.loaded = true;
    });
    return api;
}

hcg_status nccl_ready() {
    NcclApi& n = nccl();
    return n.loaded ? HCG_OK : set_error(HCG_ECUDA, n.err);
}

hcg_status nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return HCG_OK;
    return set_error(HCG_ECUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

#define SG_CUDA(call)                                                                                   \
    do {                                                                                                \
        const cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return set_error(HCG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    hcg_status reserve(size_t bytes) {
        if (bytes <= cap) return HCG_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return set_error(HCG_ENOMEM, "shard group buffer of " + std::to_string(bytes) + " bytes");
        }
        cap = bytes;
        return HCG_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct SetDev {
    int prev = -1;
    explicit SetDev(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~SetDev() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace
}  // namespace hcg

using namespace hcg;

struct hcg_shard_group {
    uint32_t G = 0;      // shards in the group
    uint32_t first = 0;  // index of this process's first shard (rank in per-process mode)
    uint64_t n_total = 0;
    uint32_t d_full = 0;
    std::vector<hcg_index*> ix;  // this process's shards
    bool own = false;            // free the shards with the group
    std::vector<int> dev;
    std::vector<ncclComm_t> comm;
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> done;
    std::vector<DevBuf> dq, packed, gathered;
    cudaEvent_t ev_in = nullptr;  // on dev[0]: the caller's stream reached the search
    cudaEvent_t merged = nullptr; // on dev[0]: the last merge has read the gathered lists
    bool p2p = false;             // one process, every GPU writes into dev[0]'s memory over NVLink
    std::mutex mu;
};

namespace {

void destroy(hcg_shard_group* g) {
    if (!g) return;
    for (size_t r = 0; r < g->dev.size(); ++r) {
        SetDev sd(g->dev[r]);
        if (r < g->st.size() && g->st[r]) cudaStreamSynchronize(g->st[r]);
        if (r < g->comm.size() && g->comm[r] && nccl().loaded) nccl().CommDestroy(g->comm[r]);
        if (r < g->dq.size()) g->dq[r].release();
        if (r < g->packed.size()) g->packed[r].release();
        if (r < g->gathered.size()) g->gathered[r].release();
        if (r < g->done.size() && g->done[r]) cudaEventDestroy(g->done[r]);
        if (r < g->st.size() && g->st[r]) cudaStreamDestroy(g->st[r]);
        if (r == 0 && g->ev_in) cudaEventDestroy(g->ev_in);
        if (r == 0 && g->merged) cudaEventDestroy(g->merged);
        if (g->own && r < g->ix.size() && g->ix[r]) hcg_free(g->ix[r]);
    }
    delete g;
}

// Streams, events and buffers of the local shards (comms are made by the caller).
hcg_status init_local(hcg_shard_group* g) {
    const size_t L = g->ix.size();
    g->st.assign(L, nullptr);
    g->done.assign(L, nullptr);
    g->dq.resize(L);
    g->packed.resize(L);
    g->gathered.resize(L);
    for (size_t r = 0; r < L; ++r) {
        SetDev sd(g->dev[r]);
        SG_CUDA(cudaStreamCreateWithFlags(&g->st[r], cudaStreamNonBlocking));
        SG_CUDA(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
        if (r == 0) SG_CUDA(cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
        if (r == 0) SG_CUDA(cudaEventCreateWithFlags(&g->merged, cudaEventDisableTiming));
    }
    return HCG_OK;
}

hcg_status check_shard(const hcg_index* ix, uint32_t shard, uint32_t G) {
    hcg_scheme s;
    uint32_t alen = 0;
    HCG_RET_IF(hcg_describe(ix, &s, nullptr, nullptr, &alen));
    if (s.dtype != HCG_U8) return set_error(HCG_EINVAL, "shard groups hold u8 indexes (packed results)");
    uint64_t base = 0, stride = 0;
    hcg_index_ids(ix, &base, &stride);
    if (base != shard || stride != G)
        return set_error(HCG_EINVAL, "shard " + std::to_string(shard) + " of " + std::to_string(G) +
                                         " must hold ids " + std::to_string(shard) + " + s * " + std::to_string(G));
    return HCG_OK;
}

int ptr_device(const void* p) {
    cudaPointerAttributes at;
    if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? at.device : -1;
}

}  // namespace

extern "C" {

hcg_status hcg_nccl_unique_id(hcg_nccl_id* out) {
    if (!out) return set_error(HCG_EINVAL, "null id");
    HCG_RET_IF(nccl_ready());
    static_assert(sizeof(hcg_nccl_id) == sizeof(ncclUniqueId), "NCCL unique id size");
    ncclUniqueId id;
    HCG_RET_IF(nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
    std::memcpy(out, &id, sizeof(id));
    return HCG_OK;
}

hcg_status hcg_shard_group_adopt(uint32_t G, hcg_index* const* shards, hcg_shard_group** out) {
    if (!out) return set_error(HCG_EINVAL, "null output handle");
    *out = nullptr;
    if (G < 1 || !shards) return set_error(HCG_EINVAL, "need G >= 1 shards");
    for (uint32_t r = 0; r < G; ++r) {
        if (!shards[r]) return set_error(HCG_EINVAL, "null shard");
        HCG_RET_IF(check_shard(shards[r], r, G));
        for (uint32_t s = 0; s < r; ++s)
            if (hcg_index_device(shards[s]) == hcg_index_device(shards[r]))
                return set_error(HCG_EINVAL, "two shards on one device");
    }
    HCG_RET_IF(nccl_ready());
    auto* g = new hcg_shard_group;
    g->G = G;
    g->first = 0;
    g->own = true;
    for (uint32_t r = 0; r < G; ++r) {
        g->ix.push_back(shards[r]);
        g->dev.push_back(hcg_index_device(shards[r]));
        g->n_total += hcg_size(shards[r]);
    }
    hcg_scheme s;
    uint32_t alen = 0;
    hcg_describe(shards[0], &s, nullptr, nullptr, &alen);
    g->d_full = s.d_full;
    hcg_status rc = init_local(g);
    if (rc == HCG_OK) {
        g->comm.assign(G, nullptr);
        rc = nccl_check(nccl().CommInitAll(g->comm.data(), int(G), g->dev.data()), "ncclCommInitAll");
    }
    // Fused exchange: when every GPU can write the first GPU's memory (NVLink
    // peers), each shard's search kernel stores its packed top-k straight
    // into the first GPU's gathered buffer -- the transfer happens in the
    // producing kernel's epilogue, no collective and no copy.
    if (rc == HCG_OK && G > 1 && !knob("HCG_SHARD_NCCL")) {
        bool ok = true;
        for (uint32_t r = 1; r < G && ok; ++r) {
            int can = 0;
            ok = cudaDeviceCanAccessPeer(&can, g->dev[r], g->dev[0]) == cudaSuccess && can;
            if (ok) {
                SetDev sd(g->dev[r]);
                const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[0], 0);
                ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
            }
            cudaGetLastError();
        }
        g->p2p = ok;
    }
    if (rc != HCG_OK) {
        g->own = false;  // the caller keeps its shards on failure
        destroy(g);
        return rc;
    }
    *out = g;
    return HCG_OK;
}

hcg_status hcg_shard_group_build(const hcg_scheme* scheme, const uint8_t* rows, uint64_t n_total, uint32_t G,
                                 const int* devices, hcg_shard_group** out) {
    if (!out) return set_error(HCG_EINVAL, "null output handle");
    *out = nullptr;
    if (!scheme) return set_error(HCG_EINVAL, "null scheme");
    if (scheme->dtype != HCG_U8) return set_error(HCG_EINVAL, "shard groups hold u8 indexes (packed results)");
    if (G < 1 || !devices) return set_error(HCG_EINVAL, "need G >= 1 devices");
    if (n_total && !rows) return set_error(HCG_EINVAL, "null rows");
    if (n_total && (n_total - 1) >= (1ull << 32)) return set_error(HCG_ECAPACITY, "packed results need ids < 2^32");
    const uint64_t rb = scheme->d_full;
    std::vector<hcg_index*> shards(G, nullptr);
    hcg_status rc = HCG_OK;
    for (uint32_t r = 0; r < G && rc == HCG_OK; ++r) {
        const uint64_t cnt = n_total > r ? (n_total - r + G - 1) / G : 0;
        SetDev sd(devices[r]);
        uint8_t* d = nullptr;
        if (cnt && cudaMalloc(&d, cnt * rb) != cudaSuccess) {
            cudaGetLastError();
            rc = set_error(HCG_ENOMEM, "shard staging");
            break;
        }
        // shard r = rows r, r + G, ...: one strided 2-D copy (host or device source)
        if (cnt && cudaMemcpy2D(d, rb, rows + r * rb, G * rb, rb, cnt, cudaMemcpyDefault) != cudaSuccess)
            rc = set_error(HCG_ECUDA, "shard rows copy");
        if (rc == HCG_OK) rc = hcg_build(scheme, d, cnt, r, G, devices[r], nullptr, &shards[r]);
        if (d) cudaFree(d);
    }
    if (rc == HCG_OK) rc = hcg_shard_group_adopt(G, shards.data(), out);
    if (rc != HCG_OK)
        for (auto* s : shards) hcg_free(s);
    return rc;
}

hcg_status hcg_shard_group_join(const hcg_nccl_id* id, uint32_t rank, uint32_t G, hcg_index* local,
                                hcg_shard_group** out) {
    if (!out) return set_error(HCG_EINVAL, "null output handle");
    *out = nullptr;
    if (!id || !local) return set_error(HCG_EINVAL, "null argument");
    if (G < 1 || rank >= G) return set_error(HCG_EINVAL, "rank must be < G");
    HCG_RET_IF(check_shard(local, rank, G));
    HCG_RET_IF(nccl_ready());
    auto* g = new hcg_shard_group;
    g->G = G;
    g->first = rank;
    g->own = false;  // the caller owns its shard
    g->ix.push_back(local);
    g->dev.push_back(hcg_index_device(local));
    g->n_total = 0;
    hcg_scheme s;
    uint32_t alen = 0;
    hcg_describe(local, &s, nullptr, nullptr, &alen);
    g->d_full = s.d_full;
    hcg_status rc = init_local(g);
    if (rc == HCG_OK) {
        SetDev sd(g->dev[0]);
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        g->comm.assign(1, nullptr);
        rc = nccl_check(nccl().CommInitRank(&g->comm[0], int(G), uid, int(rank)), "ncclCommInitRank");
    }
    if (rc != HCG_OK) {
        destroy(g);
        return rc;
    }
    *out = g;
    return HCG_OK;
}

hcg_status hcg_shard_group_free(hcg_shard_group* g) {
    destroy(g);
    return HCG_OK;
}

uint32_t hcg_shard_group_shards(const hcg_shard_group* g) { return g ? g->G : 0; }
int hcg_shard_group_device(const hcg_shard_group* g) { return g ? g->dev[0] : -1; }
uint32_t hcg_shard_group_local_shards(const hcg_shard_group* g) { return g ? uint32_t(g->ix.size()) : 0; }
uint32_t hcg_shard_group_dims(const hcg_shard_group* g) { return g ? g->d_full : 0; }

hcg_status hcg_shard_group_search(hcg_shard_group* g, const uint8_t* queries, uint32_t nq, uint32_t k,
                                  uint32_t shard_depth, uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len,
                                  void* stream) {
    if (!g) return set_error(HCG_EINVAL, "null shard group");
    if (k < 1) return set_error(HCG_EINVAL, "k must be >= 1");
    if (k > HCG_MAX_K) return set_error(HCG_ECAPACITY, "k exceeds HCG_MAX_K");
    if (shard_depth < 1) return set_error(HCG_EINVAL, "probe_depth must be >= 1");
    if (nq == 0) return HCG_OK;
    if (!queries || !out_ids || !out_sqdist || !out_len) return set_error(HCG_EINVAL, "null buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    const size_t L = g->ix.size();
    const size_t qbytes = size_t(nq) * g->d_full, pbytes = size_t(nq) * k * 8;
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    const int qdev = ptr_device(queries);
    {
        SetDev sd(g->dev[0]);
        SG_CUDA(cudaEventRecord(g->ev_in, caller));
    }
    if (g->p2p) {
        SetDev sd(g->dev[0]);
        HCG_RET_IF(g->gathered[0].reserve(pbytes * g->G));
    }
    // every shard answers the whole batch at the per-shard depth (IHLS)
    for (size_t r = 0; r < L; ++r) {
        SetDev sd(g->dev[r]);
        SG_CUDA(cudaStreamWaitEvent(g->st[r], g->ev_in, 0));
        const uint8_t* qr = queries;
        if (qdev >= 0 && qdev != g->dev[r]) {  // another GPU's memory: copy it over NVLink
            HCG_RET_IF(g->dq[r].reserve(qbytes));
            SG_CUDA(cudaMemcpyAsync(g->dq[r].p, queries, qbytes, cudaMemcpyDefault, g->st[r]));
            qr = static_cast<const uint8_t*>(g->dq[r].p);
        }
        uint64_t* out = nullptr;
        uint64_t* slice = nullptr;
        if (g->p2p) {
            // straight into slice r of the first GPU's gathered lists (NVLink
            // stores from the search kernel), after the last merge read them
            SG_CUDA(cudaStreamWaitEvent(g->st[r], g->merged, 0));
            slice = static_cast<uint64_t*>(g->gathered[0].p) + r * size_t(nq) * k;
            out = slice;
        }
        if (!out || hcg_size(g->ix[r]) == 0) {  // NCCL path, or an empty shard (padding written locally)
            HCG_RET_IF(g->packed[r].reserve(pbytes));
            if (!g->p2p) HCG_RET_IF(g->gathered[r].reserve(pbytes * g->G));
            out = static_cast<uint64_t*>(g->packed[r].p);
        }
        HCG_RET_IF(hcg_search_packed(g->ix[r], qr, nq, k, shard_depth, out, g->st[r]));
        if (slice && out != slice)
            SG_CUDA(cudaMemcpyPeerAsync(slice, g->dev[0], out, g->dev[r], pbytes, g->st[r]));
    }
    if (g->p2p) {
        for (size_t r = 1; r < L; ++r) {
            SetDev sd(g->dev[r]);
            SG_CUDA(cudaEventRecord(g->done[r], g->st[r]));
        }
        SetDev sd(g->dev[0]);
        for (size_t r = 1; r < L; ++r) SG_CUDA(cudaStreamWaitEvent(g->st[0], g->done[r], 0));
    } else {
        // aggregate: all-gather the packed top-k lists (B x k x 8 bytes per shard)
        HCG_RET_IF(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
        ncclResult_t nr = ncclSuccess;
        for (size_t r = 0; r < L && nr == ncclSuccess; ++r) {
            SetDev sd(g->dev[r]);
            nr = nccl().AllGather(g->packed[r].p, g->gathered[r].p, size_t(nq) * k, ncclUint64, g->comm[r], g->st[r]);
        }
        const ncclResult_t ne = nccl().GroupEnd();
        HCG_RET_IF(nccl_check(nr, "ncclAllGather"));
        HCG_RET_IF(nccl_check(ne, "ncclGroupEnd"));
    }
    // K4 on the first local GPU (every rank, in per-process mode)
    SetDev sd(g->dev[0]);
    HCG_RET_IF(hcg_merge_packed(static_cast<const uint64_t*>(g->gathered[0].p), g->G, nq, k, out_ids, out_sqdist,
                                out_len, g->dev[0], g->st[0]));
    SG_CUDA(cudaEventRecord(g->merged, g->st[0]));
    for (size_t r = 0; r < L; ++r) {
        SetDev sd2(g->dev[r]);
        SG_CUDA(cudaEventRecord(g->done[r], g->st[r]));
    }
    SetDev sd3(g->dev[0]);
    for (size_t r = 0; r < L; ++r) SG_CUDA(cudaStreamWaitEvent(caller, g->done[r], 0));
    return HCG_OK;
}

hcg_status hcg_shard_group_search_routed(hcg_shard_group* g, const uint8_t* queries, uint32_t nq, uint32_t k,
                                         uint32_t shard_depth, uint64_t* out_ids, uint32_t* out_sqdist,
                                         uint32_t* out_len, void* stream, uint32_t* block_first,
                                         uint32_t* block_count) {
    if (!g || !block_first || !block_count) return set_error(HCG_EINVAL, "null argument");
    if (g->ix.size() != 1 || g->G == 1) {  // one process holds every shard: it aggregates every query
        *block_first = 0;
        *block_count = nq;
        return hcg_shard_group_search(g, queries, nq, k, shard_depth, out_ids, out_sqdist, out_len, stream);
    }
    if (k < 1) return set_error(HCG_EINVAL, "k must be >= 1");
    if (k > HCG_MAX_K) return set_error(HCG_ECAPACITY, "k exceeds HCG_MAX_K");
    if (shard_depth < 1) return set_error(HCG_EINVAL, "probe_depth must be >= 1");
    const uint32_t G = g->G, me = g->first;
    auto lo = [&](uint32_t p) { return uint32_t(uint64_t(nq) * p / G); };
    *block_first = lo(me);
    *block_count = lo(me + 1) - lo(me);
    if (nq == 0) return HCG_OK;
    if (!queries || !out_ids || !out_sqdist || !out_len) return set_error(HCG_EINVAL, "null buffer");
    std::lock_guard<std::mutex> lock(g->mu);
    const size_t pbytes = size_t(nq) * k * 8;
    const uint32_t mine = *block_count;
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    SetDev sd(g->dev[0]);
    SG_CUDA(cudaEventRecord(g->ev_in, caller));
    SG_CUDA(cudaStreamWaitEvent(g->st[0], g->ev_in, 0));
    HCG_RET_IF(g->packed[0].reserve(pbytes));
    HCG_RET_IF(g->gathered[0].reserve(size_t(std::max<uint32_t>(mine, 1)) * k * 8 * G));
    uint64_t* packed = static_cast<uint64_t*>(g->packed[0].p);
    uint64_t* gathered = static_cast<uint64_t*>(g->gathered[0].p);
    HCG_RET_IF(hcg_search_packed(g->ix[0], queries, nq, k, shard_depth, packed, g->st[0]));
    // route: the partials of queries [lo(p), lo(p+1)) go to rank p, which
    // receives every shard's partials of its own block (1/G of an all-gather)
    HCG_RET_IF(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
    ncclResult_t nr = ncclSuccess;
    for (uint32_t p = 0; p < G && nr == ncclSuccess; ++p) {
        const size_t cnt_p = size_t(lo(p + 1) - lo(p)) * k;
        if (cnt_p) nr = nccl().Send(packed + size_t(lo(p)) * k, cnt_p, ncclUint64, int(p), g->comm[0], g->st[0]);
        if (nr == ncclSuccess && mine)
            nr = nccl().Recv(gathered + size_t(p) * mine * k, size_t(mine) * k, ncclUint64, int(p), g->comm[0],
                             g->st[0]);
    }
    const ncclResult_t ne = nccl().GroupEnd();
    HCG_RET_IF(nccl_check(nr, "ncclSend/ncclRecv"));
    HCG_RET_IF(nccl_check(ne, "ncclGroupEnd"));
    if (mine)
        HCG_RET_IF(hcg_merge_packed(gathered, G, mine, k, out_ids + size_t(*block_first) * k,
                                    out_sqdist + size_t(*block_first) * k, out_len + *block_first, g->dev[0],
                                    g->st[0]));
    SG_CUDA(cudaEventRecord(g->done[0], g->st[0]));
    SG_CUDA(cudaStreamWaitEvent(caller, g->done[0], 0));
    return HCG_OK;
}

}  // extern "C"
