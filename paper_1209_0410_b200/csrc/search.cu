// search.cu -- batched query path on the B200 (Alg. 2).
//
//   K3a k_locate    : one thread per (query, curve): project + quantize + curve
//                     key (fused K1), compare against the curve's common key
//                     prefix, lower_bound over the sorted suffix keys
//                     (SubIndex::rank_of, multicurves.hpp:57-58) and the window
//                     begin (SubIndex::window, multicurves.hpp:60-63).
//   K3b k_union     : one CTA per query: the C windows' ids (cp.async,
//                     prefetched one query ahead) deduplicated in shared memory
//                     without atomics (candidate_union, multicurves.hpp:87-89);
//                     unique list -> HBM.  k_union_cas: the same with a global
//                     CAS table for very large curves x depth.
//   K3c k_gather    : one WARP per query: gather the unique candidate rows
//                     (8 lanes per 128-B row, 8 rows in flight per lane, next
//                     slots prefetched), exact squared L2 (vecio.cpp:87-95) with
//                     vabsdiff4 + dp4a, warp-register top-k on packed
//                     (sqdist<<32 | slot) == the reference's (distance, id)
//                     order (vecio.cpp:101-113).
//   K4  k_merge     : one warp per query, k-way merge of per-shard / per-chunk
//                     sorted lists (hypershard aggregate).
//   K5  k_brute     : exact kNN over all rows (brute_force_knn, vecio.cpp:115-122)
//                     for recall ground truth; chunked, then merged by K4.
#include <algorithm>
#include <cstdlib>

#include "hcg_internal.cuh"
#include "hcg_host.hpp"

namespace hcg {

// Device attributes of the refine launches, queried once per device.
struct DevInfo {
    int sms = 0;
};
inline const DevInfo& dev_info(int device) {
    static DevInfo info[64];
    DevInfo& d = info[device & 63];
    if (d.sms == 0) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        d.sms = sms;
    }
    return d;
}

__device__ __forceinline__ unsigned lanemask_lt_s() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ----------------------------------------------------------------- K3a ----
// -1 / 0 / 1: the stored suffix key at e vs the query suffix qs (ws words,
// most significant first).
template <int WSMAX>
__device__ __forceinline__ int suffix_cmp(const uint64_t* e, const uint64_t (&qs)[WSMAX], int ws) {
    int o = 0;
#pragma unroll
    for (int w = WSMAX - 1; w >= 0; --w) {
        if (o == 0 && w < ws) {
            const uint64_t ev = __ldg(e + w);
            o = ev < qs[w] ? -1 : (ev > qs[w] ? 1 : 0);
        }
    }
    return o;
}

// COOP: one WARP per (query, curve) and a 32-ary lower_bound (each round the
// lanes probe 32 splitters and a ballot narrows the range 33x: ~5 dependent
// loads at 10M instead of 24) -- the small-batch latency path.
// rank_of + window of query q on curve c (one thread, or one warp with COOP:
// every lane computes the key, the lanes split the 32-ary search).  lut: the
// view's cell table in shared memory.  Returns the window begin; *rank_out
// the rank.
#ifndef HCG_SMALL_COMPACT_KEY
#define HCG_SMALL_COMPACT_KEY true
#endif
// MFIX (8 or 16): every curve has exactly 16 dims and m = MFIX -- the key is
// built by the compile-time d16 transform alone (a fraction of the generic
// code: the latency kernel runs it from a cold instruction cache).
// SMEMIN: the query row and the assignment table sit in shared memory (plain
// loads; __ldg is global-only).
template <int DMAX, int WSMAX, bool COOP, class T, int MFIX = 0, bool SMEMIN = false>
__device__ __forceinline__ uint64_t locate_one(const LocateArgs& a, const uint32_t* lut, uint32_t q, uint32_t c,
                                               int lane, uint64_t* rank_out) {
    constexpr int WMAX = DMAX / 2 > kMaxKeyWords ? kMaxKeyWords : (DMAX / 2 < 1 ? 1 : DMAX / 2);
    const CurveDev& cv = a.curves[c];
    const int d = int(cv.dims);

    uint32_t x[DMAX];
    const T* row = reinterpret_cast<const T*>(a.queries + uint64_t(q) * a.pitch);
    const uint16_t* asg = a.assign + cv.off;
#pragma unroll
    for (int s = 0; s < DMAX; ++s) {
        if constexpr (SMEMIN)
            x[s] = s < d ? cell_of(row[asg[s]], lut, a.m, a.bad) : 0u;
        else
            x[s] = s < d ? cell_of(__ldg(row + __ldg(asg + s)), lut, a.m, a.bad) : 0u;
    }
    uint64_t key[WMAX];
    if constexpr (MFIX != 0 && DMAX == 16 && WMAX >= 4)
        make_key_d16<MFIX, WMAX, HCG_SMALL_COMPACT_KEY>(x, a.kind, key);
    else
        make_key<DMAX, WMAX>(x, d, a.m, a.kind, key);

    // Compare the query against the common prefix (bits above hv).
    const int hw = int(cv.hv >> 6), hb = int(cv.hv & 63);
    const uint64_t above = hb == 63 ? 0ull : (~0ull << (hb + 1));
    const uint64_t below = hb == 63 ? ~0ull : ((2ull << hb) - 1);
    int cmp = 0;
#pragma unroll
    for (int w = WMAX - 1; w >= 0; --w) {
        if (cmp == 0 && w >= hw && w < int(cv.w)) {
            const uint64_t qa = key[w] & (w == hw ? above : ~0ull);
            const uint64_t pa = cv.prefix[w];
            cmp = qa < pa ? -1 : (qa > pa ? 1 : 0);
        }
    }
    uint64_t rank;
#ifdef HCG_PROBE_NOSEARCH  // timing probe (tuning builds): key + prefix only, no lower_bound
    if (SMEMIN) cmp = -1;
#endif
    if (cmp < 0) {
        rank = 0;
    } else if (cmp > 0) {
        rank = a.n;
    } else {
        const int ws = int(cv.ws);
        uint64_t qs[WSMAX];
#pragma unroll
        for (int w = 0; w < WSMAX; ++w) qs[w] = w < ws ? (key[w < WMAX ? w : 0] & (w == ws - 1 ? below : ~0ull)) : 0ull;
        const uint64_t* keys = cv.keys;
        const uint32_t wsu = uint32_t(ws);
        uint64_t lo = 0;
        if (COOP) {
            // 32-ary lower bound of qs in arr[lo, hi)
            auto coop = [&](const uint64_t* arr, uint64_t lo_, uint64_t hi) -> uint64_t {
                while (hi - lo_ > 32) {
                    const uint64_t len = hi - lo_;
                    const uint64_t sp = lo_ + ((uint64_t(lane) + 1) * len) / 33;  // strictly increasing, < hi
                    const unsigned b = __ballot_sync(kFull, suffix_cmp<WSMAX>(arr + sp * wsu, qs, ws) < 0);
                    const int cnt = __popc(b);
                    const uint64_t s_lo = __shfl_sync(kFull, sp, cnt > 0 ? cnt - 1 : 0);
                    const uint64_t s_hi = __shfl_sync(kFull, sp, cnt < 32 ? cnt : 31);
                    if (cnt > 0) lo_ = s_lo + 1;
                    if (cnt < 32) hi = s_hi;
                }
                const bool less = lo_ + lane < hi && suffix_cmp<WSMAX>(arr + (lo_ + lane) * wsu, qs, ws) < 0;
                return lo_ + __popc(__ballot_sync(kFull, less));
            };
            uint64_t hi = a.n;
            if (cv.samples) {
                // the sampled keys first (every S-th key; L2-resident under load),
                // then the <= S keys between two samples: one dependent DRAM round
                const uint64_t j = coop(cv.samples, 0, cv.n_samples);
                const uint64_t S = cv.sample_stride;
                lo = j == 0 ? 0 : (j - 1) * S + 1;
                hi = j * S < a.n ? j * S : a.n;
                if (hi < lo) hi = lo;
            }
            lo = coop(keys, lo, hi);
        } else {
            uint64_t len = a.n;
            if (cv.samples) {
                // two levels: lower_bound over the sampled keys (small, L2-resident),
                // then within one stride of the full array (a few DRAM sectors)
                uint64_t j = 0, sl = cv.n_samples;
                while (sl > 0) {
                    const uint64_t half = sl >> 1;
                    if (suffix_cmp<WSMAX>(cv.samples + (j + half) * wsu, qs, ws) < 0) {
                        j += half + 1;
                        sl -= half + 1;
                    } else {
                        sl = half;
                    }
                }
                // keys at positions <= (j-1)*S are < qs; the key at j*S (if any) is >= qs
                const uint64_t S = cv.sample_stride;
                lo = j == 0 ? 0 : (j - 1) * S + 1;
                const uint64_t hi = j * S < a.n ? j * S : a.n;
                len = hi > lo ? hi - lo : 0;
            }
            while (len > 0) {
                const uint64_t half = len >> 1;
                const uint64_t mid = lo + half;
                if (suffix_cmp<WSMAX>(keys + mid * wsu, qs, ws) < 0) {
                    lo = mid + 1;
                    len -= half + 1;
                } else {
                    len = half;
                }
            }
        }
        rank = lo;
    }
    const uint64_t take = a.depth < a.n ? a.depth : a.n;
    const uint64_t below_n = take / 2;
    uint64_t begin = rank >= below_n ? rank - below_n : 0;
    if (begin + take > a.n) begin = a.n - take;
    HCG_DASSERT(begin + take <= a.n && rank <= a.n);
    *rank_out = rank;
    return begin;
}

template <int DMAX, int WSMAX, bool COOP, int MINB, class T>
__global__ void __launch_bounds__(128, MINB) k_locate(LocateArgs a) {
    __shared__ uint32_t lut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = a.lut[i];
    __syncthreads();
    const uint64_t t = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> (COOP ? 5 : 0);
    const int lane = threadIdx.x & 31;
    if (t >= uint64_t(a.nq) * a.C) return;
    const uint32_t q = uint32_t(t / a.C), c = uint32_t(t % a.C);
    uint64_t rank;
    const uint64_t begin = locate_one<DMAX, WSMAX, COOP, T>(a, lut, q, c, lane, &rank);
    if (!COOP || lane == 0) {
        a.out_begin[t] = uint32_t(begin);
        if (a.out_rank) a.out_rank[t] = rank;
    }
}

#ifndef HCG_LOCATE_MINB
#define HCG_LOCATE_MINB 8
#endif
template <int DMAX, int WSMAX, class T>
static void locate_launch_t(const LocateArgs& a, cudaStream_t st) {
    const uint64_t total = uint64_t(a.nq) * a.C;
    if (total <= 1024)  // small batches: a warp per (query, curve), ~5 dependent loads
        k_locate<DMAX, WSMAX, true, 1, T><<<unsigned((total * 32 + 127) / 128), 128, 0, st>>>(a);
    else  // 8 CTAs/SM: measured 3 % faster than the 88-register default
        k_locate<DMAX, WSMAX, false, (DMAX <= 16 ? HCG_LOCATE_MINB : 1), T><<<unsigned((total + 127) / 128), 128, 0, st>>>(a);
}

template <int DMAX, int WSMAX>
static void locate_launch(const LocateArgs& a, cudaStream_t st) {
    if (a.dtype == HCG_F32)
        locate_launch_t<DMAX, WSMAX, float>(a, st);
    else
        locate_launch_t<DMAX, WSMAX, uint8_t>(a, st);
}

template <int DMAX>
static hcg_status locate_ws(const LocateArgs& a, int wsmax, cudaStream_t st) {
    constexpr int WMAX = DMAX / 2 > kMaxKeyWords ? kMaxKeyWords : DMAX / 2;
    switch (wsmax) {
        case 1: locate_launch<DMAX, 1>(a, st); break;
        case 2: locate_launch<DMAX, 2>(a, st); break;
        case 4: locate_launch<DMAX, 4>(a, st); break;
        case 8:
            if constexpr (WMAX >= 8) { locate_launch<DMAX, 8>(a, st); break; }
            return set_error(HCG_EINVAL, "suffix wider than key");
        case 16:
            if constexpr (WMAX >= 16) { locate_launch<DMAX, 16>(a, st); break; }
            return set_error(HCG_EINVAL, "suffix wider than key");
        default: return set_error(HCG_EINVAL, "bad suffix bucket");
    }
    return check_launch("k_locate");
}

hcg_status launch_locate(const LocateArgs& a, int dmax, int wsmax, cudaStream_t st) {
    if (uint64_t(a.nq) * a.C == 0) return HCG_OK;
    count_launches(1);
    switch (dmax) {
        case 8: return locate_ws<8>(a, wsmax, st);
        case 16: return locate_ws<16>(a, wsmax, st);
        case 32: return locate_ws<32>(a, wsmax, st);
        case 64: return locate_ws<64>(a, wsmax, st);
        case 128: return locate_ws<128>(a, wsmax, st);
        default: return set_error(HCG_EINVAL, "unsupported curve dimension bucket");
    }
}

// ----------------------------------------------------------------- K3b ----
constexpr int kRefineThreads = 256;
constexpr int kRefineMaxSmem = 200 * 1024;

template <int R>
__device__ __forceinline__ void write_result(const RefineArgs& a, uint32_t q, const WarpTopK<R>& fin, int lane,
                                             uint32_t U) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t e = uint32_t(lane) * R + r;
        if (e < a.k) {
            const uint64_t x = fin.a[r];
            const uint64_t o = uint64_t(q) * a.k + e;
            const bool none = x == kNone;
            const uint64_t gid = a.id_base + (x & 0xFFFFFFFFull) * a.id_stride;
            if (a.mode == kOutIds) {
                a.out_ids[o] = none ? ~0ull : gid;
                a.out_sqdist[o] = none ? 0xFFFFFFFFu : uint32_t(x >> 32);
            } else {
                a.out_packed[o] = none ? kNone : ((x & 0xFFFFFFFF00000000ull) | gid);
            }
        }
    }
    if (lane == 0 && a.mode == kOutIds) a.out_len[q] = U < a.k ? U : a.k;
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* src) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }


// Exclusive scan of one value per thread over an NT-thread block (ends with a barrier).
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan_u(uint32_t v, uint32_t* wsum) {
    constexpr int kW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < kW; ++w) before += w < warp ? wsum[w] : 0u;
    __syncthreads();
    return before + inc - v;
}

// Exclusive scan of one value per thread over a 256-thread block (ends with a barrier).
__device__ __forceinline__ uint32_t block_excl_scan256_u(uint32_t v, uint32_t* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) before += w < warp ? wsum[w] : 0u;
    __syncthreads();
    return before + inc - v;
}

// ------------------------------------------------------------- K3b ----
// Candidate union (multicurves.hpp:87-89): one CTA per query (persistent).
// The C windows' ids are read (coalesced) into shared memory, then
// deduplicated without atomics: in round r every pending position i stores
// the tag (r, i) into slot h_r(id[i]) of a u16 table; after a barrier it
// reads the slot back -- its own tag: first copy of the id, appended to the
// query's unique list in HBM; the tag of another copy of the same id:
// dropped; a different id: collision, retried with the next hash.  All copies
// of an id hit the same slot in every round, so they resolve together; the
// rare ids still pending after kUnionRounds keep their lowest position.
constexpr int kUnionRounds = 6;
constexpr uint32_t kUnionMaxT = 32 * 256;  // one u32 pending mask per thread

// One CTA deduplicating queries q0, q0 + qstep, ...
__device__ __forceinline__ void union_cta(const RefineArgs& a, uint32_t* __restrict__ lists,
                                          uint32_t* __restrict__ counts, uint32_t lstride, uint32_t tb,
                                          uint32_t q0, uint32_t qstep) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t T = a.C * a.take;
    const uint32_t** sptr = reinterpret_cast<const uint32_t**>(smem);
    uint32_t* sbeg = reinterpret_cast<uint32_t*>(sptr + a.C);  // [2][C]
    uint32_t* wsum = sbeg + 2 * a.C;                            // [8] scan scratch
    uint32_t* ids2 = wsum + 8;                                  // [2][T], cp.async double buffer
    uint32_t* tab = ids2 + 2 * T;                               // [1 << tb] tags
    const int tid = threadIdx.x;
    const uint32_t take = a.take;
    const uint32_t jn = (T + kRefineThreads - 1) / kRefineThreads;  // <= 32
    const uint32_t shift = 32 - tb;

    auto stage = [&](int buf) {
        const uint32_t* beg = sbeg + buf * a.C;
        uint32_t* dst = ids2 + buf * T;
        for (uint32_t c = 0; c < a.C; ++c) {
            const uint32_t* src = sptr[c] + beg[c];
            for (uint32_t p = tid; p < take; p += kRefineThreads) cp_async4(dst + c * take + p, src + p);
        }
    };

    for (uint32_t c = tid; c < a.C; c += kRefineThreads) sptr[c] = a.slots[c];
    uint32_t q = q0;
    if (q < a.nq)
        for (uint32_t c = tid; c < a.C; c += kRefineThreads) sbeg[c] = a.begins[uint64_t(q) * a.C + c];
    __syncthreads();
    if (q < a.nq) stage(0);
    cp_async_commit();

    for (uint32_t it = 0; q < a.nq; q += qstep, ++it) {
        const int cur = it & 1;
        const uint32_t qn = q + qstep;
        if (qn < a.nq)
            for (uint32_t c = tid; c < a.C; c += kRefineThreads)
                sbeg[(cur ^ 1) * a.C + c] = a.begins[uint64_t(qn) * a.C + c];
        cp_async_wait_all();
        __syncthreads();  // ids of q landed; next begins visible
        if (qn < a.nq) stage(cur ^ 1);  // prefetch the next query while deduping this one
        cp_async_commit();
        const uint32_t* idbuf = ids2 + cur * T;

        // positions of this thread: i = tid + 256 j, j < jn (bit j of the masks)
        uint32_t pending = 0;
        for (uint32_t j = 0; j < jn; ++j)
            if (tid + j * kRefineThreads < T) pending |= 1u << j;
        uint32_t keep = 0;
#pragma unroll 1
        for (int r = 0; r < kUnionRounds; ++r) {
            const uint32_t mul = 0x9E3779B1u + 0x7F4A7C16u * uint32_t(r);  // odd multipliers
            const uint32_t tagr = uint32_t(r + 1) << 16;
            for (uint32_t pm = pending; pm; pm &= pm - 1) {
                const uint32_t i = tid + uint32_t(__ffs(pm) - 1) * kRefineThreads;
                tab[(idbuf[i] * (mul | 1u)) >> shift] = tagr | i;
            }
            __syncthreads();
            for (uint32_t pm = pending; pm; pm &= pm - 1) {
                const uint32_t j = __ffs(pm) - 1;
                const uint32_t i = tid + j * kRefineThreads;
                const uint32_t s = idbuf[i];
                const uint32_t o = tab[(s * (mul | 1u)) >> shift];
                if (o == (tagr | i)) {
                    keep |= 1u << j;
                    pending &= ~(1u << j);
                } else if (idbuf[o & 0xFFFFu] == s) {
                    pending &= ~(1u << j);
                }
            }
            if (!__syncthreads_or(pending != 0)) break;
        }
        // Leftovers (rare): all copies of such an id are still pending, so the
        // copy at the lowest position is the first one.
        for (uint32_t pm = pending; pm; pm &= pm - 1) {
            const uint32_t j = __ffs(pm) - 1;
            const uint32_t i = tid + j * kRefineThreads;
            const uint32_t s = idbuf[i];
            bool first = true;
            for (uint32_t i2 = 0; i2 < i; ++i2)
                if (idbuf[i2] == s) {
                    first = false;
                    break;
                }
            if (first) keep |= 1u << j;
        }
        // Compact: block exclusive scan of the kept counts.
        const uint32_t mine = __popc(keep);
        const uint32_t off = block_excl_scan256_u(mine, wsum);
        uint32_t* out = lists + uint64_t(q) * lstride + off;
        uint32_t w = 0;
        for (uint32_t pm = keep; pm; pm &= pm - 1) out[w++] = idbuf[tid + uint32_t(__ffs(pm) - 1) * kRefineThreads];
        if (tid == kRefineThreads - 1) counts[q] = off + mine;
    }
    cp_async_wait_all();
}

__global__ void __launch_bounds__(kRefineThreads) k_union(RefineArgs a, uint32_t* __restrict__ lists,
                                                          uint32_t* __restrict__ counts, uint32_t lstride,
                                                          uint32_t tb) {
    union_cta(a, lists, counts, lstride, tb, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------- K3c ----
// Gather + exact L2 + top-k: one WARP per query (persistent), no shared
// memory, no barriers.  Each pass covers 32 list entries: the 4 groups of 8
// lanes own 8 rows each (one 16-B chunk per lane and row, 8 LDG.128 in flight
// per lane); the next pass's slots are prefetched while the rows load.  The
// reduce-scatter leaves row (8*grp + l8)'s squared distance in lane l8 of
// group grp, which offers (sqdist << 32 | slot) to the warp top-k.
// Score list entries [start, start+32), [start+step, ...) of one query into a
// warp top-k: the 4 groups of 8 lanes own 8 rows each per pass (one 16-B chunk
// per lane and row, 8 LDG.128 in flight per lane) and the next pass's slots
// are prefetched while the rows load.  The reduce-scatter leaves row
// (8*grp + l8)'s squared distance in lane l8 of group grp, which offers
// (sqdist << 32 | slot).  Lists are read with ld.global.cg: they were written
// by the preceding union launch.
// QUEUED (one warp per list): offers go through the warp's queue
// (WarpTopK::offer_queued; wsm: 32 R + 32 slots) -- the list holds no
// repeats, so the queue takes 32 and a pass waits for no id.
template <int R, int CR, bool SMEMLIST = false, bool QUEUED = false>
__device__ __forceinline__ void gather_list(const RefineArgs& a, const uint32_t* list, uint32_t n, uint32_t start,
                                            uint32_t step, const uint4 (&qv)[CR], int lane, WarpTopK<R>& tk,
                                            uint64_t* wsm = nullptr) {
    uint32_t qn = 0;
    const int l8 = lane & 7, grp = lane >> 3;
    const uint32_t chunks = a.pitch >> 4;
    auto ld = [&](uint32_t e) -> uint32_t { return SMEMLIST ? list[e] : __ldcg(list + e); };
    uint32_t nx[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t e = start + grp * 8 + r;
        nx[r] = e < n ? ld(e) : kEmpty;
    }
    for (uint32_t base = start; base < n; base += step) {
#pragma unroll
        for (int r = 0; r < 8; ++r) HCG_DASSERT(nx[r] == kEmpty || nx[r] < a.n_rows);
        uint4 v[8][CR];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int t = 0; t < CR; ++t) {
                const uint32_t ch = l8 + 8 * t;
                v[r][t] = (nx[r] != kEmpty && ch < chunks) ? ldg_stream(a.rows + uint64_t(nx[r]) * a.pitch + ch * 16)
                                                           : make_uint4(0, 0, 0, 0);
            }
        }
        // this lane's row after the reduce-scatter is row l8 of its group
        uint32_t me = nx[0];
#pragma unroll
        for (int r = 1; r < 8; ++r)
            if (r == l8) me = nx[r];
        // latency path (shared-memory list, few passes): the id slot of every
        // row is fetched with the rows instead of after the distance
        uint32_t idpre = me;
        if (SMEMLIST && a.idtab && me != kEmpty) idpre = __ldg(a.idtab + me);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t e = base + step + grp * 8 + r;
            nx[r] = e < n ? ld(e) : kEmpty;
        }
        uint32_t acc[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            acc[r] = 0;
#pragma unroll
            for (int t = 0; t < CR; ++t) acc[r] = sad2_16(v[r][t], qv[t], acc[r]);
        }
        const bool b2 = l8 & 4, b1 = l8 & 2, b0 = l8 & 1;
        uint32_t s4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t send = b2 ? acc[i] : acc[i + 4];
            const uint32_t keep = b2 ? acc[i + 4] : acc[i];
            s4[i] = keep + __shfl_xor_sync(kFull, send, 4);
        }
        uint32_t s2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint32_t send = b1 ? s4[i] : s4[i + 2];
            const uint32_t keep = b1 ? s4[i + 2] : s4[i];
            s2[i] = keep + __shfl_xor_sync(kFull, send, 2);
        }
        const uint32_t S = (b0 ? s2[1] : s2[0]) + __shfl_xor_sync(kFull, b0 ? s2[0] : s2[1], 1);
        if constexpr (QUEUED) {
            tk.offer_queued(me != kEmpty ? ((uint64_t(S) << 32) | me) : kNone, lane, wsm, wsm + 32 * R, qn, 32u,
                            a.idtab);
            continue;
        }
        uint32_t sl = me;
        if (SMEMLIST) {
            sl = idpre;
        } else if (a.idtab) {  // physical row -> id slot, read only for rows that can enter the top-k
            const bool pre = me != kEmpty && S <= uint32_t(tk.thr >> 32);
            if (__any_sync(kFull, pre) && pre) sl = __ldg(a.idtab + me);
        }
        tk.template offer<SMEMLIST>(me != kEmpty ? ((uint64_t(S) << 32) | sl) : kNone, lane);
    }
    if constexpr (QUEUED) tk.flush_queue(lane, wsm, wsm + 32 * R, qn, a.idtab);
}

// K3c without the union (rows in curve-0 order): the warp walks the query's C
// windows directly -- entry e is position e % take of curve e / take -- and
// offers every row; a row reached through two curves gives the same
// (distance, id) key twice and the queued merge keeps one
// (WarpTopK::offer_queued: a queue of min(32, 32 R - k) offers).  Costs the
// duplicate rows (~16 % of the windows, partly L2 hits) instead of the union
// kernel and the lists' round trip.
// SMALLC (C <= 32): lane c holds curve c's window start pointer (slots[c] +
// begin), fetched once per query and broadcast with a shuffle, so an entry
// costs one dependent load (the slot) instead of three (pointer, begin, slot).
template <int CR, bool SMALLC, class TK>
__device__ __forceinline__ void gather_windows(const RefineArgs& a, const uint32_t* begins_q, const uint4 (&qv)[CR],
                                               int lane, TK& tk, uint64_t* wsm) {
    const int l8 = lane & 7, grp = lane >> 3;
    const uint32_t chunks = a.pitch >> 4;
    const uint32_t take = a.take, n = a.C * take, C = a.C;
    // (curve, position) of this lane-group's 8 entries, advanced by 32 per pass
    uint32_t cc[8], pp[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t e = uint32_t(grp * 8 + r);
        cc[r] = e / take;
        pp[r] = e - cc[r] * take;
    }
    unsigned long long wstart = 0;
    if (SMALLC && uint32_t(lane) < C)
        wstart = reinterpret_cast<unsigned long long>(a.slots[lane] + __ldg(begins_q + lane));
    auto entry = [&](int r) -> uint32_t {
        if constexpr (SMALLC) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(__shfl_sync(kFull, wstart, int(cc[r] & 31)));
            return cc[r] < C ? __ldg(w + pp[r]) : kEmpty;
        } else {
            return cc[r] < C ? __ldg(a.slots[cc[r]] + __ldg(begins_q + cc[r]) + pp[r]) : kEmpty;
        }
    };
    uint32_t nx[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) nx[r] = entry(r);
    // the offer queue (WarpTopK::offer_queued) behind the dedup scratch
    uint32_t qn = 0;
    const uint32_t qcap = min(32u, 32u * TK::kR - a.k);
    for (uint32_t base = 0; base < n; base += 32) {
        uint4 v[8][CR];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int t = 0; t < CR; ++t) {
                const uint32_t ch = l8 + 8 * t;
                v[r][t] = (nx[r] != kEmpty && ch < chunks) ? ldg_stream(a.rows + uint64_t(nx[r]) * a.pitch + ch * 16)
                                                           : make_uint4(0, 0, 0, 0);
            }
        }
        uint32_t me = nx[0];
#pragma unroll
        for (int r = 1; r < 8; ++r)
            if (r == l8) me = nx[r];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            pp[r] += 32;
            while (pp[r] >= take && cc[r] < a.C) {
                pp[r] -= take;
                ++cc[r];
            }
            nx[r] = entry(r);
        }
        uint32_t acc[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            acc[r] = 0;
#pragma unroll
            for (int t = 0; t < CR; ++t) acc[r] = sad2_16(v[r][t], qv[t], acc[r]);
        }
        const bool b2 = l8 & 4, b1 = l8 & 2, b0 = l8 & 1;
        uint32_t s4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t send = b2 ? acc[i] : acc[i + 4];
            const uint32_t keep = b2 ? acc[i + 4] : acc[i];
            s4[i] = keep + __shfl_xor_sync(kFull, send, 4);
        }
        uint32_t s2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint32_t send = b1 ? s4[i] : s4[i + 2];
            const uint32_t keep = b1 ? s4[i + 2] : s4[i];
            s2[i] = keep + __shfl_xor_sync(kFull, send, 2);
        }
        const uint32_t S = (b0 ? s2[1] : s2[0]) + __shfl_xor_sync(kFull, b0 ? s2[0] : s2[1], 1);
        // the queue translates rows to ids when it flushes
        tk.offer_queued(me != kEmpty ? ((uint64_t(S) << 32) | me) : kNone, lane, wsm, wsm + 32 * TK::kR, qn, qcap,
                        a.idtab);
    }
    tk.flush_queue(lane, wsm, wsm + 32 * TK::kR, qn, a.idtab);
}

template <int CR>
__device__ __forceinline__ void load_query(const RefineArgs& a, uint32_t q, int lane, uint4 (&qv)[CR]) {
    const uint32_t chunks = a.pitch >> 4;
    const uint8_t* qrow = a.queries + uint64_t(q) * a.pitch;
#pragma unroll
    for (int t = 0; t < CR; ++t) {
        const uint32_t ch = (lane & 7) + 8 * t;
        qv[t] = ch < chunks ? *reinterpret_cast<const uint4*>(qrow + ch * 16) : make_uint4(0, 0, 0, 0);
    }
}

// K3c for large batches: one WARP per query (persistent grid-stride), no
// barriers.  Lists of 32 and 128 / 256 take their offers through a per-warp
// queue in shared memory (WarpTopK::offer_queued); the 64-entry list keeps
// per-pass offers, 3-4 % faster there (profiles/r02_gather_queue_ab.jsonl:
// k = 100 at D = 350 6.66 vs 7.50 ms, k = 32 2.55 vs 2.68 ms at D = 128, k =
// 64 7.04 vs 6.76 ms at D = 350).
#ifndef HCG_GATHER_QUEUE
#define HCG_GATHER_QUEUE 1
#endif
template <int R>
constexpr bool kGatherQueued = HCG_GATHER_QUEUE && R != 2;

template <int R, int CR, int MINB>
__global__ void __launch_bounds__(kRefineThreads, MINB) k_gather(RefineArgs a, const uint32_t* __restrict__ lists,
                                                                 const uint32_t* __restrict__ counts,
                                                                 uint32_t lstride) {
    __shared__ uint64_t dsm[kGatherQueued<R> ? kRefineThreads / 32 : 1][kGatherQueued<R> ? 32 * R + 32 : 1];
    const int lane = threadIdx.x & 31;
    const uint32_t qstep = gridDim.x * (kRefineThreads / 32);
    for (uint32_t q = (blockIdx.x * kRefineThreads + threadIdx.x) >> 5; q < a.nq; q += qstep) {
        const uint32_t n = __ldcg(counts + q);
        const uint32_t qq = a.qorder ? __ldg(a.qorder + q) : q;  // list q holds query qq
        uint4 qv[CR];
        load_query<CR>(a, qq, lane, qv);
        WarpTopK<R> tk;
        tk.init(int(a.k));
        gather_list<R, CR, false, kGatherQueued<R>>(a, lists + uint64_t(q) * lstride, n, 0, 32, qv, lane, tk,
                                                    dsm[kGatherQueued<R> ? threadIdx.x >> 5 : 0]);
        write_result<R>(a, qq, tk, lane, n);
    }
}

// K3c without the union: one warp per query over the raw windows.
template <int R, int CR, int MINB, bool SMALLC, int NT = kRefineThreads>
__global__ void __launch_bounds__(NT, MINB) k_gather_nu(RefineArgs a) {
    // per-warp scratch of the batched dedup + the offer queue
    __shared__ uint64_t dsm[NT / 32][32 * R + 32];
    const int lane = threadIdx.x & 31;
    uint64_t* wsm = dsm[threadIdx.x >> 5];
    const uint32_t qstep = gridDim.x * (NT / 32);
    for (uint32_t q = (blockIdx.x * NT + threadIdx.x) >> 5; q < a.nq; q += qstep) {
        const uint32_t qq = a.qorder ? __ldg(a.qorder + q) : q;
        uint4 qv[CR];
        load_query<CR>(a, qq, lane, qv);
        WarpTopK<R> tk;
        tk.init(int(a.k));
        gather_windows<CR, SMALLC>(a, a.begins + uint64_t(qq) * a.C, qv, lane, tk, wsm);
        uint32_t valid = 0;
#pragma unroll
        for (int r = 0; r < R; ++r)
            valid += (uint32_t(lane) * R + r < a.k && tk.a[r] != kNone) ? 1u : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) valid += __shfl_xor_sync(kFull, valid, o);
        write_result<R>(a, qq, tk, lane, valid);
    }
}

// K3c for small batches (latency): one CTA per query, the 8 warps split the
// list and warp 0 merges their top-k lists through shared memory.
template <int R, int CR, int NW>
__global__ void __launch_bounds__(NW * 32) k_gather_cta(RefineArgs a, const uint32_t* __restrict__ lists,
                                                        const uint32_t* __restrict__ counts, uint32_t lstride) {
    constexpr int KCAP = 32 * R;
    constexpr int kWarps = NW;
    __shared__ uint64_t mbuf[kWarps * KCAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        const uint32_t n = __ldcg(counts + q);
        uint4 qv[CR];
        load_query<CR>(a, a.qorder ? __ldg(a.qorder + q) : q, lane, qv);
        WarpTopK<R> tk;
        tk.init(int(a.k));
        gather_list<R, CR>(a, lists + uint64_t(q) * lstride, n, warp * 32, NW * 32, qv, lane, tk);
#pragma unroll
        for (int r = 0; r < R; ++r) mbuf[warp * KCAP + lane * R + r] = tk.a[r];
        __syncthreads();
        if (warp == 0) {
            WarpTopK<R> fin;
            fin.init(int(a.k));
            const uint32_t kr = (a.k + 31) & ~31u;
            for (int w = 0; w < kWarps; ++w)
                for (uint32_t i = 0; i < kr; i += 32) fin.offer(mbuf[w * KCAP + i + lane], lane);
            write_result<R>(a, a.qorder ? __ldg(a.qorder + q) : q, fin, lane, n);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------ small batches ----
// The whole search of one query in one CTA -- the latency path for small
// batches (u8 rows of <= 128 B, C x take <= kSmallMaxWalk): one launch
// instead of locate + union + gather, no HBM scratch.
//   1. warp w locates curves w, w + NW, ...: key + 32-ary cooperative
//      lower_bound + window (rank_of / window, multicurves.hpp:57-63);
//   2. all threads: candidate union (multicurves.hpp:87-89) -- the windows'
//      slots into a shared-memory CAS hash set, first copies appended
//      (warp-aggregated) to a shared unique list;
//   3. each warp gathers a slice of the list into its warp top-k (exact u32
//      distances, (distance, id) order), warp 0 merges the NW lists.
constexpr int kSmallThreads = 1024;
constexpr uint32_t kSmallMaxWalk = 8192;
constexpr uint32_t kSmallBatch = 512;
constexpr uint32_t kSmallMaxCurves = 32;
constexpr uint32_t kSmallMaxAssign = 512;

__host__ __device__ __forceinline__ uint32_t small_table_bits(uint32_t T) {
    uint32_t tb = 5;
    while ((1u << tb) * 7u < T * 10u) ++tb;
    return tb;
}

// mbuf (half the warps' lists) | CurveDev[C] | wptr[C] | assignment (u16) | query row | lut | table | list
template <int R>
__host__ __device__ __forceinline__ size_t small_smem_bytes(uint32_t C, uint32_t T, uint32_t n_assign, uint32_t pitch) {
    return size_t(kSmallThreads / 64) * 32 * R * 8 + size_t(C) * sizeof(CurveDev) + size_t(C) * 8 +
           ((size_t(n_assign) * 2 + 15) & ~size_t(15)) + ((size_t(pitch) + 15) & ~size_t(15)) + 256 * 4 +
           (size_t(4) << small_table_bits(T)) + size_t(T) * 4;
}

template <int M, int WSMAX, int R>
__global__ void __launch_bounds__(kSmallThreads) k_search_small(LocateArgs la, RefineArgs a, uint32_t n_assign) {
    constexpr int NW = kSmallThreads / 32;
    constexpr int KCAP = 32 * R;
    constexpr int JN = kSmallMaxWalk / kSmallThreads;  // window entries per thread
    extern __shared__ __align__(16) unsigned char ssm[];
    uint64_t* mbuf = reinterpret_cast<uint64_t*>(ssm);                       // NW/2 x KCAP
    CurveDev* scv = reinterpret_cast<CurveDev*>(mbuf + (NW / 2) * KCAP);      // C
    const uint32_t** wptr = reinterpret_cast<const uint32_t**>(scv + a.C);   // C: slots[c] + begin
    uint16_t* sasg = reinterpret_cast<uint16_t*>(wptr + a.C);                 // n_assign
    uint8_t* sq = reinterpret_cast<uint8_t*>(sasg) + ((size_t(n_assign) * 2 + 15) & ~size_t(15));  // pitch
    uint32_t* lut = reinterpret_cast<uint32_t*>(sq + ((a.pitch + 15) & ~15u));  // 256
    const uint32_t T = a.C * a.take, tb = small_table_bits(T), tmask = (1u << tb) - 1;
    uint32_t* table = lut + 256;                                            // 1 << tb
    uint32_t* list = table + (1u << tb);                                    // T
    __shared__ uint32_t count;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // phase timestamps of the first query (a.prof: tuning builds only)
    auto stamp = [&](int i) {
        if (a.prof && blockIdx.x == 0 && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.prof[i] = t;
        }
    };
    // what the locate reads per curve, staged once: one round trip instead of a chain
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(la.curves);
        uint32_t* dst = reinterpret_cast<uint32_t*>(scv);
        for (uint32_t i = tid; i < a.C * (sizeof(CurveDev) / 4); i += kSmallThreads) dst[i] = __ldg(src + i);
        for (uint32_t i = tid; i < n_assign; i += kSmallThreads) sasg[i] = __ldg(la.assign + i);
        for (int i = tid; i < 256; i += kSmallThreads) lut[i] = __ldg(la.lut + i);
    }
    LocateArgs ls = la;
    ls.curves = scv;
    ls.assign = sasg;
    ls.queries = sq;
    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        stamp(0);
        for (uint32_t i = tid; i < (a.pitch >> 2); i += kSmallThreads)
            reinterpret_cast<uint32_t*>(sq)[i] = __ldg(reinterpret_cast<const uint32_t*>(la.queries + uint64_t(q) * la.pitch) + i);
        for (uint32_t i = tid; i <= tmask; i += kSmallThreads) table[i] = kEmpty;
        if (tid == 0) count = 0;
        __syncthreads();
        // 1. locate: a warp per curve
        for (uint32_t c = warp; c < a.C; c += NW) {
            uint64_t rank;
            const uint64_t b = locate_one<16, WSMAX, true, uint8_t, M, true>(ls, lut, 0, c, lane, &rank);
            HCG_DASSERT(b + a.take <= a.n_rows);
            if (lane == 0) wptr[c] = a.slots[c] + b;
        }
        __syncthreads();
        stamp(1);
        // 2. union: every thread loads its window entries first (independent
        // loads in flight together), then inserts them into the hash set
        uint32_t sl[JN];
#pragma unroll
        for (int j = 0; j < JN; ++j) {
            const uint32_t i = uint32_t(tid) + uint32_t(j) * kSmallThreads;
            sl[j] = kEmpty;
            if (i < T) {
                const uint32_t c = i / a.take;
                sl[j] = __ldg(wptr[c] + (i - c * a.take));
            }
        }
#pragma unroll
        for (int j = 0; j < JN; ++j) {
            if (uint32_t(j) * kSmallThreads >= T) break;  // block-uniform
            const uint32_t s = sl[j];
            bool fresh = false;
            if (s != kEmpty) {
                uint32_t h = hash_slot(s) >> (32 - tb);
                while (true) {
                    const uint32_t prev = atomicCAS(&table[h], kEmpty, s);
                    if (prev == kEmpty) {
                        fresh = true;
                        break;
                    }
                    if (prev == s) break;
                    h = (h + 1) & tmask;
                }
            }
            const unsigned bal = __ballot_sync(kFull, fresh);
            if (bal) {
                const int leader = __ffs(bal) - 1;
                uint32_t base = 0;
                if (lane == leader) base = atomicAdd(&count, uint32_t(__popc(bal)));
                base = __shfl_sync(kFull, base, leader);
                HCG_DASSERT(!fresh || (base + __popc(bal & lanemask_lt_s()) < T && s < a.n_rows));
                if (fresh) list[base + __popc(bal & lanemask_lt_s())] = s;
            }
        }
        __syncthreads();
        stamp(2);
        // 3. gather + exact L2 + warp top-k over slices of the list
        const uint32_t n = count;
        uint4 qv[1];
        {
            const uint32_t ch = uint32_t(lane & 7);
            qv[0] = ch < (a.pitch >> 4) ? reinterpret_cast<const uint4*>(sq)[ch] : make_uint4(0, 0, 0, 0);
        }
        WarpTopK<R> tk;
        tk.init(int(a.k));
        gather_list<R, 1, true>(a, list, n, uint32_t(warp) * 32, NW * 32, qv, lane, tk);
        stamp(3);
        // 4. tree merge of the warps' sorted lists: the upper half hands its
        // lists to the lower half (shared memory), which merges them slice by
        // slice (merge_sorted32 keeps the 32R smallest); log2(NW) rounds
#pragma unroll 1
        for (int half = NW / 2; half >= 1; half >>= 1) {
            __syncthreads();
            if (warp >= half && warp < 2 * half) {
#pragma unroll
                for (int r = 0; r < R; ++r) mbuf[(warp - half) * KCAP + lane * R + r] = tk.a[r];
            }
            __syncthreads();
            if (warp < half) {
#pragma unroll
                for (int r = 0; r < R; ++r)  // slice r of the partner's list, ascending over the lanes
                    merge_sorted32<R>(tk.a, mbuf[warp * KCAP + lane * R + r], lane);
            }
        }
        if (warp == 0) write_result<R>(a, q, tk, lane, n);
        stamp(4);
        __syncthreads();
    }
}

template <int M, int WSMAX, int R>
hcg_status small_launch(const LocateArgs& la, const RefineArgs& a, uint32_t n_assign, int device, cudaStream_t st) {
    auto kern = k_search_small<M, WSMAX, R>;
    static bool cfg[64] = {};
    if (!cfg[device & 63]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(small_smem_bytes<R>(kSmallMaxCurves, kSmallMaxWalk, kSmallMaxAssign, 128))) !=
            cudaSuccess)
            return set_error(HCG_ECUDA, "small-batch search: cannot opt in to dynamic shared memory");
        cfg[device & 63] = true;
    }
    count_launches(1);
    kern<<<a.nq, kSmallThreads, small_smem_bytes<R>(a.C, a.C * a.take, n_assign, a.pitch), st>>>(la, a, n_assign);
    return check_launch("k_search_small");
}

template <int M, int WSMAX>
hcg_status small_dispatch_r(const LocateArgs& la, const RefineArgs& a, uint32_t n_assign, int device,
                            cudaStream_t st) {
    switch (a.k <= 32 ? 1 : a.k <= 64 ? 2 : a.k <= 128 ? 4 : 8) {
        case 1: return small_launch<M, WSMAX, 1>(la, a, n_assign, device, st);
        case 2: return small_launch<M, WSMAX, 2>(la, a, n_assign, device, st);
        case 4: return small_launch<M, WSMAX, 4>(la, a, n_assign, device, st);
        default: return small_launch<M, WSMAX, 8>(la, a, n_assign, device, st);
    }
}

// The default scheme's shapes (16 dims per curve, m = 8 raw / 16 lifted).
// One wave of CTAs at most: 2 per SM (1024 threads each) while the shared
// memory allows (k <= 64), else 1.  Measured at 10M, D = 350: batch 256 69 µs
// fused vs 91 µs on the three-kernel path, batch 512 (two waves) 129 vs 96 µs.
bool small_eligible(const LocateArgs& la, const RefineArgs& a, bool dims16, int wsmax, int device) {
    static const bool off = knob("HCG_NO_SMALL") != nullptr;  // A/B: locate + union + gather for every batch
    const uint32_t wave = uint32_t(dev_info(device).sms) * (a.k <= 64 ? 2u : 1u);
    return !off && dims16 && (la.m == 8 || la.m == 16) && a.dtype == HCG_U8 && la.dtype == HCG_U8 && a.nq >= 1 &&
           a.nq <= std::min(kSmallBatch, wave) && a.pitch <= 128 && uint64_t(a.C) * a.take <= kSmallMaxWalk &&
           wsmax <= 4 && a.C <= kSmallMaxCurves && a.C * 16 <= kSmallMaxAssign && a.mode != kOutCandidates;
}

hcg_status launch_search_small(const LocateArgs& la, const RefineArgs& a, int wsmax, int device, cudaStream_t st) {
    const uint32_t n_assign = a.C * 16;  // every curve has 16 dims here
    if (la.m == 8) {
        switch (wsmax) {
            case 1: return small_dispatch_r<8, 1>(la, a, n_assign, device, st);
            case 2: return small_dispatch_r<8, 2>(la, a, n_assign, device, st);
            default: return small_dispatch_r<8, 4>(la, a, n_assign, device, st);
        }
    }
    switch (wsmax) {
        case 1: return small_dispatch_r<16, 1>(la, a, n_assign, device, st);
        case 2: return small_dispatch_r<16, 2>(la, a, n_assign, device, st);
        default: return small_dispatch_r<16, 4>(la, a, n_assign, device, st);
    }
}

// ------------------------------------------------------- K3c, f32 rows ----
// Float descriptors (the reference's native component type), scored exactly
// as squared_distance (vecio.cpp:87-95) does: acc = 0; for i in index order
// acc += (double(a_i) - double(b_i))^2, each subtract, multiply and add
// rounded on its own (no FMA contraction) -- the same double, bit for bit,
// so ids and (distance, id) tie order match the reference by construction.
// A sequential sum needs one lane per row: each pass a warp takes 32 rows,
// lane r streams row r through registers (16 floats at a time, loads issued
// ahead of their terms) against the query held as doubles in shared memory,
// and offers (double bits, slot) to the pair top-k.  Padding components are
// zero on both sides and add exact zeros.  The sums are FP64-latency chains:
// occupancy (no tile in shared memory) is what hides them -- a 32-row
// shared-memory tile per warp ran 39 ms per 100K queries at 12 warps / SM,
// double-buffered (6 warps / SM) 70 ms.
constexpr uint32_t kF32Rows = 32;  // rows per warp pass (one per lane)

constexpr int kF32Threads = 256;  // k_gather_f32
constexpr int kF32CtaWarps = 8;   // k_gather_cta_f32 / k_brute_f32
// Shared bytes per warp: the query row as doubles (converted once per query).
__host__ __device__ __forceinline__ uint32_t f32_warp_smem(uint32_t pitch) { return 2 * pitch; }

__device__ __forceinline__ double sq_term(float a, double b) {
    const double d = __dsub_rn(double(a), b);
    return __dmul_rn(d, d);
}

template <bool DIRECT>
__device__ __forceinline__ uint32_t f32_entry(const uint32_t* list, uint32_t e, uint32_t n) {
    if (DIRECT) return e < n ? e : kEmpty;
    return e < n ? __ldcg(list + e) : kEmpty;
}

// Query row q -> the warp's query buffer (qs: pitch / 4 doubles, converted
// once per query instead of once per candidate row).
__device__ __forceinline__ void stage_query_f32(const uint8_t* queries, uint32_t pitch, uint32_t q, uint8_t* qs,
                                                int lane) {
    __syncwarp();  // the previous query's reads are done
    const float* src = reinterpret_cast<const float*>(queries + uint64_t(q) * pitch);
    double* dst = reinterpret_cast<double*>(qs);
    for (uint32_t i = lane; i < (pitch >> 2); i += 32) dst[i] = double(src[i]);
    __syncwarp();
}

// Scores entries [start, start + 32), [start + step, ...) of a list (DIRECT:
// the entries are the row slots themselves, i.e. rows [start, n)).
template <int R, bool DIRECT>
__device__ __forceinline__ void gather_list_f32(const uint8_t* rows, uint32_t pitch, const uint32_t* list, uint32_t n,
                                                uint32_t start, uint32_t step, const uint8_t* qs, uint8_t*,
                                                int lane, WarpTopK2<R>& tk, const uint32_t* idtab) {
    const uint32_t chunks = pitch >> 4;
    const double2* qd = reinterpret_cast<const double2*>(qs);
    for (uint32_t base = start; base < n; base += step) {
        const uint32_t me = f32_entry<DIRECT>(list, base + lane, n);
        double acc = 0.0;
        if (me != kEmpty) {
            // lane = row: the row streams through registers 4 chunks (16
            // floats) at a time, the loads of a group issued before its terms
            const float4* src = reinterpret_cast<const float4*>(rows + uint64_t(me) * pitch);
            for (uint32_t c0 = 0; c0 < chunks; c0 += 4) {
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    v[u] = c0 + u < chunks ? __ldg(src + c0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t c = c0 + u;
                    if (c < chunks) {
                        const double2 q01 = qd[2 * c], q23 = qd[2 * c + 1];
                        acc = __dadd_rn(acc, sq_term(v[u].x, q01.x));
                        acc = __dadd_rn(acc, sq_term(v[u].y, q01.y));
                        acc = __dadd_rn(acc, sq_term(v[u].z, q23.x));
                        acc = __dadd_rn(acc, sq_term(v[u].w, q23.y));
                    }
                }
            }
        }
        const uint64_t sb = uint64_t(__double_as_longlong(acc));
        uint32_t sl = me;
        if (idtab) {  // physical row -> id slot for rows that can enter the top-k
            const bool pre = me != kEmpty && sb <= tk.ta;
            if (__any_sync(kFull, pre) && pre) sl = __ldg(idtab + me);
        }
        tk.offer(me != kEmpty ? sb : kNone, me != kEmpty ? sl : 0xFFFFFFFFu, lane);
    }
}

template <int R>
__device__ __forceinline__ void write_result_f32(const RefineArgs& a, uint32_t q, const WarpTopK2<R>& fin, int lane,
                                                 uint32_t U) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t e = uint32_t(lane) * R + r;
        if (e < a.k) {
            const uint64_t o = uint64_t(q) * a.k + e;
            const bool none = fin.a[r] == kNone;
            a.out_ids[o] = none ? ~0ull : a.id_base + uint64_t(fin.b[r]) * a.id_stride;
            a.out_sqdist_f64[o] = none ? __longlong_as_double(0x7FF0000000000000ll) : __longlong_as_double(fin.a[r]);
        }
    }
    if (lane == 0) a.out_len[q] = U < a.k ? U : a.k;
}

template <int R>
__global__ void __launch_bounds__(kF32Threads) k_gather_f32(RefineArgs a, const uint32_t* __restrict__ lists,
                                                            const uint32_t* __restrict__ counts,
                                                            uint32_t lstride) {
    extern __shared__ __align__(128) uint8_t f32_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* tile = nullptr;
    uint8_t* qs = f32_smem + warp * f32_warp_smem(a.pitch);
    const uint32_t qstep = gridDim.x * (kF32Threads / 32);
    for (uint32_t q = (blockIdx.x * kF32Threads + threadIdx.x) >> 5; q < a.nq; q += qstep) {
        const uint32_t n = __ldcg(counts + q);
        const uint32_t qq = a.qorder ? __ldg(a.qorder + q) : q;  // list q holds query qq
        stage_query_f32(a.queries, a.pitch, qq, qs, lane);
        WarpTopK2<R> tk;
        tk.init(int(a.k));
        gather_list_f32<R, false>(a.rows, a.pitch, lists + uint64_t(q) * lstride, n, 0, kF32Rows, qs, tile, lane, tk,
                                  a.idtab);
        write_result_f32<R>(a, qq, tk, lane, n);
    }
}

// Merge NW warp-local pair lists (shared memory) into warp 0's top-k.
template <int R, int NW>
__device__ __forceinline__ void merge_warps_f32(WarpTopK2<R>& tk, uint64_t* ma, uint32_t* mb, uint32_t k, int lane,
                                                int warp) {
    constexpr int KCAP = 32 * R;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        ma[warp * KCAP + lane * R + r] = tk.a[r];
        mb[warp * KCAP + lane * R + r] = tk.b[r];
    }
    __syncthreads();
    if (warp == 0) {
        tk.init(int(k));
        const uint32_t kr = (k + 31) & ~31u;
        for (int w = 0; w < NW; ++w)
            for (uint32_t i = 0; i < kr; i += 32) tk.offer(ma[w * KCAP + i + lane], mb[w * KCAP + i + lane], lane);
    }
}

template <int R, int NW>
__global__ void __launch_bounds__(NW * 32) k_gather_cta_f32(RefineArgs a, const uint32_t* __restrict__ lists,
                                                            const uint32_t* __restrict__ counts, uint32_t lstride) {
    extern __shared__ __align__(128) uint8_t f32_smem[];
    __shared__ uint64_t ma[NW * 32 * R];
    __shared__ uint32_t mb[NW * 32 * R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* tile = nullptr;
    uint8_t* qs = f32_smem + warp * f32_warp_smem(a.pitch);
    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        const uint32_t n = __ldcg(counts + q);
        const uint32_t qq = a.qorder ? __ldg(a.qorder + q) : q;
        stage_query_f32(a.queries, a.pitch, qq, qs, lane);
        WarpTopK2<R> tk;
        tk.init(int(a.k));
        gather_list_f32<R, false>(a.rows, a.pitch, lists + uint64_t(q) * lstride, n, warp * kF32Rows, NW * kF32Rows,
                                  qs, tile, lane, tk, a.idtab);
        merge_warps_f32<R, NW>(tk, ma, mb, a.k, lane, warp);
        if (warp == 0) write_result_f32<R>(a, qq, tk, lane, n);
        __syncthreads();
    }
}

template <class K>
hcg_status f32_smem_opt_in(K kern, size_t smem) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return set_error(HCG_ECAPACITY, "f32 gather: shared-memory tile too large");
    return HCG_OK;
}

template <int R>
hcg_status gather_f32_launch(const RefineArgs& a, const uint32_t* lists, const uint32_t* counts, uint32_t lstride,
                             int sms, cudaStream_t st) {
    const size_t wsm = f32_warp_smem(a.pitch);
    if (a.nq * 2 < uint32_t(sms) * 16 * 8) {
        auto kern = k_gather_cta_f32<R, kF32CtaWarps>;
        HCG_RET_IF(f32_smem_opt_in(kern, kF32CtaWarps * wsm));
        kern<<<a.nq, kF32CtaWarps * 32, kF32CtaWarps * wsm, st>>>(a, lists, counts, lstride);
        return check_launch("k_gather_cta_f32");
    }
    constexpr int W = kF32Threads / 32;
    auto kern = k_gather_f32<R>;
    HCG_RET_IF(f32_smem_opt_in(kern, W * wsm));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kF32Threads, W * wsm);
    const uint32_t blocks = std::min<uint32_t>((a.nq + W - 1) / W, uint32_t(sms) * uint32_t(std::max(per_sm, 1)));
    kern<<<blocks, kF32Threads, W * wsm, st>>>(a, lists, counts, lstride);
    return check_launch("k_gather_f32");
}

// K3b (register variant, the default for C x take <= 32 x 256): each thread
// holds its <= JMAX window ids in registers (coalesced loads, no staging).
// Round r: every pending id stores (id << 32 | position) into slot h_r(id) of
// a u64 shared table; after a barrier it reads the slot back -- the same id:
// the id is resolved, and this copy is its first copy iff the stored position
// is its own; another id: collision, retried with the next hash.  All copies
// of an id hit the same slot, so they resolve in the same round.  Ids still
// colliding after kRegRounds go through an atomicCAS pass on the cleared table
// (measured: a CAS pass for every round-1 collision instead is 1.6x slower).
// Kept ids are compacted with one block scan.
constexpr int kRegRounds = 4;
constexpr int kListRounds = 6;

template <int JMAX, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) k_union_reg(RefineArgs a, uint32_t* __restrict__ lists,
                                                  uint32_t* __restrict__ counts, uint32_t lstride, uint32_t tb) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(smem);  // [1 << tb]
    const uint32_t** sptr = reinterpret_cast<const uint32_t**>(tab + (size_t(1) << tb));
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sptr + a.C);  // [NT/32] scan scratch
    const uint32_t T = a.C * a.take;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t take = a.take, shift = 32 - tb, tmask = (1u << tb) - 1;
    for (uint32_t c = tid; c < a.C; c += NT) sptr[c] = a.slots[c];
    __syncthreads();
    constexpr uint32_t kWarps = NT / 32;
    // Layouts: a warp per curve (coalesced 128-B window reads) when the warps
    // divide evenly over the curves; else a fixed curve per thread; else a walk.
    const int layout = kWarps % a.C == 0 ? 0 : (NT % a.C == 0 ? 1 : 2);

    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        // (the previous query's scan barriers ordered every read of tab / wsum)
        const uint32_t qq = a.qorder ? __ldg(a.qorder + q) : q;  // list q holds query qq
        uint32_t id[JMAX];
        uint32_t pending = 0;
        if (layout == 0) {
            const uint32_t c = warp % a.C, step = 32 * (kWarps / a.C);
            const uint32_t* src = sptr[c] + __ldg(a.begins + uint64_t(qq) * a.C + c);
            uint32_t p = lane + 32 * (warp / a.C);
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                id[j] = 0;
                if (p < take) {
                    id[j] = __ldg(src + p);
                    pending |= 1u << j;
                }
                p += step;
            }
        } else if (layout == 1) {
            const uint32_t c = tid % a.C, step = NT / a.C;
            const uint32_t* src = sptr[c] + __ldg(a.begins + uint64_t(qq) * a.C + c);
            uint32_t p = tid / a.C;
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                id[j] = 0;
                if (p < take) {
                    id[j] = __ldg(src + p);
                    pending |= 1u << j;
                }
                p += step;
            }
        } else {
            const uint32_t* bq = a.begins + uint64_t(qq) * a.C;
            uint32_t c = 0, p = tid;
            while (p >= take && c + 1 < a.C) {
                p -= take;
                ++c;
            }
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                const uint32_t i = tid + j * NT;
                id[j] = 0;
                if (i < T) {
                    id[j] = __ldg(sptr[c] + __ldg(bq + c) + p);
                    pending |= 1u << j;
                }
                p += NT;
                while (p >= take && c + 1 < a.C) {
                    p -= take;
                    ++c;
                }
            }
        }
        uint32_t keep = 0;
        // Round 1 over every id (register-resident); about a quarter of the
        // ids collide and stay pending.
        bool left;
        {
            const uint32_t mul = 0x9E3779B1u;
#pragma unroll
            for (int j = 0; j < JMAX; ++j)
                if ((pending >> j) & 1)
                    tab[(id[j] * mul) >> shift] = (uint64_t(id[j]) << 32) | uint32_t(tid + j * NT);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                if ((pending >> j) & 1) {
                    const uint64_t o = tab[(id[j] * mul) >> shift];
                    if (uint32_t(o >> 32) == id[j]) {
                        pending &= ~(1u << j);
                        if (uint32_t(o) == uint32_t(tid + j * NT)) keep |= 1u << j;
                    }
                }
            }
            left = __syncthreads_or(pending != 0);
        }
        // Later rounds over a compacted list: the pending (id, position) pairs
        // move to shared memory (aliasing the table: round 1's reads are
        // done) and the rounds cost what is left, not JMAX predicated slots
        // per thread.  A u16 table of list indices at twice the slots resolves
        // them in ~2 rounds.  Copies of an id resolve together, as before.
        uint32_t lkeep = 0;  // kept list entries of this thread (bit u: entry tid + u * NT)
        bool listed = false;
        uint2* lst = reinterpret_cast<uint2*>(smem);  // [cap] (id, position)
        const uint32_t cap = (1u << tb) >> 1;
        if (left && a.union_list) {
            const uint32_t np = __popc(pending);
            const uint32_t loff = block_excl_scan_u<NT>(np, wsum);
            uint32_t P = 0;
#pragma unroll
            for (int w = 0; w < int(kWarps); ++w) P += wsum[w];
            if (P <= cap) {  // block-uniform
                listed = true;
                uint32_t wpos = loff;
#pragma unroll
                for (int j = 0; j < JMAX; ++j)
                    if ((pending >> j) & 1) lst[wpos++] = make_uint2(id[j], uint32_t(tid + j * NT));
                pending = 0;
                __syncthreads();
                uint16_t* t16 = reinterpret_cast<uint16_t*>(lst + cap);  // [2 << tb]
                const uint32_t shift16 = shift - 1;
                uint32_t lpend = 0;
                for (uint32_t u = 0; tid + u * NT < P; ++u) lpend |= 1u << u;
                bool lleft = true;
#pragma unroll 1
                for (int r = 1; r <= kListRounds && lleft; ++r) {
                    const uint32_t mul = 0x9E3779B1u + 0x7F4A7C16u * uint32_t(r) * 2u;  // odd
                    for (uint32_t pm = lpend; pm; pm &= pm - 1) {
                        const uint32_t i = tid + uint32_t(__ffs(pm) - 1) * NT;
                        t16[(lst[i].x * mul) >> shift16] = uint16_t(i);
                    }
                    __syncthreads();
                    for (uint32_t pm = lpend; pm; pm &= pm - 1) {
                        const uint32_t u = uint32_t(__ffs(pm) - 1), i = tid + u * NT;
                        const uint32_t o = t16[(lst[i].x * mul) >> shift16];
                        if (lst[o].x == lst[i].x) {
                            lpend &= ~(1u << u);
                            if (o == i) lkeep |= 1u << u;
                        }
                    }
                    lleft = __syncthreads_or(lpend != 0);
                }
                // leftovers (rare): every copy of such an id is still pending;
                // the lowest list index is its first copy
                for (uint32_t pm = lpend; pm; pm &= pm - 1) {
                    const uint32_t u = uint32_t(__ffs(pm) - 1), i = tid + u * NT;
                    bool first = true;
                    for (uint32_t i2 = 0; i2 < i && first; ++i2) first = lst[i2].x != lst[i].x;
                    if (first) lkeep |= 1u << u;
                }
                left = false;
            }
        }
#pragma unroll 1
        for (int r = 1; r < kRegRounds && left; ++r) {
            const uint32_t mul = 0x9E3779B1u + 0x7F4A7C16u * uint32_t(r) * 2u;  // odd
#pragma unroll
            for (int j = 0; j < JMAX; ++j)
                if ((pending >> j) & 1)
                    tab[(id[j] * mul) >> shift] = (uint64_t(id[j]) << 32) | uint32_t(tid + j * NT);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                if ((pending >> j) & 1) {
                    const uint64_t o = tab[(id[j] * mul) >> shift];
                    if (uint32_t(o >> 32) == id[j]) {
                        pending &= ~(1u << j);
                        if (uint32_t(o) == uint32_t(tid + j * NT)) keep |= 1u << j;
                    }
                }
            }
            left = __syncthreads_or(pending != 0);  // also orders this round's reads before the next stores
        }
        if (left) {  // rare: CAS set over the cleared table
            for (uint32_t i = tid; i <= tmask; i += NT) tab[i] = ~0ull;
            __syncthreads();
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                if ((pending >> j) & 1) {
                    const unsigned long long mine = (uint64_t(id[j]) << 32) | uint32_t(tid + j * NT);
                    uint32_t h = hash_slot(id[j]) >> shift;
                    while (true) {
                        const unsigned long long prev = atomicCAS(&tab[h], ~0ull, mine);
                        if (prev == ~0ull) {
                            keep |= 1u << j;
                            break;
                        }
                        if (uint32_t(prev >> 32) == id[j]) break;
                        h = (h + 1) & tmask;
                    }
                }
            }
        }
        const uint32_t mine = __popc(keep) + __popc(lkeep);
        const uint32_t off = block_excl_scan_u<NT>(mine, wsum);
        uint32_t* out = lists + uint64_t(q) * lstride + off;
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < JMAX; ++j)
            if ((keep >> j) & 1) out[w++] = id[j];
        for (uint32_t pm = lkeep; pm; pm &= pm - 1) out[w++] = lst[tid + uint32_t(__ffs(pm) - 1) * NT].x;
        HCG_DASSERT(off + mine <= T && off + mine <= lstride);
        if (tid == NT - 1) counts[q] = off + mine;
        if (listed) __syncthreads();  // list reads before the next query's table writes
    }
}

// Sort keys of a batch: curve 0's window start per query (+ iota values).
// (window start >> shift: a coarse order is enough for locality)
__global__ void k_qkeys(const uint32_t* __restrict__ begins, uint32_t C, uint32_t nq, uint32_t shift,
                        uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    keys[q] = begins[uint64_t(q) * C] >> shift;
    vals[q] = q;
}

// Candidate-union tap: unique slots -> ids.
__global__ void k_lists_to_ids(RefineArgs a, const uint32_t* __restrict__ lists, const uint32_t* __restrict__ counts,
                               uint32_t lstride) {  // lstride: entries per query list
    const uint32_t q = blockIdx.x;
    if (q >= a.nq) return;
    const uint32_t n = counts[q];
    const uint32_t lim = n < a.cap ? n : a.cap;
    if (a.out_ids)
        for (uint32_t i = threadIdx.x; i < lim; i += blockDim.x)
        {
            const uint32_t p = lists[uint64_t(q) * lstride + i];
            a.out_ids[uint64_t(q) * a.cap + i] = a.id_base + uint64_t(a.idtab ? a.idtab[p] : p) * a.id_stride;
        }
    if (threadIdx.x == 0) a.out_len[q] = n;
}

// K3b for large curves x depth (T > kUnionMaxT or beyond the shared budget):
// the same candidate union with an atomicCAS hash set in a per-CTA GLOBAL
// scratch table (cleared per query), ids read straight from the curves;
// unique ids are appended (warp-aggregated) to the query's list in HBM.
__global__ void __launch_bounds__(kRefineThreads) k_union_cas(RefineArgs a, uint32_t* __restrict__ lists,
                                                              uint32_t* __restrict__ counts, uint32_t lstride,
                                                              uint32_t tb, uint32_t* __restrict__ gtables) {
    __shared__ uint32_t cnt;
    const uint32_t T = a.C * a.take;
    uint32_t* table = gtables + (uint64_t(blockIdx.x) << tb);
    const uint32_t tsize = 1u << tb, tmask = tsize - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt_s();
    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        for (uint32_t i = tid; i < tsize; i += kRefineThreads) table[i] = kEmpty;
        if (tid == 0) cnt = 0;
        __syncthreads();
        uint32_t* out = lists + uint64_t(q) * lstride;
        for (uint32_t c = 0; c < a.C; ++c) {
            const uint32_t* sl = a.slots[c] + a.begins[uint64_t(q) * a.C + c];
            for (uint32_t p0 = warp * 32; p0 < a.take; p0 += kRefineThreads) {
                const uint32_t p = p0 + lane;
                const bool has = p < a.take;
                const uint32_t s = has ? __ldg(sl + p) : 0u;
                bool fresh = false;
                if (has) {
                    uint32_t h = hash_slot(s) >> (32 - tb);
                    while (true) {
                        const uint32_t prev = atomicCAS(&table[h], kEmpty, s);
                        if (prev == kEmpty) {
                            fresh = true;
                            break;
                        }
                        if (prev == s) break;
                        h = (h + 1) & tmask;
                    }
                }
                const unsigned b = __ballot_sync(kFull, fresh);
                if (b) {
                    const int leader = __ffs(b) - 1;
                    uint32_t base = 0;
                    if (lane == leader) base = atomicAdd(&cnt, uint32_t(__popc(b)));
                    base = __shfl_sync(kFull, base, leader);
                    if (fresh) {
                        HCG_DASSERT(base + __popc(b & lt) < lstride && s < a.n_rows);
                        out[base + __popc(b & lt)] = s;
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) counts[q] = cnt;
        __syncthreads();
    }
    (void)T;
}

namespace {
int r_bucket(uint32_t k) { return k <= 32 ? 1 : k <= 64 ? 2 : k <= 128 ? 4 : 8; }

template <class K>
hcg_status opt_in_smem(K kern, int device, bool* configured) {
    if (device < 64 && !configured[device]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRefineMaxSmem) != cudaSuccess ||
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess)
            return set_error(HCG_ECUDA, "refine: cannot opt in to dynamic shared memory");
        configured[device] = true;
    }
    return HCG_OK;
}

uint32_t persistent_grid(const void* kern, size_t smem, int device, uint32_t nq) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRefineThreads, smem);
    return std::min<uint32_t>(nq, uint32_t(dev_info(device).sms * std::max(per_sm, 1)));
}

size_t union_smem_bytes(uint32_t C, uint32_t T, uint32_t tb) {
    return size_t(C) * 16 + 32 + size_t(T) * 8 + (size_t(4) << tb);
}


template <int JMAX, int NT>
hcg_status union_reg_launch(const RefineArgs& a, uint32_t* lists, uint32_t* counts, uint32_t lstride, uint32_t tb,
                            int device, cudaStream_t st) {
    // occupancy over registers: 6 CTAs/SM measured 1.45x faster than the
    // compiler's 64-register choice at JMAX=12 (latency-bound kernel)
    auto kern = k_union_reg<JMAX, NT, (NT == 256 ? (JMAX <= 12 ? 6 : (JMAX <= 16 ? 5 : 3)) : 1)>;
    const size_t smem = (size_t(8) << tb) + size_t(a.C) * 12 + 4 * (NT / 32) + 64;
    static bool cfg[64] = {};
    HCG_RET_IF(opt_in_smem(kern, device, cfg));
    static int per_sm_cache[64][32] = {};  // by device and table bits (the smem size)
    int& per_sm = per_sm_cache[device & 63][tb & 31];
    if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
        per_sm = std::max(per_sm, 1);
    }
    const uint32_t grid = std::min<uint32_t>(a.nq, uint32_t(dev_info(device).sms * per_sm));
    kern<<<grid, NT, smem, st>>>(a, lists, counts, lstride, tb);
    return check_launch("k_union_reg");
}

template <int NT>
hcg_status union_reg_dispatch(const RefineArgs& a, uint32_t* lists, uint32_t* counts, uint32_t lstride, uint32_t tb,
                              int device, cudaStream_t st) {
    constexpr uint32_t kWarps = NT / 32;
    const uint32_t jn = kWarps % a.C == 0 ? (a.take + 32 * (kWarps / a.C) - 1) / (32 * (kWarps / a.C))
                        : NT % a.C == 0   ? (a.take + NT / a.C - 1) / (NT / a.C)
                                          : (a.C * a.take + NT - 1) / NT;
    if (jn > 32) return set_error(HCG_ECAPACITY, "union: more than 32 ids per thread");
    if (jn <= 4) return union_reg_launch<4, NT>(a, lists, counts, lstride, tb, device, st);
    if (jn <= 8) return union_reg_launch<8, NT>(a, lists, counts, lstride, tb, device, st);
    if (jn <= 12) return union_reg_launch<12, NT>(a, lists, counts, lstride, tb, device, st);
    if (jn <= 16) return union_reg_launch<16, NT>(a, lists, counts, lstride, tb, device, st);
    if (jn <= 24) return union_reg_launch<24, NT>(a, lists, counts, lstride, tb, device, st);
    return union_reg_launch<32, NT>(a, lists, counts, lstride, tb, device, st);
}

// 256-thread CTAs measured best at T = 2800 (128: +15 %, 512: +18 %, 1024: +75 % union time).
hcg_status launch_union_reg(const RefineArgs& a, uint32_t* lists, uint32_t* counts, uint32_t lstride, uint32_t tb,
                            int device, cudaStream_t st) {
    // small candidate sets (the sharded per-shard depths): 128-thread CTAs,
    // union at T = 640 / 1072 / 1808: 0.42 / 0.67 / 1.06 ms vs 0.55 / 0.73 /
    // 0.98 ms with 256 threads
    if (a.C * a.take <= 1280 && 128 % a.C == 0) return union_reg_dispatch<128>(a, lists, counts, lstride, tb, device, st);
    return union_reg_dispatch<256>(a, lists, counts, lstride, tb, device, st);
}

// Query chunk so the per-call list scratch stays within kListBudget.
constexpr size_t kListBudget = size_t(2) << 30;

// Largest candidate walk C x take a query may have (the union's hash table
// is sized from it; 2^27 entries keeps every table index in 32 bits).
constexpr uint64_t kMaxWalk = uint64_t(1) << 27;

// The union-less K3c (k_gather_nu) serves k <= 128, u8 rows in curve-0
// order and batches of >= 16K queries; everything else runs the separate
// union (K3b) + K3c.  One predicate for the scratch query and the launch.
// k <= 16 is faster union-less at every depth; wider lists pay for their
// merges in the walk, which beats the union + gather from moderate walks on;
// the union gather's 64-entry list (k <= 64) takes per-pass offers, the
// others a queue (k_gather), so the crossover moves up at k = 64.  Measured at
// 10M, C = 8, 100K queries, same box interleaved
// (profiles/r02_gather_queue4.jsonl, ms): C x take = 2800 (D = 350) k = 64:
// union-less 6.39 vs union 6.79; k = 100: 6.89 vs 6.66; k = 128: 7.72 (the
// previous union gather) vs 6.72; C x take = 1024 (D = 128): the union at
// every k > 16 (r02_gather_queue2.jsonl: 2.54-3.00 vs 2.70-4.41 ms); C x take
// = 8192 (D = 1024): union-less 15.9-19.2 vs 23.4-23.7 at every k.
constexpr uint32_t kUnionlessWalk = 2048;     // C x take from which 16 < k <= 64 walks union-less
constexpr uint32_t kUnionlessWalkWide = 4096; // ... 64 < k <= 112
constexpr uint32_t kUnionlessWalkR8 = 6144;   // ... 112 < k <= 128
// The union-less walk's list widths R = 1 / 2 / 4 / 8 by k (launch_gather_nu).
#ifndef HCG_NU_R1_MAXK
#define HCG_NU_R1_MAXK 16
#endif
constexpr uint32_t kNuR1MaxK = HCG_NU_R1_MAXK, kNuR2MaxK = 48, kNuR4MaxK = 112;

template <int R>
bool unionless_path(const RefineArgs& a) {
    static const bool off = knob("HCG_NO_UNIONLESS") != nullptr;  // A/B: separate union for every k
    static const bool wide = knob("HCG_UNIONLESS_WIDE") != nullptr;  // A/B: union-less for every k <= 128
    if (R > 4 || a.k > 128 || off) return false;
    const uint64_t walk = uint64_t(a.C) * a.take;
    const uint64_t need = a.k <= kNuR1MaxK ? 0 : a.k <= 64 ? kUnionlessWalk
                          : a.k <= kNuR4MaxK ? kUnionlessWalkWide : kUnionlessWalkR8;
    if (!wide && walk < need) return false;
    return a.mode != kOutCandidates && a.dtype == HCG_U8 && a.nq >= 16384 && a.idtab != nullptr;
}

// The union-less walk's list width: offers are queued and a full queue of
// min(32, 32 R - k) is merged + deduplicated at a time
// (WarpTopK::offer_queued); each width serves the k that leave a queue of
// >= 16.
#ifndef HCG_NU_MINB1
#define HCG_NU_MINB1 3
#endif
#ifndef HCG_NU_MINB2
#define HCG_NU_MINB2 3
#endif
#ifndef HCG_NU_MINB4
#define HCG_NU_MINB4 2
#endif
#ifndef HCG_NU_MINB8
#define HCG_NU_MINB8 2
#endif
template <int CR, bool SMALLC>
hcg_status launch_gather_nu(const RefineArgs& a, int device, int sms, cudaStream_t st) {
    auto nk = a.k <= kNuR1MaxK   ? k_gather_nu<1, CR, HCG_NU_MINB1, SMALLC>
              : a.k <= kNuR2MaxK ? k_gather_nu<2, CR, HCG_NU_MINB2, SMALLC>
              : a.k <= kNuR4MaxK ? k_gather_nu<4, CR, HCG_NU_MINB4, SMALLC>
                                 : k_gather_nu<8, CR, HCG_NU_MINB8, SMALLC>;
    const int kb = a.k <= kNuR1MaxK ? 0 : a.k <= kNuR2MaxK ? 1 : a.k <= kNuR4MaxK ? 2 : 3;
    static int per_sm_cache[64][4] = {};
    int& per_sm = per_sm_cache[device & 63][kb];
    if (per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nk, kRefineThreads, 0);
        per_sm = std::max(per_sm, 1);
    }
    const uint32_t blocks = std::min<uint32_t>((a.nq + 7) / 8, uint32_t(sms * per_sm));
    count_launches(1);
    nk<<<blocks, kRefineThreads, 0, st>>>(a);
    return check_launch("k_gather_nu");
}

template <int R, int CR>
hcg_status refine_dispatch(const RefineArgs& a_in, void* scratch, size_t* scratch_bytes, int device, cudaStream_t st) {
    if (uint64_t(a_in.C) * a_in.take > kMaxWalk)
        return set_error(HCG_ECAPACITY, "candidate walk curves x probe depth exceeds 2^27 entries");
    const uint32_t T = a_in.C * a_in.take;
    uint32_t tb = 5;
    while ((uint64_t(1) << tb) * 7 < uint64_t(T) * 10) ++tb;
    if (tb > 28) return set_error(HCG_ECAPACITY, "candidate set too large");
    const bool nu = unionless_path<R>(a_in);
    const uint32_t lstride = (T + 31) & ~31u;  // 128-B aligned per-query lists
    // the shared-memory union's tag table at <= ~0.35 load factor
    const uint32_t utb = std::min<uint32_t>(tb + 1, 16);
    const size_t usmem = union_smem_bytes(a_in.C, T, utb);
    const bool smem_union = T <= kUnionMaxT && usmem <= 160 * 1024;
    static const bool force_smem_union = knob("HCG_UNION_SMEM") != nullptr;
    const bool reg_union = T <= 32u * 256 && (size_t(8) << tb) <= 128 * 1024 && !force_smem_union;
    const int sms = dev_info(device).sms;
    const uint32_t chunk = uint32_t(std::max<size_t>(1, std::min<size_t>(a_in.nq, kListBudget / (size_t(lstride) * 4))));
    const uint32_t cas_ctas = uint32_t(sms) * 4;
    // the union-less walk reads the windows in place: no lists, counts or tables
    const size_t lists_bytes = nu ? 0 : size_t(chunk) * lstride * 4;
    const size_t counts_bytes = nu ? 0 : (size_t(chunk) * 4 + 255) & ~size_t(255);
    const size_t table_bytes = (nu || smem_union) ? 0 : (size_t(cas_ctas) << tb) * 4;
    // Large batches run in curve-0 window order: queries processed at the
    // same time share candidate rows (rows are stored in curve-0 order), so
    // part of the gather hits L2 (measured 5.15 -> 4.75 ms at 100K queries).
    static const bool no_qsort = knob("HCG_NO_QSORT") != nullptr;
    const bool qsort = !no_qsort && (nu || reg_union) && a_in.mode != kOutCandidates && a_in.nq >= 16384 &&
                       (nu || chunk >= a_in.nq) && a_in.idtab != nullptr;  // both gathers map list q -> qorder[q]
    const size_t qsort_bytes = qsort ? size_t(a_in.nq) * 24 + radix_counts_bytes(a_in.nq) + 256 : 0;
    if (!scratch) {
        *scratch_bytes = lists_bytes + counts_bytes + table_bytes + qsort_bytes;
        return HCG_OK;
    }
    if (a_in.nq == 0) return HCG_OK;
    uint32_t* lists = static_cast<uint32_t*>(scratch);
    uint32_t* counts = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + lists_bytes);
    uint32_t* gtab = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + lists_bytes + counts_bytes);
    const uint32_t* qorder = nullptr;
    if (qsort) {
        uint8_t* base = static_cast<uint8_t*>(scratch) + lists_bytes + counts_bytes + table_bytes;
        uint64_t* k0 = reinterpret_cast<uint64_t*>(base);
        uint64_t* k1 = k0 + a_in.nq;
        uint32_t* v0 = reinterpret_cast<uint32_t*>(k1 + a_in.nq);
        uint32_t* v1 = v0 + a_in.nq;
        uint32_t* cnt = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(v1 + a_in.nq) + 255) & ~uintptr_t(255));
        uint32_t* totals = cnt + (radix_counts_bytes(a_in.nq) / 4 - 256);
        count_launches(1);
        // one 8-bit pass over the window start's top bits (n / 256 rows per bucket)
        constexpr uint32_t qbits = 8;  // measured: 8 / 16 / 24 bits within 0.5 % of each other
        uint32_t nbits = 1;
        while (nbits < 32 && (uint64_t(1) << nbits) < a_in.n_rows) ++nbits;
        const uint32_t shift = nbits > qbits ? nbits - qbits : 0u;
        k_qkeys<<<unsigned((a_in.nq + 255) / 256), 256, 0, st>>>(a_in.begins, a_in.C, a_in.nq, shift, k0, v0);
        HCG_RET_IF(check_launch("k_qkeys"));
        uint32_t dmask = 0;
        for (uint32_t d = 0; d * 8 < std::min(qbits, nbits); ++d) dmask |= 1u << d;
        HCG_RET_IF(radix_sort_pairs(&k0, &v0, &k1, &v1, a_in.nq, dmask, cnt, totals, st));
        qorder = v0;
    }
    // 3 CTAs/SM (72 registers): with rows and batches in curve-0 order fewer
    // queries in flight share more of their rows in L2 -- 4.70 ms vs 4.89 at
    // 4 CTAs/SM (1-2: 4.70, 5: spills); before the reorder 4 was best
    auto gk = k_gather<R, CR, R <= 4 ? 3 : 2>;
    static bool cfg_u[64] = {};
    if (smem_union) HCG_RET_IF(opt_in_smem(k_union, device, cfg_u));
    static int g_per_sm_cache[64] = {};
    int& g_per_sm = g_per_sm_cache[device & 63];
    if (g_per_sm == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_per_sm, gk, kRefineThreads, 0);
        g_per_sm = std::max(g_per_sm, 1);
    }
    if (nu) {
        // large batches: skip the union, walk the windows directly.  k <= 32
        // at 3 CTAs/SM (72 registers): 2 leaves DRAM latency uncovered, 4
        // forces 64 registers and spills the top-k (profiles/r01_nu_occupancy_ab.txt).
        RefineArgs a = a_in;
        a.qorder = qorder;
        if (a.ev_mid) cudaEventRecord(a.ev_mid, st);  // timed split: (batch order) | fused gather
        return a.C <= 32 ? launch_gather_nu<CR, true>(a, device, sms, st) : launch_gather_nu<CR, false>(a, device, sms, st);
    }
    for (uint32_t q0 = 0; q0 < a_in.nq; q0 += chunk) {
        RefineArgs a = a_in;
        a.qorder = qorder;
        a.nq = std::min(chunk, a_in.nq - q0);
        a.queries = a_in.queries + uint64_t(q0) * a_in.pitch;
        a.begins = a_in.begins + uint64_t(q0) * a_in.C;
        if (a.out_ids) a.out_ids += uint64_t(q0) * (a_in.mode == kOutCandidates ? a_in.cap : a_in.k);
        if (a.out_sqdist) a.out_sqdist += uint64_t(q0) * a_in.k;
        if (a.out_len) a.out_len += q0;
        if (a.out_packed) a.out_packed += uint64_t(q0) * a_in.k;
        if (reg_union) {
            HCG_RET_IF(launch_union_reg(a, lists, counts, lstride, tb, device, st));
        } else if (smem_union) {
            const uint32_t ugrid = persistent_grid(reinterpret_cast<const void*>(k_union), usmem, device, a.nq);
            k_union<<<ugrid, kRefineThreads, usmem, st>>>(a, lists, counts, lstride, utb);
        } else {
            k_union_cas<<<std::min(a.nq, cas_ctas), kRefineThreads, 0, st>>>(a, lists, counts, lstride, tb, gtab);
        }
        HCG_RET_IF(check_launch("candidate union"));
        count_launches(2);  // the union and its consumer (gather or the lists -> ids tap)
        if (a.ev_mid && q0 + chunk >= a_in.nq) cudaEventRecord(a.ev_mid, st);
        if (a.mode == kOutCandidates) {
            k_lists_to_ids<<<a.nq, 128, 0, st>>>(a, lists, counts, lstride);
            HCG_RET_IF(check_launch("k_lists_to_ids"));
            continue;
        }
        if (a.dtype == HCG_F32) {
            if (a.out_sqdist_f64) a.out_sqdist_f64 += uint64_t(q0) * a_in.k;
            HCG_RET_IF(gather_f32_launch<R>(a, lists, counts, lstride, sms, st));
            continue;
        }
        if (a.nq * 2 < uint32_t(sms) * uint32_t(std::max(g_per_sm, 1)) * 8) {
            // fewer queries than half the resident warps: spread each query over a CTA (latency)
            bool wide = false;
            if constexpr (R <= 2) {
                if (a.nq <= uint32_t(sms)) {  // very small batches: 32 warps per query
                    k_gather_cta<R, CR, 32><<<a.nq, 1024, 0, st>>>(a, lists, counts, lstride);
                    wide = true;
                }
            }
            if (!wide) k_gather_cta<R, CR, 8><<<a.nq, kRefineThreads, 0, st>>>(a, lists, counts, lstride);
            HCG_RET_IF(check_launch("k_gather_cta"));
            continue;
        }
        const uint32_t blocks = std::min<uint32_t>((a.nq + 7) / 8, uint32_t(sms * std::max(g_per_sm, 1)));
        gk<<<blocks, kRefineThreads, 0, st>>>(a, lists, counts, lstride);
        HCG_RET_IF(check_launch("k_gather"));
    }
    return HCG_OK;
}

template <int R>
hcg_status refine_cr(const RefineArgs& a, void* scratch, size_t* sb, int device, cudaStream_t st) {
    const uint32_t chunks = a.pitch / 16;
    if (chunks <= 8) return refine_dispatch<R, 1>(a, scratch, sb, device, st);
    if (chunks <= 16) return refine_dispatch<R, 2>(a, scratch, sb, device, st);
    return refine_dispatch<R, 4>(a, scratch, sb, device, st);
}
}  // namespace

bool refine_unionless(const RefineArgs& a) {
    switch (r_bucket(a.k)) {
        case 1: return unionless_path<1>(a);
        case 2: return unionless_path<2>(a);
        case 4: return unionless_path<4>(a);
        default: return unionless_path<8>(a);
    }
}

hcg_status launch_refine(const RefineArgs& a, void* scratch, size_t* scratch_bytes, int device, cudaStream_t st) {
    if (scratch_bytes) *scratch_bytes = 0;
    switch (r_bucket(a.k)) {
        case 1: return refine_cr<1>(a, scratch, scratch_bytes, device, st);
        case 2: return refine_cr<2>(a, scratch, scratch_bytes, device, st);
        case 4: return refine_cr<4>(a, scratch, scratch_bytes, device, st);
        default: return refine_cr<8>(a, scratch, scratch_bytes, device, st);
    }
}

// ------------------------------------------------------------------ K4 ----
template <int R>
__global__ void __launch_bounds__(256) k_merge(const uint64_t* __restrict__ packed, uint32_t parts, uint32_t nq,
                                               uint32_t k, uint64_t* __restrict__ out_ids,
                                               uint32_t* __restrict__ out_sq, uint32_t* __restrict__ out_len) {
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= nq) return;
    const uint32_t q = uint32_t(gw);
    WarpTopK<R> tk;
    tk.init(int(k));
    for (uint32_t p = 0; p < parts; ++p) {
        const uint64_t* src = packed + (uint64_t(p) * nq + q) * k;
        for (uint32_t i = 0; i < k; i += 32) {
            const uint64_t cand = i + lane < k ? src[i + lane] : kNone;
            tk.offer(cand, lane);
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t e = uint32_t(lane) * R + r;
        if (e < k) {
            const uint64_t x = tk.a[r];
            const bool none = x == kNone;
            HCG_DASSERT(e < k && q < nq);
            out_ids[uint64_t(q) * k + e] = none ? ~0ull : (x & 0xFFFFFFFFull);
            out_sq[uint64_t(q) * k + e] = none ? 0xFFFFFFFFu : uint32_t(x >> 32);
            cnt += none ? 0 : 1;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
    if (lane == 0) out_len[q] = cnt;
}

hcg_status launch_merge(const uint64_t* packed, uint32_t parts, uint32_t nq, uint32_t k, uint64_t* out_ids,
                        uint32_t* out_sqdist, uint32_t* out_len, cudaStream_t st) {
    if (nq == 0) return HCG_OK;
    count_launches(1);
    const unsigned blocks = unsigned((uint64_t(nq) * 32 + 255) / 256);
    switch (r_bucket(k)) {
        case 1: k_merge<1><<<blocks, 256, 0, st>>>(packed, parts, nq, k, out_ids, out_sqdist, out_len); break;
        case 2: k_merge<2><<<blocks, 256, 0, st>>>(packed, parts, nq, k, out_ids, out_sqdist, out_len); break;
        case 4: k_merge<4><<<blocks, 256, 0, st>>>(packed, parts, nq, k, out_ids, out_sqdist, out_len); break;
        default: k_merge<8><<<blocks, 256, 0, st>>>(packed, parts, nq, k, out_ids, out_sqdist, out_len); break;
    }
    return check_launch("k_merge");
}

// ------------------------------------------------------------------ K5 ----
constexpr uint32_t kBruteChunk = 32768;

template <int R, int QPW>
__global__ void __launch_bounds__(256) k_brute(BruteArgs a, uint64_t* __restrict__ part) {
    extern __shared__ uint32_t bsm[];
    const uint32_t wpr = a.pitch / 4, rstride = wpr + 1;
    uint32_t* tile = bsm;
    uint32_t* qs = bsm + 256 * rstride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t chunk = blockIdx.x;
    const uint32_t qb = blockIdx.y * 8 * QPW;
    for (uint32_t i = tid; i < 8 * QPW * wpr; i += 256) {
        const uint32_t qi = i / wpr, w = i - qi * wpr, q = qb + qi;
        qs[i] = q < a.nq ? reinterpret_cast<const uint32_t*>(a.queries + uint64_t(q) * a.pitch)[w] : 0u;
    }
    WarpTopK<R> tk[QPW];
#pragma unroll
    for (int j = 0; j < QPW; ++j) tk[j].init(int(a.k));
    const uint64_t r0 = uint64_t(chunk) * kBruteChunk;
    const uint64_t r1 = min(a.n, r0 + kBruteChunk);
    for (uint64_t t0 = r0; t0 < r1; t0 += 256) {
        __syncthreads();
        for (uint32_t i = tid; i < 256 * wpr; i += 256) {
            const uint32_t row = i / wpr, w = i - row * wpr;
            const uint64_t gr = t0 + row;
            tile[row * rstride + w] = gr < r1 ? reinterpret_cast<const uint32_t*>(a.rows + gr * a.pitch)[w] : 0u;
        }
        __syncthreads();
        for (int s = 0; s < 8; ++s) {
            const uint32_t rr = s * 32 + lane;
            const uint64_t gr = t0 + rr;
            const bool valid = gr < r1;
            uint32_t acc[QPW];
#pragma unroll
            for (int j = 0; j < QPW; ++j) acc[j] = 0;
            for (uint32_t w = 0; w < wpr; ++w) {
                const uint32_t rv = tile[rr * rstride + w];
#pragma unroll
                for (int j = 0; j < QPW; ++j) {
                    const uint32_t d = __vabsdiffu4(rv, qs[(warp * QPW + j) * wpr + w]);
                    acc[j] = __dp4a(d, d, acc[j]);
                }
            }
            const uint64_t gid = a.id_base + (a.idtab && valid ? __ldg(a.idtab + gr) : gr) * a.id_stride;
#pragma unroll
            for (int j = 0; j < QPW; ++j) tk[j].offer(valid ? ((uint64_t(acc[j]) << 32) | gid) : kNone, lane);
        }
    }
#pragma unroll
    for (int j = 0; j < QPW; ++j) {
        const uint32_t q = qb + warp * QPW + j;
        if (q < a.nq) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t e = uint32_t(lane) * R + r;
                if (e < a.k) part[(uint64_t(chunk) * a.nq + q) * a.k + e] = tk[j].a[r];
            }
        }
    }
}

size_t brute_scratch_bytes(const BruteArgs& a) {
    const uint64_t chunks = (a.n + kBruteChunk - 1) / kBruteChunk;
    const size_t cc = size_t(chunks) * a.nq * a.k * (a.dtype == HCG_F32 ? 12 : 8);
    return brute_tc_eligible(a) ? std::max(cc, brute_tc_scratch_bytes(a)) : cc;
}

template <int R, int QPW>
static hcg_status brute_launch(const BruteArgs& a, uint64_t* scratch, cudaStream_t st) {
    const uint32_t chunks = uint32_t((a.n + kBruteChunk - 1) / kBruteChunk);
    const uint32_t wpr = a.pitch / 4;
    const size_t smem = (size_t(256) * (wpr + 1) + size_t(8) * QPW * wpr) * 4;
    auto kern = k_brute<R, QPW>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return set_error(HCG_ECAPACITY, "brute-force tile too large");
    dim3 grid(chunks, (a.nq + 8 * QPW - 1) / (8 * QPW));
    kern<<<grid, 256, smem, st>>>(a, scratch);
    return check_launch("k_brute");
}

// f32 rows: warp per (query, chunk of rows) through the exact gather path,
// then a pair merge over the chunks.  Scratch: chunks x nq x k (u64 key, u32 slot).
template <int R>
__global__ void __launch_bounds__(kF32CtaWarps * 32) k_brute_f32(BruteArgs a, uint64_t* __restrict__ part_a,
                                                                 uint32_t* __restrict__ part_b) {
    extern __shared__ __align__(128) uint8_t f32_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t chunk = blockIdx.x, q = blockIdx.y * kF32CtaWarps + warp;
    if (q >= a.nq) return;
    uint8_t* tile = nullptr;
    uint8_t* qs = f32_smem + warp * f32_warp_smem(a.pitch);
    const uint64_t r0 = uint64_t(chunk) * kBruteChunk;
    const uint32_t r1 = uint32_t(min(a.n, r0 + kBruteChunk));
    stage_query_f32(a.queries, a.pitch, q, qs, lane);
    WarpTopK2<R> tk;
    tk.init(int(a.k));
    gather_list_f32<R, true>(a.rows, a.pitch, nullptr, r1, uint32_t(r0), kF32Rows, qs, tile, lane, tk, a.idtab);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t e = uint32_t(lane) * R + r;
        if (e < a.k) {
            part_a[(uint64_t(chunk) * a.nq + q) * a.k + e] = tk.a[r];
            part_b[(uint64_t(chunk) * a.nq + q) * a.k + e] = tk.b[r];
        }
    }
}

template <int R>
__global__ void __launch_bounds__(256) k_merge_f32(const uint64_t* __restrict__ part_a,
                                                   const uint32_t* __restrict__ part_b, uint32_t parts, BruteArgs a,
                                                   uint64_t* __restrict__ out_ids, double* __restrict__ out_sq,
                                                   uint32_t* __restrict__ out_len) {
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= a.nq) return;
    const uint32_t q = uint32_t(gw), k = a.k;
    WarpTopK2<R> tk;
    tk.init(int(k));
    for (uint32_t p = 0; p < parts; ++p) {
        const uint64_t off = (uint64_t(p) * a.nq + q) * k;
        for (uint32_t i = 0; i < k; i += 32) {
            const bool in = i + lane < k;
            tk.offer(in ? part_a[off + i + lane] : kNone, in ? part_b[off + i + lane] : 0xFFFFFFFFu, lane);
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t e = uint32_t(lane) * R + r;
        if (e < k) {
            const bool none = tk.a[r] == kNone;
            out_ids[uint64_t(q) * k + e] = none ? ~0ull : a.id_base + uint64_t(tk.b[r]) * a.id_stride;
            out_sq[uint64_t(q) * k + e] = none ? __longlong_as_double(0x7FF0000000000000ll) : __longlong_as_double(tk.a[r]);
            cnt += none ? 0 : 1;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
    if (lane == 0) out_len[q] = cnt;
}

template <int R>
static hcg_status brute_f32_launch(const BruteArgs& a, uint64_t* scratch, uint64_t* out_ids, double* out_sq,
                                   uint32_t* out_len, cudaStream_t st) {
    const uint32_t chunks = uint32_t((a.n + kBruteChunk - 1) / kBruteChunk);
    uint64_t* pa = scratch;
    uint32_t* pb = reinterpret_cast<uint32_t*>(scratch + uint64_t(chunks) * a.nq * a.k);
    const size_t smem = kF32CtaWarps * size_t(f32_warp_smem(a.pitch));
    HCG_RET_IF(f32_smem_opt_in(k_brute_f32<R>, smem));
    k_brute_f32<R><<<dim3(chunks, (a.nq + kF32CtaWarps - 1) / kF32CtaWarps), kF32CtaWarps * 32, smem, st>>>(a, pa, pb);
    HCG_RET_IF(check_launch("k_brute_f32"));
    k_merge_f32<R><<<unsigned((uint64_t(a.nq) * 32 + 255) / 256), 256, 0, st>>>(pa, pb, chunks, a, out_ids, out_sq,
                                                                                 out_len);
    return check_launch("k_merge_f32");
}

hcg_status launch_brute(const BruteArgs& a, uint64_t* scratch, uint64_t* out_ids, uint32_t* out_sqdist,
                        uint32_t* out_len, double* out_sqdist_f64, cudaStream_t st) {
    if (a.nq == 0) return HCG_OK;
    const uint32_t chunks = uint32_t((a.n + kBruteChunk - 1) / kBruteChunk);
    if (a.dtype == HCG_F32) {
        switch (r_bucket(a.k)) {
            case 1: return brute_f32_launch<1>(a, scratch, out_ids, out_sqdist_f64, out_len, st);
            case 2: return brute_f32_launch<2>(a, scratch, out_ids, out_sqdist_f64, out_len, st);
            case 4: return brute_f32_launch<4>(a, scratch, out_ids, out_sqdist_f64, out_len, st);
            default: return brute_f32_launch<8>(a, scratch, out_ids, out_sqdist_f64, out_len, st);
        }
    }
    if (brute_tc_eligible(a)) return launch_brute_tc(a, scratch, out_ids, out_sqdist, out_len, st);
    hcg_status rc;
    switch (r_bucket(a.k)) {
        case 1: rc = brute_launch<1, 4>(a, scratch, st); break;
        case 2: rc = brute_launch<2, 2>(a, scratch, st); break;
        case 4: rc = brute_launch<4, 1>(a, scratch, st); break;
        default: rc = brute_launch<8, 1>(a, scratch, st); break;
    }
    if (rc != HCG_OK) return rc;
    return launch_merge(scratch, chunks, a.nq, a.k, out_ids, out_sqdist, out_len, st);
}

}  // namespace hcg
