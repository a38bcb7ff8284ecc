// search.cu -- batched query path on the B200 (Alg. 2).
//
//   K3a k_locate : one thread per (query, curve): project + quantize + curve
//                  key (fused K1), compare against the curve's common key
//                  prefix, lower_bound over the sorted suffix keys
//                  (SubIndex::rank_of, multicurves.hpp:57-58) and the window
//                  begin (SubIndex::window, multicurves.hpp:60-63).
//   K3b k_refine : one CTA per query: read every curve's window of slots
//                  (coalesced), dedup them in a shared-memory hash set
//                  (candidate_union, multicurves.hpp:87-89), gather the
//                  candidate descriptors with 128-bit streaming loads (8 lanes
//                  per 128-B row, 8 rows in flight per lane), exact integer
//                  squared L2 (vecio.cpp:87-95) with vabsdiff4+dp4a, and a
//                  warp-register top-k on packed (sqdist<<32 | slot), which is
//                  the reference's (distance, id) order (vecio.cpp:101-113).
//   K4  k_merge  : one warp per query, k-way merge of per-shard / per-chunk
//                  sorted lists (hypershard aggregate).
//   K5  k_brute  : exact kNN over all rows (brute_force_knn, vecio.cpp:115-122)
//                  for recall ground truth; chunked, then merged by K4.
#include <algorithm>

#include "hcg_internal.cuh"
#include "hcg_host.hpp"

namespace hcg {

__device__ __forceinline__ unsigned lanemask_lt_s() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ----------------------------------------------------------------- K3a ----
template <int DMAX, int WSMAX>
__global__ void __launch_bounds__(128) k_locate(LocateArgs a) {
    constexpr int WMAX = DMAX / 2 > kMaxKeyWords ? kMaxKeyWords : (DMAX / 2 < 1 ? 1 : DMAX / 2);
    __shared__ uint32_t lut[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = a.lut[i];
    __syncthreads();
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(a.nq) * a.C) return;
    const uint32_t q = uint32_t(t / a.C), c = uint32_t(t % a.C);
    const CurveDev& cv = a.curves[c];
    const int d = int(cv.dims);

    uint32_t x[DMAX];
    const uint8_t* row = a.queries + uint64_t(q) * a.pitch;
    const uint16_t* asg = a.assign + cv.off;
#pragma unroll
    for (int s = 0; s < DMAX; ++s) x[s] = s < d ? lut[__ldg(row + __ldg(asg + s))] : 0u;
    uint64_t key[WMAX];
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
        uint64_t lo = 0, len = a.n;
        while (len > 0) {
            const uint64_t half = len >> 1;
            const uint64_t mid = lo + half;
            const uint64_t* e = keys + mid * ws;
            int o = 0;
#pragma unroll
            for (int w = WSMAX - 1; w >= 0; --w) {
                if (o == 0 && w < ws) {
                    const uint64_t ev = __ldg(e + w);
                    o = ev < qs[w] ? -1 : (ev > qs[w] ? 1 : 0);
                }
            }
            if (o < 0) {
                lo = mid + 1;
                len -= half + 1;
            } else {
                len = half;
            }
        }
        rank = lo;
    }
    const uint64_t take = a.depth < a.n ? a.depth : a.n;
    const uint64_t below_n = take / 2;
    uint64_t begin = rank >= below_n ? rank - below_n : 0;
    if (begin + take > a.n) begin = a.n - take;
    a.out_begin[t] = uint32_t(begin);
    if (a.out_rank) a.out_rank[t] = rank;
}

template <int DMAX, int WSMAX>
static void locate_launch(const LocateArgs& a, cudaStream_t st) {
    const uint64_t total = uint64_t(a.nq) * a.C;
    k_locate<DMAX, WSMAX><<<unsigned((total + 127) / 128), 128, 0, st>>>(a);
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

template <int R, int CR>
__global__ void __launch_bounds__(kRefineThreads) k_refine(RefineArgs a, uint32_t table_bits, uint32_t* gtables) {
    constexpr int KCAP = 32 * R;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* mbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* sbeg = reinterpret_cast<uint32_t*>(mbuf + 8 * KCAP);
    uint32_t* scount = sbeg + a.C;
    uint32_t* list = scount + 4;
    uint32_t* table = gtables ? gtables + (uint64_t(blockIdx.x) << table_bits) : list + uint64_t(a.C) * a.take;
    const uint32_t tsize = 1u << table_bits, tmask = tsize - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, l8 = lane & 7, grp = lane >> 3;
    const uint32_t chunks = a.pitch >> 4;
    const unsigned lt = lanemask_lt_s();

    for (uint32_t q = blockIdx.x; q < a.nq; q += gridDim.x) {
        for (uint32_t i = tid; i < tsize; i += kRefineThreads) table[i] = kEmpty;
        for (uint32_t c = tid; c < a.C; c += kRefineThreads) sbeg[c] = a.begins[uint64_t(q) * a.C + c];
        if (tid == 0) *scount = 0;
        uint4 qv[CR];
        const uint8_t* qrow = a.queries + uint64_t(q) * a.pitch;
#pragma unroll
        for (int t = 0; t < CR; ++t) {
            const uint32_t ch = l8 + 8 * t;
            qv[t] = ch < chunks ? *reinterpret_cast<const uint4*>(qrow + ch * 16) : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();

        // -- candidate union: windows of every curve, dedup in the hash set.
        for (uint32_t c = 0; c < a.C; ++c) {
            const uint32_t* sl = a.slots[c] + sbeg[c];
            for (uint32_t p0 = warp * 32; p0 < a.take; p0 += kRefineThreads) {
                const uint32_t p = p0 + lane;
                const bool has = p < a.take;
                const uint32_t s = has ? __ldg(sl + p) : 0u;
                bool fresh = false;
                if (has) {
                    uint32_t h = hash_slot(s) >> (32 - table_bits);
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
                    if (lane == leader) base = atomicAdd(scount, uint32_t(__popc(b)));
                    base = __shfl_sync(kFull, base, leader);
                    if (fresh) list[base + __popc(b & lt)] = s;
                }
            }
        }
        __syncthreads();
        const uint32_t U = *scount;

        if (a.mode == kOutCandidates) {
            const uint32_t lim = U < a.cap ? U : a.cap;
            if (a.out_ids)
                for (uint32_t i = tid; i < lim; i += kRefineThreads)
                    a.out_ids[uint64_t(q) * a.cap + i] = a.id_base + uint64_t(list[i]) * a.id_stride;
            if (tid == 0) a.out_len[q] = U;
            __syncthreads();
            continue;
        }

        // -- gather + exact distance + per-warp top-k.
        WarpTopK<R> tk;
        tk.init(int(a.k));
        for (uint32_t base = warp * 32; base < U; base += kRefineThreads) {
            const uint32_t e0 = base + grp * 8;
            uint32_t sl[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) sl[r] = e0 + r < U ? list[e0 + r] : kEmpty;
            uint4 v[8][CR];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
                for (int t = 0; t < CR; ++t) {
                    const uint32_t ch = l8 + 8 * t;
                    v[r][t] = (sl[r] != kEmpty && ch < chunks)
                                  ? ldg_stream(a.rows + uint64_t(sl[r]) * a.pitch + ch * 16)
                                  : make_uint4(0, 0, 0, 0);
                }
            }
            uint32_t acc[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                acc[r] = 0;
#pragma unroll
                for (int t = 0; t < CR; ++t) acc[r] = sad2_16(v[r][t], qv[t], acc[r]);
            }
            // Reduce-scatter over the 8 lanes of the group: lane l8 ends with row l8.
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
            const uint32_t mine = e0 + l8 < U ? list[e0 + l8] : kEmpty;
            const uint64_t cand = mine != kEmpty ? ((uint64_t(S) << 32) | mine) : kNone;
            tk.offer(cand, lane);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) mbuf[warp * KCAP + lane * R + r] = tk.a[r];
        __syncthreads();
        if (warp == 0) {
            WarpTopK<R> fin;
            fin.init(int(a.k));
            const uint32_t kr = (a.k + 31) & ~31u;
            for (int w = 0; w < 8; ++w)
                for (uint32_t i = 0; i < kr; i += 32) fin.offer(mbuf[w * KCAP + i + lane], lane);
            write_result<R>(a, q, fin, lane, U);
        }
        __syncthreads();
    }
}

namespace {
int r_bucket(uint32_t k) { return k <= 32 ? 1 : k <= 64 ? 2 : k <= 128 ? 4 : 8; }

template <int R, int CR>
hcg_status refine_launch(const RefineArgs& a, uint32_t table_bits, bool gtab, void* scratch, size_t* scratch_bytes,
                         int device, cudaStream_t st) {
    auto kern = k_refine<R, CR>;
    const size_t fixed = size_t(8) * 32 * R * 8 + size_t(a.C) * 4 + 16 + size_t(a.C) * a.take * 4;
    const size_t smem = fixed + (gtab ? 0 : (size_t(4) << table_bits));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return set_error(HCG_ECAPACITY, "refine shared memory request too large");
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRefineThreads, smem);
    if (per_sm < 1) return set_error(HCG_ECAPACITY, "refine kernel does not fit on an SM");
    uint32_t grid = a.nq;
    if (gtab) grid = std::min<uint32_t>(a.nq, uint32_t(sms * per_sm));
    const size_t need = gtab ? (size_t(grid) << table_bits) * 4 : 0;
    if (!scratch) {
        *scratch_bytes = need;
        return HCG_OK;
    }
    if (a.nq == 0) return HCG_OK;
    kern<<<grid, kRefineThreads, smem, st>>>(a, table_bits, gtab ? static_cast<uint32_t*>(scratch) : nullptr);
    return check_launch("k_refine");
}

template <int R>
hcg_status refine_cr(const RefineArgs& a, uint32_t tb, bool gtab, void* scratch, size_t* sb, int device,
                     cudaStream_t st) {
    const uint32_t chunks = a.pitch / 16;
    if (chunks <= 8) return refine_launch<R, 1>(a, tb, gtab, scratch, sb, device, st);
    if (chunks <= 16) return refine_launch<R, 2>(a, tb, gtab, scratch, sb, device, st);
    return refine_launch<R, 4>(a, tb, gtab, scratch, sb, device, st);
}
}  // namespace

hcg_status launch_refine(const RefineArgs& a, void* scratch, size_t* scratch_bytes, int device, cudaStream_t st) {
    if (scratch_bytes) *scratch_bytes = 0;
    const uint64_t T = uint64_t(a.C) * a.take;
    // Hash set at <= 0.7 load factor, at least 32 slots.
    uint32_t tb = 5;
    while ((uint64_t(1) << tb) * 7 < T * 10) ++tb;
    if (tb > 30) return set_error(HCG_ECAPACITY, "candidate set too large");
    const size_t list_bytes = T * 4;
    if (list_bytes > 150 * 1024) return set_error(HCG_ECAPACITY, "curves x depth exceeds the per-query candidate capacity");
    const bool gtab = list_bytes + (size_t(4) << tb) > 160 * 1024;
    switch (r_bucket(a.k)) {
        case 1: return refine_cr<1>(a, tb, gtab, scratch, scratch_bytes, device, st);
        case 2: return refine_cr<2>(a, tb, gtab, scratch, scratch_bytes, device, st);
        case 4: return refine_cr<4>(a, tb, gtab, scratch, scratch_bytes, device, st);
        default: return refine_cr<8>(a, tb, gtab, scratch, scratch_bytes, device, st);
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
            const uint64_t gid = a.id_base + gr * a.id_stride;
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
    return size_t(chunks) * a.nq * a.k * 8;
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

hcg_status launch_brute(const BruteArgs& a, uint64_t* scratch, uint64_t* out_ids, uint32_t* out_sqdist,
                        uint32_t* out_len, cudaStream_t st) {
    if (a.nq == 0) return HCG_OK;
    const uint32_t chunks = uint32_t((a.n + kBruteChunk - 1) / kBruteChunk);
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
