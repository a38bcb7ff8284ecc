// build.cu -- index build on the B200: K1 key generation and K2 stable LSD
// radix sort of each curve's (key, slot) list.
//
// Reference behaviour (Alg. 1; multicurves.hpp:47-51,77):
// every vector is projected onto each curve's subspace, quantized, turned into
// an extended key, and each curve keeps its (key, id) entries sorted by key
// then id.  Here the input is already in slot (= id) order, so a STABLE sort
// by key alone reproduces the (key, id) order exactly.
//
// HBM layout produced per curve c:
//   keys[c]  : n x ws u64, suffix of the key below the curve's common prefix
//   slots[c] : n u32, row index of each sorted entry
#include <algorithm>
#include <vector>

#include "hcg_internal.cuh"
#include "hcg_host.hpp"

namespace hcg {

// ------------------------------------------------------------------ K1 ----
template <int DMAX>
struct KeyWords {
    static constexpr int value = DMAX / 2 > kMaxKeyWords ? kMaxKeyWords : (DMAX / 2 < 1 ? 1 : DMAX / 2);
};

// One thread per row: key of curve c (full width, SoA words) plus an OR/AND
// reduction over all keys that later yields the common prefix.
template <int DMAX, class T>
__global__ void __launch_bounds__(256) k_keygen(const uint8_t* __restrict__ rows, uint64_t n,
                                                uint32_t pitch, const uint16_t* __restrict__ assign_c,
                                                int d, int m, int kind, const uint32_t* __restrict__ lut_g,
                                                uint64_t* __restrict__ keys_soa, int W,
                                                unsigned long long* __restrict__ or_and, unsigned* bad) {
    constexpr int WMAX = KeyWords<DMAX>::value;
    __shared__ uint32_t lut[256];
    __shared__ uint16_t asg[DMAX];
    __shared__ uint64_t red_or[8][WMAX];
    __shared__ uint64_t red_and[8][WMAX];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    lut[tid] = lut_g[tid];
    if (tid < DMAX) asg[tid] = tid < d ? assign_c[tid] : 0;
    __syncthreads();

    const uint64_t i = uint64_t(blockIdx.x) * 256 + tid;
    const bool valid = i < n;
    uint64_t key[WMAX];
    if (valid) {
        uint32_t x[DMAX];
        const T* row = reinterpret_cast<const T*>(rows + i * pitch);
#pragma unroll
        for (int s = 0; s < DMAX; ++s) x[s] = s < d ? cell_of(__ldg(row + asg[s]), lut, m, bad) : 0u;
        make_key<DMAX, WMAX>(x, d, m, kind, key);
#pragma unroll
        for (int w = 0; w < WMAX; ++w)
            if (w < W) keys_soa[uint64_t(w) * n + i] = key[w];
    }
#pragma unroll
    for (int w = 0; w < WMAX; ++w) {
        uint64_t o = valid ? key[w] : 0ull;
        uint64_t a = valid ? key[w] : ~0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            o |= __shfl_xor_sync(kFull, o, off);
            a &= __shfl_xor_sync(kFull, a, off);
        }
        if (lane == 0) {
            red_or[warp][w] = o;
            red_and[warp][w] = a;
        }
    }
    __syncthreads();
    if (tid < W && tid < WMAX) {
        uint64_t o = 0, a = ~0ull;
        for (int k = 0; k < 8; ++k) {
            o |= red_or[k][tid];
            a &= red_and[k][tid];
        }
        atomicOr(or_and + tid, (unsigned long long)o);
        atomicAnd(or_and + W + tid, (unsigned long long)a);
    }
}

// ------------------------------------------------------------------ K2 ----
constexpr int kSortThreads = 256;
constexpr int kSortIpt = 8;
constexpr int kSortTile = kSortThreads * kSortIpt;  // 2048

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < 8 ? wsum[lane] : 0;
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, s, off);
            if (lane >= off) s += t;
        }
        if (lane < 8) wsum[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t before = warp ? wsum[warp - 1] : 0;
    const uint32_t r = before + inc - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kSortThreads) k_upsweep(const uint64_t* __restrict__ keys, uint64_t n,
                                                          int shift, uint32_t* __restrict__ counts,
                                                          uint32_t tiles) {
    __shared__ uint32_t h[8][256];
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 8 * 256; i += kSortThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t base = uint64_t(blockIdx.x) * kSortTile;
#pragma unroll
    for (int t = 0; t < kSortIpt; ++t) {
        const uint64_t idx = base + uint64_t(t) * kSortThreads + tid;
        if (idx < n) atomicAdd(&h[warp][(keys[idx] >> shift) & 255], 1u);
    }
    __syncthreads();
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += h[w][tid];
    counts[uint64_t(tid) * tiles + blockIdx.x] = s;
}

// One block per digit: exclusive scan of that digit's per-tile counts.
__global__ void __launch_bounds__(1024) k_scan_rows(uint32_t* __restrict__ counts, uint32_t tiles,
                                                    uint32_t* __restrict__ totals) {
    __shared__ uint32_t wsum[32];
    uint32_t* row = counts + uint64_t(blockIdx.x) * tiles;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < tiles; base += 1024) {
        const uint32_t v = base + tid < tiles ? row[base + tid] : 0;
        uint32_t inc = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, inc, off);
            if (lane >= off) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            uint32_t s = wsum[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, s, off);
                if (lane >= off) s += t;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const uint32_t excl = (warp ? wsum[warp - 1] : 0) + inc - v;
        if (base + tid < tiles) row[base + tid] = carry + excl;
        carry += wsum[31];
        __syncthreads();
    }
    if (tid == 0) totals[blockIdx.x] = carry;
}

// Stable scatter of one tile.  Warp w owns elements [w*256, w*256+256) of the
// tile and walks them in 8 coalesced rounds, so (warp, round, lane) is the
// original order; ranks come from per-warp digit counters and match_any.
// The tile is re-ordered in shared memory first so the global writes leave in
// per-digit runs.
__global__ void __launch_bounds__(kSortThreads) k_downsweep(
    const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t n, int shift, const uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ totals, uint32_t tiles) {
    __shared__ uint32_t whist[8][256];
    __shared__ uint32_t tile_off[256];
    __shared__ uint32_t gbase[256];
    __shared__ uint32_t wsum[8];
    __shared__ uint64_t skeys[kSortTile];
    __shared__ uint32_t svals[kSortTile];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 8 * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
    const uint32_t gex = block_excl_scan256(totals[tid], wsum);
    gbase[tid] = gex + counts[uint64_t(tid) * tiles + blockIdx.x];

    const uint64_t base = uint64_t(blockIdx.x) * kSortTile;
    const uint64_t wbase = base + uint64_t(warp) * (32 * kSortIpt);
    uint64_t k[kSortIpt];
    uint32_t v[kSortIpt], dg[kSortIpt], lr[kSortIpt];
#pragma unroll
    for (int t = 0; t < kSortIpt; ++t) {
        const uint64_t idx = wbase + uint64_t(t) * 32 + lane;
        const bool ok = idx < n;
        k[t] = ok ? kin[idx] : 0ull;
        v[t] = ok ? vin[idx] : 0u;
        dg[t] = ok ? uint32_t((k[t] >> shift) & 255) : 256u;
    }
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int t = 0; t < kSortIpt; ++t) {
        const unsigned peers = __match_any_sync(kFull, dg[t]);
        const uint32_t rank = __popc(peers & lt);
        const uint32_t b = dg[t] < 256 ? whist[warp][dg[t]] : 0u;
        __syncwarp();
        if (dg[t] < 256 && rank == 0) whist[warp][dg[t]] = b + __popc(peers);
        __syncwarp();
        lr[t] = b + rank;
    }
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t c = whist[w][tid];
        whist[w][tid] = run;
        run += c;
    }
    tile_off[tid] = block_excl_scan256(run, wsum);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kSortIpt; ++t) {
        if (dg[t] < 256) {
            const uint32_t li = tile_off[dg[t]] + whist[warp][dg[t]] + lr[t];
            skeys[li] = k[t];
            svals[li] = v[t];
        }
    }
    __syncthreads();
    const uint32_t tile_n = uint32_t(min(uint64_t(kSortTile), n - base));
    for (uint32_t i = tid; i < tile_n; i += kSortThreads) {
        const uint64_t key = skeys[i];
        const uint32_t d = uint32_t((key >> shift) & 255);
        const uint64_t g = uint64_t(gbase[d]) + (i - tile_off[d]);
        HCG_DASSERT(g < n);
        kout[g] = key;
        vout[g] = svals[i];
    }
}

// Raise *bad if any of the n x d floats (row pitch `pitch` bytes) is NaN / Inf.
__global__ void k_check_finite(const uint8_t* __restrict__ rows, uint64_t n, uint32_t pitch, uint32_t d,
                               unsigned* bad) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    const uint64_t r = i / d, j = i - r * d;
    const uint32_t b = reinterpret_cast<const uint32_t*>(rows + r * pitch)[j];
    if ((b & 0x7F800000u) == 0x7F800000u) *bad = 1u;
}

// Physical row order (see api.cu reorder_rows): dst[i] = src[perm[i]] for
// rows of `pitch` bytes (16-B vectors, a warp per 2 rows at pitch 128).
__global__ void k_permute_rows(const uint8_t* __restrict__ src, const uint32_t* __restrict__ perm, uint64_t n,
                               uint32_t pitch, uint8_t* __restrict__ dst) {
    const uint32_t vpr = pitch / 16;
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * vpr) return;
    const uint64_t r = i / vpr, v = i - r * vpr;
    reinterpret_cast<uint4*>(dst + r * pitch)[v] = __ldg(reinterpret_cast<const uint4*>(src + uint64_t(perm[r]) * pitch) + v);
}

// inv[perm[i]] = i
__global__ void k_invert(const uint32_t* __restrict__ perm, uint64_t n, uint32_t* __restrict__ inv) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) inv[perm[i]] = uint32_t(i);
}

// v[i] = map[v[i]]
__global__ void k_map(uint32_t* __restrict__ v, uint64_t n, const uint32_t* __restrict__ map) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = __ldg(map + v[i]);
}

// samples[j] = keys[j * kSampleStride] (ws words each)
__global__ void k_sample(const uint64_t* __restrict__ keys, uint64_t n_samples, uint32_t ws, uint32_t stride,
                         uint64_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_samples * ws) return;
    const uint64_t j = i / ws, w = i - j * ws;
    out[i] = keys[j * stride * ws + w];
}

__global__ void k_iota(uint32_t* v, uint64_t n, uint32_t base) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = base + uint32_t(i);
}

__global__ void k_offset(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n, uint32_t base) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = base + in[i];
}

__device__ __forceinline__ int cmp_words(const uint64_t* a, const uint64_t* b, int ws) {
    for (int w = ws - 1; w >= 0; --w) {
        const uint64_t x = a[w], y = b[w];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// Stable merge by rank (incremental insert, multicurves.hpp:52):
// resident entry i lands at i + #(new < key_i), new entry j at j + #(resident <= key_j),
// so equal keys keep the resident (lower-id) entries first.
__global__ void k_rank_merge(const uint64_t* __restrict__ ak, const uint32_t* __restrict__ as, uint64_t na,
                             const uint64_t* __restrict__ bk, const uint32_t* __restrict__ bs, uint64_t nb, int ws,
                             uint64_t* __restrict__ ck, uint32_t* __restrict__ cs) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= na + nb) return;
    const bool from_a = t < na;
    const uint64_t i = from_a ? t : t - na;
    const uint64_t* key = (from_a ? ak : bk) + i * ws;
    const uint64_t* other = from_a ? bk : ak;
    uint64_t lo = 0, len = from_a ? nb : na;
    while (len > 0) {  // from_a: lower_bound in B; else upper_bound in A
        const uint64_t half = len >> 1, mid = lo + half;
        const int c = cmp_words(other + mid * ws, key, ws);
        if (c < 0 || (!from_a && c == 0)) {
            lo = mid + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    const uint64_t pos = i + lo;
    HCG_DASSERT(pos < na + nb);
    for (int w = 0; w < ws; ++w) ck[pos * ws + w] = key[w];
    cs[pos] = from_a ? as[i] : bs[i];
}

__global__ void k_gather_word(const uint64_t* __restrict__ src, const uint32_t* __restrict__ perm,
                              uint64_t* __restrict__ dst, uint64_t n) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

// Sorted suffix keys, AoS (ws words per entry), bits above hv cleared.
__global__ void k_pack_suffix(const uint64_t* __restrict__ keys_soa, const uint32_t* __restrict__ perm,
                              uint64_t n, int ws, uint64_t top_mask, uint64_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = perm[i];
    for (int w = 0; w < ws; ++w) {
        uint64_t v = keys_soa[uint64_t(w) * n + s];
        if (w == ws - 1) v &= top_mask;
        out[i * ws + w] = v;
    }
}

// Re-expand sorted suffix keys to full-width keys (parity tap).
__global__ void k_expand_keys(const uint64_t* __restrict__ suffix, uint64_t n, int ws, int w_full,
                              CurveDev cv, uint64_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int w = 0; w < w_full; ++w) out[i * w_full + w] = cv.prefix[w] | (w < ws ? suffix[i * ws + w] : 0ull);
}

// ---------------------------------------------------------------- host ----
namespace {
inline unsigned blocks_for(uint64_t n, unsigned t) { return unsigned((n + t - 1) / t); }

template <int DMAX>
void launch_keygen(const uint8_t* rows, uint64_t n, uint32_t pitch, const uint16_t* assign_c, int d, int m,
                   int kind, const uint32_t* lut, uint64_t* keys_soa, int W, unsigned long long* or_and,
                   int dtype, unsigned* bad, cudaStream_t st) {
    if (dtype == HCG_F32)
        k_keygen<DMAX, float><<<blocks_for(n, 256), 256, 0, st>>>(rows, n, pitch, assign_c, d, m, kind, lut,
                                                                  keys_soa, W, or_and, bad);
    else
        k_keygen<DMAX, uint8_t><<<blocks_for(n, 256), 256, 0, st>>>(rows, n, pitch, assign_c, d, m, kind, lut,
                                                                    keys_soa, W, or_and, bad);
}
}  // namespace

hcg_status keygen_rows(const uint8_t* rows, uint64_t n, uint32_t pitch, const uint16_t* assign_c, int d, int m,
                       int kind, const uint32_t* lut, uint64_t* keys_soa, int W, unsigned long long* or_and,
                       int dmax, int dtype, unsigned* bad, cudaStream_t st) {
    if (n == 0) return HCG_OK;
    switch (dmax) {
        case 8: launch_keygen<8>(rows, n, pitch, assign_c, d, m, kind, lut, keys_soa, W, or_and, dtype, bad, st); break;
        case 16: launch_keygen<16>(rows, n, pitch, assign_c, d, m, kind, lut, keys_soa, W, or_and, dtype, bad, st); break;
        case 32: launch_keygen<32>(rows, n, pitch, assign_c, d, m, kind, lut, keys_soa, W, or_and, dtype, bad, st); break;
        case 64: launch_keygen<64>(rows, n, pitch, assign_c, d, m, kind, lut, keys_soa, W, or_and, dtype, bad, st); break;
        case 128: launch_keygen<128>(rows, n, pitch, assign_c, d, m, kind, lut, keys_soa, W, or_and, dtype, bad, st); break;
        default: return set_error(HCG_EINVAL, "unsupported curve dimension bucket");
    }
    return check_launch("k_keygen");
}

// Stable LSD radix sort of (key, val) pairs over the 8-bit digits selected by
// digit_mask (bit s -> digit at shift 8s).  Double-buffered; on return *k/*v
// hold the result.
hcg_status radix_sort_pairs(uint64_t** k, uint32_t** v, uint64_t** k_alt, uint32_t** v_alt, uint64_t n,
                            uint32_t digit_mask, uint32_t* counts, uint32_t* totals, cudaStream_t st) {
    if (n == 0 || digit_mask == 0) return HCG_OK;
    const uint32_t tiles = uint32_t((n + kSortTile - 1) / kSortTile);
    for (int s = 0; s < 8; ++s) {
        if (!((digit_mask >> s) & 1)) continue;
        const int shift = 8 * s;
        count_launches(3);
        k_upsweep<<<tiles, kSortThreads, 0, st>>>(*k, n, shift, counts, tiles);
        k_scan_rows<<<256, 1024, 0, st>>>(counts, tiles, totals);
        k_downsweep<<<tiles, kSortThreads, 0, st>>>(*k, *v, *k_alt, *v_alt, n, shift, counts, totals, tiles);
        std::swap(*k, *k_alt);
        std::swap(*v, *v_alt);
    }
    return check_launch("radix pass");
}

size_t radix_counts_bytes(uint64_t n) {
    const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
    return size_t(tiles) * 256 * 4 + 256 * 4;
}

void launch_check_finite(const uint8_t* rows, uint64_t n, uint32_t pitch, uint32_t d, unsigned* bad,
                         cudaStream_t st) {
    if (n) k_check_finite<<<blocks_for(n * d, 256), 256, 0, st>>>(rows, n, pitch, d, bad);
}

void launch_permute_rows(const uint8_t* src, const uint32_t* perm, uint64_t n, uint32_t pitch, uint8_t* dst,
                         cudaStream_t st) {
    if (n) k_permute_rows<<<blocks_for(n * (pitch / 16), 256), 256, 0, st>>>(src, perm, n, pitch, dst);
}
void launch_invert(const uint32_t* perm, uint64_t n, uint32_t* inv, cudaStream_t st) {
    if (n) k_invert<<<blocks_for(n, 256), 256, 0, st>>>(perm, n, inv);
}
void launch_map(uint32_t* v, uint64_t n, const uint32_t* map, cudaStream_t st) {
    if (n) k_map<<<blocks_for(n, 256), 256, 0, st>>>(v, n, map);
}

void launch_sample(const uint64_t* keys, uint64_t n_samples, uint32_t ws, uint32_t stride, uint64_t* out,
                   cudaStream_t st) {
    if (n_samples) k_sample<<<blocks_for(n_samples * ws, 256), 256, 0, st>>>(keys, n_samples, ws, stride, out);
}
void launch_iota(uint32_t* v, uint64_t n, uint32_t base, cudaStream_t st) {
    if (n) k_iota<<<blocks_for(n, 256), 256, 0, st>>>(v, n, base);
}
void launch_offset(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t base, cudaStream_t st) {
    if (n) k_offset<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n, base);
}
void launch_rank_merge(const uint64_t* ak, const uint32_t* as, uint64_t na, const uint64_t* bk, const uint32_t* bs,
                       uint64_t nb, int ws, uint64_t* ck, uint32_t* cs, cudaStream_t st) {
    if (na + nb) k_rank_merge<<<blocks_for(na + nb, 256), 256, 0, st>>>(ak, as, na, bk, bs, nb, ws, ck, cs);
}
void launch_gather_word(const uint64_t* src, const uint32_t* perm, uint64_t* dst, uint64_t n, cudaStream_t st) {
    if (n) k_gather_word<<<blocks_for(n, 256), 256, 0, st>>>(src, perm, dst, n);
}
void launch_pack_suffix(const uint64_t* keys_soa, const uint32_t* perm, uint64_t n, int ws, uint64_t top_mask,
                        uint64_t* out, cudaStream_t st) {
    if (n) k_pack_suffix<<<blocks_for(n, 256), 256, 0, st>>>(keys_soa, perm, n, ws, top_mask, out);
}
void launch_expand_keys(const uint64_t* suffix, uint64_t n, int ws, int w_full, const CurveDev& cv, uint64_t* out,
                        cudaStream_t st) {
    if (n) k_expand_keys<<<blocks_for(n, 256), 256, 0, st>>>(suffix, n, ws, w_full, cv, out);
}

}  // namespace hcg
