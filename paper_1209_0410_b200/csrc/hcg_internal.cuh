// hcg_internal.cuh -- shared device helpers and host/device structs of the
// B200 Hypercurves hot path (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hcg.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

// Device bounds checks, compiled in with -DHCG_DEBUG_BOUNDS (HCG_DEBUG_BOUNDS=1
// at build time); the normal build compiles them out.  compute-sanitizer is
// unavailable on the GPU pool, so the -m gpu suite is also run against this
// build (tools/debug_bounds.sh).
#ifdef HCG_DEBUG_BOUNDS
#include <cstdio>
#define HCG_DASSERT(c)                                                                        \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("hcg bounds check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);          \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define HCG_DASSERT(c) \
    do {               \
    } while (0)
#endif

namespace hcg {

constexpr int kMaxKeyWords = HCG_MAX_KEY_BITS / 64;  // 16
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint64_t kNone = ~0ull;
constexpr unsigned kFull = 0xFFFFFFFFu;

// Per-curve description used by the locate kernel.  The sorted subindex c is
// stored as suffix keys: every key of the curve shares the bits above `hv`
// (the highest bit that varies over the database), so only bits [0, hv] are
// kept, right-aligned in `ws` words (least significant word first).
struct CurveDev {
    const uint64_t* keys;   // n x ws suffix words, sorted
    const uint32_t* slots;  // n, slot (row index) of each sorted entry
    uint64_t prefix[kMaxKeyWords];  // full-width common key with bits <= hv cleared
    uint32_t hv;    // highest varying bit
    uint32_t ws;    // suffix words
    uint32_t w;     // full key words = ceil(dims * m / 64)
    uint32_t dims;  // projected dimensions feeding this curve
    uint32_t off;   // offset of this curve's slots in the assignment table
    const uint64_t* samples;  // every sample_stride-th key (ws words each): the L2-resident upper levels
    uint32_t n_samples;
    uint32_t sample_stride;
};
constexpr uint32_t kSampleStride = 32;  // default stride of the sampled keys (16-256 measured: 32 within 1 % of best)

// ---------------------------------------------------------------- keys ----
// Skilling's axes->transpose on m-bit coordinates held in registers; the
// coordinate count d is runtime (<= DMAX).  Branch-free form of the
// per-bit-plane rotation (reference: proj/src/curve.cpp:100-123).
template <int DMAX>
__device__ __forceinline__ void hilbert_transpose(uint32_t (&x)[DMAX], int d, int m) {
    for (uint32_t q = 1u << (m - 1); q > 1; q >>= 1) {
        const uint32_t low = q - 1;
#pragma unroll
        for (int i = 0; i < DMAX; ++i) {
            if (i < d) {
                const bool set = (x[i] & q) != 0;
                const uint32_t t = (x[0] ^ x[i]) & low;
                const uint32_t x0 = x[0] ^ (set ? low : t);
                if (i != 0) x[i] ^= set ? 0u : t;
                x[0] = x0;
            }
        }
    }
#pragma unroll
    for (int i = 1; i < DMAX; ++i)
        if (i < d) x[i] ^= x[i - 1];
    uint32_t last = 0;
#pragma unroll
    for (int i = 0; i < DMAX; ++i)
        if (i == d - 1) last = x[i];
    uint32_t fix = 0;
    for (uint32_t q = 1u << (m - 1); q > 1; q >>= 1)
        if (last & q) fix ^= q - 1;
#pragma unroll
    for (int i = 0; i < DMAX; ++i)
        if (i < d) x[i] ^= fix;
}

// key <<= s (1 <= s <= 128) on a WMAX-word little-endian integer.
template <int WMAX>
__device__ __forceinline__ void key_shl(uint64_t (&k)[WMAX], int s) {
    const int ws = s >> 6, bs = s & 63;
#pragma unroll
    for (int w = WMAX - 1; w >= 0; --w) {
        const uint64_t a0 = k[w];
        const uint64_t a1 = w >= 1 ? k[w - 1] : 0ull;
        const uint64_t a2 = w >= 2 ? k[w - 2] : 0ull;
        const uint64_t a3 = w >= 3 ? k[w - 3] : 0ull;
        const uint64_t hi = ws == 0 ? a0 : (ws == 1 ? a1 : a2);
        const uint64_t lo = ws == 0 ? a1 : (ws == 1 ? a2 : a3);
        k[w] = bs ? ((hi << bs) | (lo >> (64 - bs))) : hi;
    }
}

// Curve key of one projected point: plane j (MSB first) of coordinate i lands
// at key bit width-1-(j*d+i) (reference: proj/src/curve.cpp:62-75).
// cells: the m-bit quantized coordinates (LUT output).
// The default scheme's shape, 16 dims per curve at m = 8 or 16, with the
// loops unrolled at compile time: the Skilling transform on constants and the
// bit-plane interleave as a 16 x 16 bit-matrix transpose (4 block-swap
// stages) -- T[b] bit i = bit b of x[i]; plane b = brev16(T[b]) sits at key
// bits [16 b, 16 b + 16), the same key as the generic loop below.
// COMPACT: the bit-plane loop stays rolled (a tenth of the code; the
// latency kernel runs it once per query, from cold instruction caches).
template <int M, int WMAX, bool COMPACT = false>
__device__ __forceinline__ void make_key_d16(uint32_t (&x)[16], int kind, uint64_t (&key)[WMAX]) {
    if (kind == HCG_HILBERT) {
#pragma unroll(COMPACT ? 1 : M)
        for (uint32_t q = 1u << (M - 1); q > 1; q >>= 1) {
            const uint32_t low = q - 1;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const bool set = (x[i] & q) != 0;
                const uint32_t t = (x[0] ^ x[i]) & low;
                const uint32_t x0 = x[0] ^ (set ? low : t);
                if (i != 0) x[i] ^= set ? 0u : t;
                x[0] = x0;
            }
        }
#pragma unroll
        for (int i = 1; i < 16; ++i) x[i] ^= x[i - 1];
        uint32_t fix = 0;
#pragma unroll
        for (uint32_t q = 1u << (M - 1); q > 1; q >>= 1) fix ^= (x[15] & q) ? q - 1 : 0u;
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] ^= fix;
    }
#pragma unroll
    for (int j = 8; j >= 1; j >>= 1) {
        const uint32_t mask = j == 8 ? 0x00FFu : j == 4 ? 0x0F0Fu : j == 2 ? 0x3333u : 0x5555u;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (i & j) continue;
            const uint32_t t = ((x[i] >> j) ^ x[i + j]) & mask;
            x[i] ^= t << j;
            x[i + j] ^= t;
        }
    }
#pragma unroll
    for (int w = 0; w < WMAX; ++w) key[w] = 0;
#pragma unroll
    for (int b = 0; b < M; ++b) {
        const uint64_t plane = __brev(x[b]) >> 16;
        if (b / 4 < WMAX) key[b / 4] |= plane << (16 * (b % 4));
    }
}

template <int DMAX, int WMAX>
__device__ __forceinline__ void make_key(uint32_t (&x)[DMAX], int d, int m, int kind,
                                         uint64_t (&key)[WMAX]) {
    if constexpr (DMAX == 16 && WMAX >= 4) {
        if (d == 16 && m == 16) {
            make_key_d16<16, WMAX>(x, kind, key);
            return;
        }
        if (d == 16 && m == 8) {
            make_key_d16<8, WMAX>(x, kind, key);
            return;
        }
    }
    if (kind == HCG_HILBERT && d > 1) hilbert_transpose<DMAX>(x, d, m);
#pragma unroll
    for (int w = 0; w < WMAX; ++w) key[w] = 0;
    for (int j = 0; j < m; ++j) {
        const int sh = m - 1 - j;
        uint64_t c0 = 0, c1 = 0;
#pragma unroll
        for (int i = 0; i < DMAX; ++i) {
            if (i < d) {
                const uint64_t bit = (x[i] >> sh) & 1u;
                const int p = d - 1 - i;
                if (DMAX > 64 && p >= 64) c1 |= bit << (p - 64);
                else c0 |= bit << p;
            }
        }
        if (j > 0) key_shl<WMAX>(key, d);
        key[0] |= c0;
        if (WMAX > 1 && DMAX > 64) key[1] |= c1;
    }
}

// Quantized cell of one descriptor component (curve.cpp:166-174):
//  u8 : the view's 256-entry table (built on the host by the same rule);
//  f32: float_to_ordinal(x) >> (32 - m) on the device; a NaN / Inf component
//       raises *bad (the reference throws "non-finite component").
__device__ __forceinline__ uint32_t cell_of(uint8_t v, const uint32_t* lut, int, unsigned*) { return lut[v]; }
__device__ __forceinline__ uint32_t cell_of(float v, const uint32_t*, int m, unsigned* bad) {
    const uint32_t b = __float_as_uint(v);
    if ((b & 0x7F800000u) == 0x7F800000u) *bad = 1u;
    const uint32_t ord = (b >> 31) ? ~b : (b | 0x80000000u);
    return ord >> (32 - m);
}

// ------------------------------------------------------------ distance ----
// Squared L2 of 16 bytes, exact in u32: |a-b| per byte then a byte dot product.
__device__ __forceinline__ uint32_t sad2_16(const uint4& a, const uint4& b, uint32_t acc) {
    uint32_t d;
    d = __vabsdiffu4(a.x, b.x); acc = __dp4a(d, d, acc);
    d = __vabsdiffu4(a.y, b.y); acc = __dp4a(d, d, acc);
    d = __vabsdiffu4(a.z, b.z); acc = __dp4a(d, d, acc);
    d = __vabsdiffu4(a.w, b.w); acc = __dp4a(d, d, acc);
    return acc;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ------------------------------------------------------------ warp top-k ----
// Bitonic sort of one u64 per lane, ascending over the warp (15 exchanges).
__device__ __forceinline__ uint64_t warp_sort_asc(uint64_t c, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t y = __shfl_xor_sync(kFull, c, j);
            const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
            c = keep_min ? (c < y ? c : y) : (c < y ? y : c);
        }
    }
    return c;
}

// Keep the N = 32*R smallest of a sorted blocked list a (element e in lane
// e / R, register e % R) and a warp-sorted b (one per lane): c_i = min(a_i,
// b_{N-1-i}) is bitonic and holds exactly those N, a bitonic merge sorts it.
template <int R>
__device__ __forceinline__ void merge_sorted32(uint64_t (&a)[R], uint64_t b, int lane) {
    constexpr int N = 32 * R;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int t = lane * R + r - (N - 32);
        const uint64_t y = __shfl_sync(kFull, b, (31 - t) & 31);
        if (t >= 0 && y < a[r]) a[r] = y;
    }
#pragma unroll
    for (int j = N / 2; j >= 1; j >>= 1) {
        if (j >= R) {
            const int lj = j / R;
            const bool lower = (lane & lj) == 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t y = __shfl_xor_sync(kFull, a[r], lj);
                a[r] = lower ? (a[r] < y ? a[r] : y) : (a[r] < y ? y : a[r]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if ((r & j) == 0) {
                    const uint64_t x = a[r], y = a[r | j];
                    a[r] = x < y ? x : y;
                    a[r | j] = x < y ? y : x;
                }
            }
        }
    }
}

// Offers passing the threshold in one call at or above which WarpTopK sorts
// them and merges the whole batch instead of inserting them one by one.
#ifndef HCG_TOPK_BATCH_MIN
#define HCG_TOPK_BATCH_MIN 6
#endif
constexpr int kTopkBatchMin = HCG_TOPK_BATCH_MIN;

// A warp holds a sorted (ascending) list of KCAP = 32*R packed (sqdist<<32 |
// slot) values in registers, blocked layout: element e lives in lane e / R,
// register e % R.  Packing makes the reference's (distance, id) order
// (vecio.cpp:102-105) a plain integer order.
template <int R>
struct WarpTopK {
    static constexpr int kR = R;
    uint64_t a[R];
    uint64_t thr;  // current k-th smallest (kNone until k elements seen)
    int thr_lane, thr_reg;

    __device__ __forceinline__ void init(int k) {
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = kNone;
        thr = kNone;
        thr_lane = (k - 1) / R;
        thr_reg = (k - 1) % R;
    }

    __device__ __forceinline__ void update_thr() {
        // arithmetic select: a runtime-indexed a[thr_reg] would spill the
        // list to local memory
        uint64_t mine = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) mine |= a[r] & (0ull - uint64_t(r == thr_reg));
        thr = __shfl_sync(kFull, mine, thr_lane);
    }

    // Insert a warp-uniform value x (must be distinct from every held value).
    __device__ __forceinline__ void insert(uint64_t x, int lane) {
        const uint64_t prev_last = __shfl_up_sync(kFull, a[R - 1], 1);
        const bool first_lt = lane == 0 || prev_last < x;
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            const uint64_t p = r == 0 ? prev_last : a[r - 1];
            const bool p_lt = r == 0 ? first_lt : (a[r - 1] < x);
            if (!p_lt) a[r] = p;
            else if (a[r] > x) a[r] = x;
        }
        update_thr();
    }

    // Offer one candidate per lane (kNone = no candidate).  Many passing
    // offers (the fill phase of a large k) are sorted and merged in one go;
    // BATCH1 extends that to R = 1 (the latency kernel: its warps each fill
    // a fresh list from few passes).
    template <bool BATCH1 = false>
    __device__ __forceinline__ void offer(uint64_t cand, int lane) {
        unsigned m = __ballot_sync(kFull, cand < thr);
        if ((R >= 2 || BATCH1) && __popc(m) >= kTopkBatchMin) {
            merge_sorted32<R>(a, warp_sort_asc(cand < thr ? cand : kNone, lane), lane);
            update_thr();
            return;
        }
        while (m) {
            const int src = __ffs(m) - 1;
            const uint64_t x = __shfl_sync(kFull, cand, src);
            insert(x, lane);
            m &= ~(1u << src);
            m &= __ballot_sync(kFull, cand < thr);
        }
    }

    // Drop values equal to their predecessor from the sorted list (after a
    // merge, copies of one value are adjacent) and close the gaps: the kept
    // values move down through the warp's shared scratch `wsm` (32 * R
    // slots), kNone fills the tail.
    __device__ __forceinline__ void dedup_sorted(int lane, uint64_t* wsm) {
        const uint64_t prev_last = __shfl_up_sync(kFull, a[R - 1], 1);
        uint32_t dmask = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint64_t p = r == 0 ? prev_last : a[r - 1];
            if (a[r] != kNone && (r > 0 || lane > 0) && a[r] == p) dmask |= 1u << r;
        }
        if (!__any_sync(kFull, dmask != 0)) return;
        const uint32_t cnt = __popc(dmask);
        uint32_t incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += t;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        uint32_t removed = incl - cnt;
        constexpr uint32_t N = 32 * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t idx = uint32_t(lane) * R + r;
            if ((dmask >> r) & 1u) {
                ++removed;
            } else {
                HCG_DASSERT(idx >= removed && idx - removed < N);
                wsm[idx - removed] = a[r];
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t idx = uint32_t(lane) * R + r;
            if (idx >= N - total) wsm[idx] = kNone;
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = wsm[uint32_t(lane) * R + r];
        __syncwarp();
    }

    // offer() for candidate streams that may repeat a value (the same row
    // reached through two curves) and for long lists: offers that may beat the
    // threshold are appended to the warp's shared queue wq (qcap <= 32 slots,
    // qn entries, warp-uniform) and a full queue is sorted, merged and
    // deduplicated in one go, so a pass with a few passing offers costs a
    // ballot and a store instead of a merge or one insertion each.  Offers
    // carry the physical row in the low word; the queue translates it through
    // idtab (row -> id) when it flushes, one load latency per flush instead of
    // one per pass, so the filter compares distances only (ties pass and the
    // merge sorts them out).  A merge of qcap values pushes out at most qcap
    // repeats: exact while 32 * R - qcap >= k.  The threshold only falls, so
    // nothing the queue holds is lost; flush_queue() after the last offer.
    __device__ __forceinline__ void offer_queued(uint64_t cand, int lane, uint64_t* wsm, uint64_t* wq, uint32_t& qn,
                                                 uint32_t qcap, const uint32_t* idtab) {
        const bool pass = cand != kNone && uint32_t(cand >> 32) <= uint32_t(thr >> 32);
        unsigned m = __ballot_sync(kFull, pass);
        while (m) {
            const uint32_t take = min(uint32_t(__popc(m)), qcap - qn);
            const bool mine = (m >> lane) & 1u;
            const uint32_t rank = __popc(m & ((1u << lane) - 1u));
            const bool store = mine && rank < take;
            if (store) wq[qn + rank] = cand;
            m &= ~__ballot_sync(kFull, store);
            qn += take;
            if (qn == qcap) {
                flush_queue(lane, wsm, wq, qn, idtab);
                m &= __ballot_sync(kFull, uint32_t(cand >> 32) <= uint32_t(thr >> 32));
            }
        }
    }

    __device__ __forceinline__ void flush_queue(int lane, uint64_t* wsm, const uint64_t* wq, uint32_t& qn,
                                                const uint32_t* idtab) {
        if (qn == 0) return;
        __syncwarp();
        uint64_t c = kNone;
        if (uint32_t(lane) < qn) {
            c = wq[lane];
            if (idtab) c = (c & 0xFFFFFFFF00000000ull) | __ldg(idtab + uint32_t(c));
        }
        merge_sorted32<R>(a, warp_sort_asc(c, lane), lane);
        dedup_sorted(lane, wsm);
        update_thr();
        __syncwarp();  // every lane read its entry before the queue refills
        qn = 0;
    }
};

// Warp top-k over (u64 key, u32 slot) pairs for f32 indexes: key = the bits of
// the non-negative double squared distance (order preserving), ties by slot
// (= id order).  Same blocked layout and insertion as WarpTopK.
template <int R>
struct WarpTopK2 {
    uint64_t a[R];
    uint32_t b[R];
    uint64_t ta;
    uint32_t tb;
    int thr_lane, thr_reg;

    __device__ static __forceinline__ bool lt(uint64_t xa, uint32_t xb, uint64_t ya, uint32_t yb) {
        return xa < ya || (xa == ya && xb < yb);
    }

    __device__ __forceinline__ void init(int k) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            a[r] = kNone;
            b[r] = 0xFFFFFFFFu;
        }
        ta = kNone;
        tb = 0xFFFFFFFFu;
        thr_lane = (k - 1) / R;
        thr_reg = (k - 1) % R;
    }

    __device__ __forceinline__ void insert(uint64_t xa, uint32_t xb, int lane) {
        const uint64_t pa = __shfl_up_sync(kFull, a[R - 1], 1);
        const uint32_t pb = __shfl_up_sync(kFull, b[R - 1], 1);
        const bool first_lt = lane == 0 || lt(pa, pb, xa, xb);
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
            const uint64_t qa = r == 0 ? pa : a[r - 1];
            const uint32_t qb = r == 0 ? pb : b[r - 1];
            const bool q_lt = r == 0 ? first_lt : lt(a[r - 1], b[r - 1], xa, xb);
            if (!q_lt) {
                a[r] = qa;
                b[r] = qb;
            } else if (lt(xa, xb, a[r], b[r])) {
                a[r] = xa;
                b[r] = xb;
            }
        }
        uint64_t ma = 0;
        uint32_t mb = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ma |= a[r] & (0ull - uint64_t(r == thr_reg));
            mb |= b[r] & (0u - uint32_t(r == thr_reg));
        }
        ta = __shfl_sync(kFull, ma, thr_lane);
        tb = __shfl_sync(kFull, mb, thr_lane);
    }

    __device__ __forceinline__ void offer(uint64_t ca, uint32_t cb, int lane) {
        unsigned m = __ballot_sync(kFull, lt(ca, cb, ta, tb));
        while (m) {
            const int src = __ffs(m) - 1;
            const uint64_t xa = __shfl_sync(kFull, ca, src);
            const uint32_t xb = __shfl_sync(kFull, cb, src);
            insert(xa, xb, lane);
            m &= ~(1u << src);
            m &= __ballot_sync(kFull, lt(ca, cb, ta, tb));
        }
    }
};

__device__ __forceinline__ uint32_t hash_slot(uint32_t s) { return s * 2654435761u; }

}  // namespace hcg
