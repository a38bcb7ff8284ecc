// brute_tc.cu -- K5 on the 5th-generation tensor cores: exact kNN ground truth
// (brute_force_knn, proj/src/vecio.cpp:115-122) for uint8 rows of 128 bytes.
//
// The exact squared distance of uint8 vectors is
//     S(q, x) = |q|^2 + |x|^2 - 2 q.x
// and q.x <= 128 * 255^2 < 2^31, so an unsigned-8-bit tensor-core product
// with 32-bit integer accumulation (tcgen05.mma kind::i8) gives S exactly; no
// re-centring is needed because the UMMA instruction takes unsigned operands.
//
// One CTA per (tile of 128 queries, chunk of rows); warp roles:
//   warp 0     TMA producer: the 128 x 128 B query tile once, then row tiles
//              of 256 x 128 B into a 4-stage ring (SWIZZLE_128B, K-major)
//   warp 1     TMEM owner (512 columns = two 128 x 256 s32 accumulators) and
//              MMA issuer: 4 x tcgen05.mma (K = 32 B each) per row tile
//   warps 4-11 epilogue: tcgen05.ld of the accumulator (lane = query,
//              column = row), S = |q|^2 + |x|^2 - 2 q.x, a per-thread sorted
//              top-KT of packed (S << 32 | slot) -- the reference's (distance,
//              id) order; warp quad e (warps 4+4e .. 7+4e) takes columns
//              [128e, 128e + 128) of every tile
// Two accumulators let the epilogue of tile t overlap the MMAs of tile t+1.
// Per-(query, chunk, column group) lists go through K4 (k_merge), as for the
// CUDA-core K5.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "hcg_host.hpp"
#include "hcg_internal.cuh"

namespace hcg {

namespace {
constexpr int kBM = 128;          // queries per tile (UMMA M)
constexpr int kBN = 256;          // rows per tile (UMMA N)
constexpr int kRowBytes = 128;    // K: one SWIZZLE_128B atom per row
constexpr int kStages = 4;
constexpr int kEpiGroups = 2;     // epilogue warp quads; quad e scores columns [e*128, e*128+128) of a tile (4 quads: 1.2x slower)
constexpr int kEpiCols = kBN / kEpiGroups;
constexpr int kThreads = 128 + 128 * kEpiGroups;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kATileBytes = kBM * kRowBytes;  // 16 KB
constexpr uint32_t kBTileBytes = kBN * kRowBytes;  // 32 KB
constexpr int kEpiThreads = 128 * kEpiGroups;  // warps 4 ..
// + per-epilogue-thread spill of 32 distances for the rare insertion path
// + the distance spill + a double buffer of row norms (one tile each)
constexpr int kNormRing = 8;      // row-norm tiles in flight (prefetched kNormAhead tiles ahead)
constexpr int kNormAhead = 6;
constexpr size_t kSmemBytes = 1024 + kATileBytes + size_t(kStages) * kBTileBytes + 256 + 32 * kEpiThreads * 4 +
                              size_t(kNormRing) * kBN * 4;

// ---- PTX helpers (tcgen05 / TMA / mbarrier) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, unsigned 8-bit operands, s32 accumulators.
__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B (8-row groups of
// 128-B rows, 1024 B apart), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);       // start address
    d |= uint64_t(1) << 16;                      // leading byte offset (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;              // stride byte offset: next 8-row group
    d |= uint64_t(1) << 46;                      // version (sm_100)
    d |= uint64_t(2) << 61;                      // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor: kind::i8, u8 x u8 -> s32, both K-major, M x N.
constexpr uint32_t idesc_u8(int M, int N) {
    return (2u << 4)                 // D format: s32
           | (0u << 7) | (0u << 10)  // A, B: unsigned 8-bit
           | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int KT>
__device__ __forceinline__ void topk_insert(uint64_t (&a)[KT], uint64_t v) {
#pragma unroll
    for (int i = KT - 1; i > 0; --i) a[i] = v < a[i - 1] ? a[i - 1] : (v < a[i] ? v : a[i]);
    a[0] = v < a[0] ? v : a[0];
}

// |row|^2 of every row (u32, exact), zero past n up to the padded length.
__global__ void k_row_norms(const uint8_t* __restrict__ rows, uint64_t n, uint64_t n_pad, uint32_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    uint32_t s = 0;
    if (i < n) {
        const uint4* r = reinterpret_cast<const uint4*>(rows + i * kRowBytes);
#pragma unroll
        for (int c = 0; c < kRowBytes / 16; ++c) {
            const uint4 v = __ldg(r + c);
            s = __dp4a(v.x, v.x, s);
            s = __dp4a(v.y, v.y, s);
            s = __dp4a(v.z, v.z, s);
            s = __dp4a(v.w, v.w, s);
        }
    }
    out[i] = s;
}

template <int KT>
__global__ void __launch_bounds__(kThreads, 1)
    k_brute_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_x,
               const uint8_t* __restrict__ queries, const uint32_t* __restrict__ xnorm, uint32_t nq, uint64_t n,
               uint32_t k, uint32_t chunks, uint32_t tiles_per_chunk, uint64_t* __restrict__ part,
               const uint32_t* __restrict__ idtab) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B alignment for SWIZZLE_128B tiles (pointer arithmetic on the shared
    // array keeps the address space visible to the compiler: LDS, not LD)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* sa = smem;
    unsigned char* sb = smem + kATileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sb + size_t(kStages) * kBTileBytes);
    uint64_t* full = bars;                  // [kStages]
    uint64_t* empty = bars + kStages;       // [kStages]
    uint64_t* a_full = bars + 2 * kStages;  // [1]
    uint64_t* acc_full = a_full + 1;        // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    uint32_t* spill = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(bars) + 256);  // [32][kEpiThreads]
    uint32_t* nbuf = spill + 32 * kEpiThreads;                                                      // [kNormRing][kBN]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qt = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
    const uint64_t n_tiles = (n + kBN - 1) / kBN;
    const uint64_t t_begin = uint64_t(chunk) * tiles_per_chunk;
    const uint64_t t_end = std::min<uint64_t>(n_tiles, t_begin + tiles_per_chunk);
    const int n_local = t_end > t_begin ? int(t_end - t_begin) : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(a_full, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4 * kEpiGroups);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            mbar_expect_tx(a_full, kATileBytes);
            tma_load_2d(sa, &map_q, a_full, 0, int(qt * kBM));
            for (int t = 0; t < n_local; ++t) {
                const int s = t % kStages;
                mbar_wait(&empty[s], ((t / kStages) & 1) ^ 1);
                mbar_expect_tx(&full[s], kBTileBytes);
                tma_load_2d(sb + size_t(s) * kBTileBytes, &map_x, &full[s], 0, int((t_begin + t) * kBN));
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_u8(kBM, kBN);
            mbar_wait(a_full, 0);
            const uint32_t a0 = smem_u32(sa);
            for (int t = 0; t < n_local; ++t) {
                const int s = t % kStages, b = t & 1;
                mbar_wait(&acc_empty[b], ((t >> 1) & 1) ^ 1);
                mbar_wait(&full[s], (t / kStages) & 1);
                tc_fence_after();
                const uint32_t b0 = smem_u32(sb + size_t(s) * kBTileBytes);
#pragma unroll
                for (int ks = 0; ks < kRowBytes / 32; ++ks)
                    mma_u8(tmem + uint32_t(b) * kBN, smem_desc_sw128(a0 + ks * 32), smem_desc_sw128(b0 + ks * 32), idesc,
                           ks > 0 ? 1u : 0u);
                tc_commit(&empty[s]);     // smem stage free once these MMAs have read it
                tc_commit(&acc_full[b]);  // accumulator b complete
            }
        }
    } else if (warp >= 4) {  // ---- epilogue
        const int ew = warp - 4, g = warp & 3, half = ew >> 2;  // half: the column group
        const uint32_t q = qt * kBM + uint32_t(g * 32 + lane);
        const bool q_ok = q < nq;
        uint32_t qn = 0;
        if (q_ok) {
            const uint4* r = reinterpret_cast<const uint4*>(queries + uint64_t(q) * kRowBytes);
#pragma unroll
            for (int c = 0; c < kRowBytes / 16; ++c) {
                const uint4 v = __ldg(r + c);
                qn = __dp4a(v.x, v.x, qn);
                qn = __dp4a(v.y, v.y, qn);
                qn = __dp4a(v.z, v.z, qn);
                qn = __dp4a(v.w, v.w, qn);
            }
        }
        uint64_t top[KT];
#pragma unroll
        for (int i = 0; i < KT; ++i) top[i] = kNone;
        // Row norms: the epilogue streams each tile's 256 norms (cp.async,
        // 64 x 16 B) into a shared ring kNormAhead tiles ahead of scoring;
        // one commit group per tile (empty past the end) keeps the counts
        // uniform for cp.async.wait_group.
        const int et = threadIdx.x - 128;
        auto fetch_norms = [&](int t) {
            if (t < n_local && et < kBN / 4)
                cp_async16(nbuf + (t % kNormRing) * kBN + et * 4, xnorm + (t_begin + t) * kBN + et * 4);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        for (int i = 0; i < kNormAhead; ++i) fetch_norms(i);
        asm volatile("cp.async.wait_group %0;" ::"n"(kNormAhead - 1) : "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        for (int t = 0; t < n_local; ++t) {
            const int b = t & 1;
            fetch_norms(t + kNormAhead);  // its buffer last served tile t + kNormAhead - kNormRing < t
            mbar_wait(&acc_full[b], (t >> 1) & 1);
            tc_fence_after();
            const uint32_t* tn = nbuf + (t % kNormRing) * kBN + half * kEpiCols;
            const uint64_t row0 = (t_begin + t) * kBN + uint64_t(half) * kEpiCols;
#pragma unroll 1
            for (int c0 = 0; c0 < kEpiCols; c0 += 32) {
                uint32_t dot[32];
                tmem_ld32(tmem + (uint32_t(g * 32) << 16) + uint32_t(b) * kBN + uint32_t(half) * kEpiCols + c0, dot);
                // Fast path (almost every column): S and one compare against
                // the current k-th distance, no branches in the unrolled body.
                const uint4* xn4 = reinterpret_cast<const uint4*>(tn + c0);
                // t = |x|^2 - 2 q.x (S = |q|^2 + t, all < 2^31): one IMAD and
                // one IMNMX per column; the minimum decides the slow path.
                const uint32_t thr = uint32_t(top[KT - 1] >> 32);
                const int32_t thr_t = thr == 0xFFFFFFFFu ? INT32_MAX : int32_t(thr) - int32_t(qn);
                int32_t m8[8];  // independent partial minima: no 32-long dependency chain
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                    const uint4 xv = xn4[j4];
                    const int32_t t0 = int32_t(xv.x) - 2 * int32_t(dot[j4 * 4 + 0]);
                    const int32_t t1 = int32_t(xv.y) - 2 * int32_t(dot[j4 * 4 + 1]);
                    const int32_t t2 = int32_t(xv.z) - 2 * int32_t(dot[j4 * 4 + 2]);
                    const int32_t t3 = int32_t(xv.w) - 2 * int32_t(dot[j4 * 4 + 3]);
                    dot[j4 * 4 + 0] = uint32_t(t0);
                    dot[j4 * 4 + 1] = uint32_t(t1);
                    dot[j4 * 4 + 2] = uint32_t(t2);
                    dot[j4 * 4 + 3] = uint32_t(t3);
                    m8[j4] = min(min(t0, t1), min(t2, t3));
                }
                const int32_t tmin = min(min(min(m8[0], m8[1]), min(m8[2], m8[3])),
                                         min(min(m8[4], m8[5]), min(m8[6], m8[7])));
                const uint64_t base = row0 + c0;  // columns past n are TMA zero fill
                if (tmin <= thr_t && base < n) {
                    // slow path (a lane's chunk holds a new top-KT candidate; the
                    // warp runs it when any lane does, ~40 % of chunks at k=10):
                    // spill, then visit only the passing columns
                    uint32_t pass = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        spill[j * kEpiThreads + et] = dot[j];
                        pass |= uint32_t(int32_t(dot[j]) <= thr_t) << j;
                    }
                    if (n - base < 32) pass &= (1u << (n - base)) - 1u;
#pragma unroll 1
                    for (; pass; pass &= pass - 1) {
                        const int j = __ffs(pass) - 1;
                        const uint64_t v = (uint64_t(qn + spill[j * kEpiThreads + et]) << 32) |
                                           (idtab ? __ldg(idtab + base + j) : uint32_t(base + j));
                        if (v < top[KT - 1]) topk_insert<KT>(top, v);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
            asm volatile("cp.async.wait_group %0;" ::"n"(kNormAhead - 1) : "memory");
            asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");  // norms of t+1 visible to all epilogue threads
        }
        if (q_ok) {
            const uint64_t p = uint64_t(chunk) * kEpiGroups + uint64_t(half);
            uint64_t* dst = part + (p * nq + q) * k;
#pragma unroll
            for (int i = 0; i < KT; ++i)
                if (uint32_t(i) < k) dst[i] = top[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// Ids: part holds (S << 32 | slot); k_merge wants (S << 32 | id).
__global__ void k_slots_to_ids(uint64_t* part, uint64_t count, uint64_t id_base, uint64_t id_stride) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t v = part[i];
    if (v != kNone) part[i] = (v & 0xFFFFFFFF00000000ull) | (id_base + (v & 0xFFFFFFFFull) * id_stride);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cuuint64_t(kRowBytes), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(kRowBytes)};
    const cuuint32_t box[2] = {cuuint32_t(kRowBytes), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TcPlan {
    uint32_t qtiles, chunks, tiles_per_chunk;
    uint64_t n_pad;
};

TcPlan plan(const BruteArgs& a, int sms) {
    TcPlan p;
    p.qtiles = (a.nq + kBM - 1) / kBM;
    const uint64_t n_tiles = (a.n + kBN - 1) / kBN;
    p.chunks = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(n_tiles, uint64_t(std::max(1, sms)) / p.qtiles)));
    p.tiles_per_chunk = uint32_t((n_tiles + p.chunks - 1) / p.chunks);
    p.chunks = uint32_t((n_tiles + p.tiles_per_chunk - 1) / p.tiles_per_chunk);
    p.n_pad = n_tiles * kBN;
    return p;
}

int device_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

template <int KT>
hcg_status launch_tc(const BruteArgs& a, const TcPlan& p, const CUtensorMap& mq, const CUtensorMap& mx,
                     const uint32_t* xn, uint64_t* part, cudaStream_t st) {
    static bool cfg[64] = {};  // the opt-in is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !cfg[dev]) {
        if (cudaFuncSetAttribute(k_brute_tc<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes)) !=
            cudaSuccess)
            return set_error(HCG_ECUDA, "brute_tc: shared memory opt-in failed");
        if (dev < 64) cfg[dev] = true;
    }
    k_brute_tc<KT><<<p.qtiles * p.chunks, kThreads, kSmemBytes, st>>>(mq, mx, a.queries, xn, a.nq, a.n, a.k, p.chunks,
                                                                       p.tiles_per_chunk, part, a.idtab);
    return check_launch("k_brute_tc");
}
}  // namespace

bool brute_tc_eligible(const BruteArgs& a) {
    static const bool off = knob("HCG_BRUTE_CUDA_CORES") != nullptr;
    return !off && a.dtype == HCG_U8 && a.pitch == uint32_t(kRowBytes) && a.k <= 32 && a.n > 0 && a.nq > 0 &&
           a.n < (uint64_t(1) << 31) &&
           encode_fn() != nullptr;
}

size_t brute_tc_scratch_bytes(const BruteArgs& a) {
    const TcPlan p = plan(a, device_sms());
    return (((size_t(p.chunks) * kEpiGroups * a.nq * a.k) + 31) & ~size_t(31)) * 8 + size_t(p.n_pad) * 4 + 256;
}

hcg_status launch_brute_tc(const BruteArgs& a, void* scratch, uint64_t* out_ids, uint32_t* out_sqdist,
                           uint32_t* out_len, cudaStream_t st) {
    const TcPlan p = plan(a, device_sms());
    uint64_t* part = static_cast<uint64_t*>(scratch);
    const size_t part_n = size_t(p.chunks) * kEpiGroups * a.nq * a.k;
    uint32_t* xn = reinterpret_cast<uint32_t*>(part + ((part_n + 31) & ~size_t(31)));  // 256-B aligned
    CUtensorMap mq, mx;
    if (!make_map(&mq, a.queries, a.nq, kBM) || !make_map(&mx, a.rows, a.n, kBN))
        return set_error(HCG_ECUDA, "brute_tc: tensor map encoding failed");
    k_row_norms<<<unsigned((p.n_pad + 255) / 256), 256, 0, st>>>(a.rows, a.n, p.n_pad, xn);
    HCG_RET_IF(check_launch("k_row_norms"));
    hcg_status rc;
    if (a.k <= 8)
        rc = launch_tc<8>(a, p, mq, mx, xn, part, st);
    else if (a.k <= 16)
        rc = launch_tc<16>(a, p, mq, mx, xn, part, st);
    else
        rc = launch_tc<32>(a, p, mq, mx, xn, part, st);
    if (rc != HCG_OK) return rc;
    k_slots_to_ids<<<unsigned((part_n + 255) / 256), 256, 0, st>>>(part, part_n, a.id_base, a.id_stride);
    HCG_RET_IF(check_launch("k_slots_to_ids"));
    return launch_merge(part, p.chunks * kEpiGroups, a.nq, a.k, out_ids, out_sqdist, out_len, st);
}

}  // namespace hcg
