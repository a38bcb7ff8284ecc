// gather_bench.cu -- what can a B200 do on the refine kernel's access pattern:
// random 128-byte descriptor rows out of a >L2 array (1.28 GB), summed so the
// loads cannot be elided.  Variants:
//   ldg<U>   : 8 lanes per row, U rows in flight per lane (LDG.128 into registers)
//   cpasync  : LDGSTS (cp.async.cg 16 B) into a per-warp shared ring
//   bulk     : cp.async.bulk (TMA engine, 128 B per row) into a per-warp ring,
//              completion on an mbarrier per stage
//   gather4  : cp.async.bulk.tensor.2d.tile::gather4 (TMA, 4 rows of a 2-D
//              tensor map per instruction) into a per-warp ring
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const uint8_t* __restrict__ rows, const uint32_t* __restrict__ idx,
                                             uint64_t nidx, uint32_t* out) {
    const int lane = threadIdx.x & 31, l8 = lane & 7, grp = lane >> 3;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    const uint64_t w = uint64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    uint32_t acc = 0;
    for (uint64_t base = w * 4 * U; base < nidx; base += warps * 4 * U) {
        uint32_t s[U];
#pragma unroll
        for (int r = 0; r < U; ++r) s[r] = __ldg(idx + base + grp * U + r);
        uint4 v[U];
#pragma unroll
        for (int r = 0; r < U; ++r) v[r] = ldg_stream(rows + uint64_t(s[r]) * 128 + l8 * 16);
#pragma unroll
        for (int r = 0; r < U; ++r) acc += v[r].x ^ v[r].y ^ v[r].z ^ v[r].w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// LDGSTS ring: per warp S stages of 32 rows (4 KB each).
template <int S>
__global__ void __launch_bounds__(128) k_cpasync(const uint8_t* __restrict__ rows, const uint32_t* __restrict__ idx,
                                                 uint64_t nidx, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    uint8_t* ring = sm + wl * S * 4096;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    const uint64_t w = uint64_t(blockIdx.x) * (blockDim.x / 32) + wl;
    uint32_t acc = 0;
    const uint64_t nb = nidx / 32;
    uint64_t b_issue = w, b_use = w;
    int issued = 0;
    auto issue = [&](uint64_t b, int stage) {
        // 32 rows x 8 chunks = 256 16-B copies; 8 per lane
        const uint32_t my = __ldg(idx + b * 32 + lane);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            // lane handles chunk c of all rows via shuffles: row r = (lane + 32*c)/8
            const int e = lane + 32 * c, r = e >> 3, ch = e & 7;
            const uint32_t sr = __shfl_sync(0xffffffff, my, r);
            const uint8_t* src = rows + uint64_t(sr) * 128 + ch * 16;
            uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + stage * 4096 + r * 128 + ch * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src));
        }
        asm volatile("cp.async.commit_group;");
    };
    for (int st = 0; st < S; ++st) {
        if (b_issue < nb) issue(b_issue, st);
        else asm volatile("cp.async.commit_group;");
        b_issue += warps;
    }
    int stage = 0;
    for (; b_use < nb; b_use += warps) {
        asm volatile("cp.async.wait_group %0;" :: "n"(S - 1));
        __syncwarp();
        const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + stage * 4096);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += p[i * 32 + lane];
        __syncwarp();
        if (b_issue < nb) issue(b_issue, stage);
        else asm volatile("cp.async.commit_group;");
        b_issue += warps;
        stage = (stage + 1) % S;
        ++issued;
    }
    asm volatile("cp.async.wait_all;");
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// cp.async.bulk (TMA engine) ring: per warp S stages of 32 rows, one mbarrier per stage.
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase));
}

template <int S>
__global__ void __launch_bounds__(128) k_bulk(const uint8_t* __restrict__ rows, const uint32_t* __restrict__ idx,
                                              uint64_t nidx, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    uint8_t* ring = sm + wl * S * 4096;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (blockDim.x / 32) * S * 4096) + wl * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    const uint64_t w = uint64_t(blockIdx.x) * (blockDim.x / 32) + wl;
    const uint64_t nb = nidx / 32;
    uint32_t acc = 0;
    auto issue = [&](uint64_t b, int stage) {
        const uint32_t my = __ldg(idx + b * 32 + lane);
        if (lane == 0) mbar_expect(&bars[stage], 32 * 128);
        __syncwarp();
        const uint8_t* src = rows + uint64_t(my) * 128;
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + stage * 4096 + lane * 128);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                     :: "r"(dst), "l"(src), "r"((uint32_t)__cvta_generic_to_shared(&bars[stage])) : "memory");
    };
    uint64_t b_issue = w;
    for (int s = 0; s < S && b_issue < nb; ++s, b_issue += warps) issue(b_issue, s);
    int stage = 0;
    uint32_t phase = 0;
    for (uint64_t b = w; b < nb; b += warps) {
        mbar_wait(&bars[stage], phase);
        const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + stage * 4096);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += p[i * 32 + lane];
        __syncwarp();
        if (b_issue < nb) {
            issue(b_issue, stage);
            b_issue += warps;
        }
        if (++stage == S) {
            stage = 0;
            phase ^= 1;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// tile::gather4: per warp S stages of 32 rows; lanes 0..7 each issue one
// gather4 (4 rows x 128 B) per stage, one mbarrier per stage.
template <int S>
__global__ void __launch_bounds__(128) k_gather4(const __grid_constant__ CUtensorMap map, const uint32_t* __restrict__ idx,
                                                 uint64_t nidx, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    uint8_t* ring = sm + wl * S * 4096;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (blockDim.x / 32) * S * 4096) + wl * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncwarp();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x / 32);
    const uint64_t w = uint64_t(blockIdx.x) * (blockDim.x / 32) + wl;
    const uint64_t nb = nidx / 32;
    uint32_t acc = 0;
    auto issue = [&](uint64_t b, int stage) {
        const uint32_t my = __ldg(idx + b * 32 + lane);
        if (lane == 0) mbar_expect(&bars[stage], 32 * 128);
        __syncwarp();
        const int r0 = __shfl_sync(0xffffffff, my, (lane * 4) & 31), r1 = __shfl_sync(0xffffffff, my, (lane * 4 + 1) & 31),
                  r2 = __shfl_sync(0xffffffff, my, (lane * 4 + 2) & 31), r3 = __shfl_sync(0xffffffff, my, (lane * 4 + 3) & 31);
        if (lane < 8) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + stage * 4096 + lane * 512);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"((uint32_t)__cvta_generic_to_shared(&bars[stage])), "r"(0),
                "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    };
    uint64_t b_issue = w;
    for (int s = 0; s < S && b_issue < nb; ++s, b_issue += warps) issue(b_issue, s);
    int stage = 0;
    uint32_t phase = 0;
    for (uint64_t b = w; b < nb; b += warps) {
        mbar_wait(&bars[stage], phase);
        const uint32_t* p = reinterpret_cast<const uint32_t*>(ring + stage * 4096);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += p[i * 32 + lane];
        __syncwarp();
        if (b_issue < nb) {
            issue(b_issue, stage);
            b_issue += warps;
        }
        if (++stage == S) {
            stage = 0;
            phase ^= 1;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint64_t n = 10000000, nidx = 256ull << 20;  // 268M rows = 34 GB gathered
    uint8_t* rows;
    uint32_t *idx, *out;
    CK(cudaMalloc(&rows, n * 128));
    CK(cudaMemset(rows, 7, n * 128));
    CK(cudaMalloc(&idx, nidx * 4));
    CK(cudaMalloc(&out, 148 * 64 * 256 * 4));
    std::vector<uint32_t> h(nidx);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        v = uint32_t(x % n);
    }
    CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double bytes = double(nidx) * 128;
    auto report = [&](const char* name, float ms) {
        printf("%-28s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
    };
#define RUN(name, launch)                                   \
    do {                                                    \
        launch; CK(cudaDeviceSynchronize());                \
        float best = 1e30f;                                 \
        for (int it = 0; it < 3; ++it) {                    \
            cudaEventRecord(a); launch; cudaEventRecord(b); \
            CK(cudaEventSynchronize(b));                    \
            float ms; cudaEventElapsedTime(&ms, a, b);      \
            best = ms < best ? ms : best;                   \
        }                                                   \
        report(name, best);                                 \
    } while (0)
    for (int bps : {4, 6, 8}) {
        char nm[64];
        snprintf(nm, 64, "ldg<4>  %d blk/SM", bps);
        RUN(nm, (k_ldg<4><<<148 * bps, 256>>>(rows, idx, nidx, out)));
        snprintf(nm, 64, "ldg<8>  %d blk/SM", bps);
        RUN(nm, (k_ldg<8><<<148 * bps, 256>>>(rows, idx, nidx, out)));
        snprintf(nm, 64, "ldg<16> %d blk/SM", bps);
        RUN(nm, (k_ldg<16><<<148 * bps, 256>>>(rows, idx, nidx, out)));
    }
    for (int S : {2, 4}) {
        const int smem = 4 * S * 4096;
        if (S == 2) { CK(cudaFuncSetAttribute(k_cpasync<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
        if (S == 4) { CK(cudaFuncSetAttribute(k_cpasync<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
        for (int bps : {2, 4, 8}) {
            if (bps * smem > 220 * 1024) continue;
            char nm[64];
            snprintf(nm, 64, "cpasync S=%d %d blk/SM", S, bps);
            if (S == 2) RUN(nm, (k_cpasync<2><<<148 * bps, 128, smem>>>(rows, idx, nidx, out)));
            else RUN(nm, (k_cpasync<4><<<148 * bps, 128, smem>>>(rows, idx, nidx, out)));
        }
    }
    for (int S : {4, 8}) {
        const int smem = 4 * S * 4096 + 4 * S * 8;
        if (S == 4) { CK(cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
        if (S == 8) { CK(cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
        for (int bps : {1, 2, 3}) {
            if (bps * smem > 220 * 1024) continue;
            char nm[64];
            snprintf(nm, 64, "bulk S=%d %d blk/SM", S, bps);
            if (S == 4) RUN(nm, (k_bulk<4><<<148 * bps, 128, smem>>>(rows, idx, nidx, out)));
            else RUN(nm, (k_bulk<8><<<148 * bps, 128, smem>>>(rows, idx, nidx, out)));
        }
    }
    {
        void* fp = nullptr;
        cudaDriverEntryPointQueryResult qr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr));
        CUtensorMap map;
        const cuuint64_t dims[2] = {128, n};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {128, 1};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = reinterpret_cast<EncodeFn>(fp)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, rows, dims, strides, box, estr,
                                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) printf("tensor map encode failed: %d\n", int(r));
        for (int S : {4, 8}) {
            const int smem = 4 * S * 4096 + 4 * S * 8;
            if (S == 4) { CK(cudaFuncSetAttribute(k_gather4<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
            if (S == 8) { CK(cudaFuncSetAttribute(k_gather4<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); }
            for (int bps : {1, 2, 3}) {
                if (bps * smem > 220 * 1024) continue;
                char nm[64];
                snprintf(nm, 64, "gather4 S=%d %d blk/SM", S, bps);
                if (S == 4) RUN(nm, (k_gather4<4><<<148 * bps, 128, smem>>>(map, idx, nidx, out)));
                else RUN(nm, (k_gather4<8><<<148 * bps, 128, smem>>>(map, idx, nidx, out)));
            }
        }
    }
    // sequential copy for reference
    uint8_t* dst;
    CK(cudaMalloc(&dst, n * 128));
    bytes = 2.0 * n * 128;
    RUN("memcpy D2D (read+write)", (cudaMemcpyAsync(dst, rows, n * 128 * 1, cudaMemcpyDeviceToDevice)));
    return 0;
}
