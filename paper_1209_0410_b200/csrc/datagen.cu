// datagen.cu -- the counter-based synthetic SIFT-like generator of SURVEY.md
// §8(d), on the device.  Integer-only, so every row is bit-identical to the
// CPU oracle's (oracle/hc_oracle.cpp gen_row) and any row can be regenerated
// independently -- a shard generates exactly its own `id mod G` rows.
#include "hcg_internal.cuh"
#include "hcg_host.hpp"

namespace hcg {

namespace {
constexpr int kNC = 4096, kD = 128, kR = 12;

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t H(uint64_t s, uint64_t a, uint64_t b) {
    return sm64(s ^ sm64(a * 0x100000001b3ull ^ sm64(b)));
}
}  // namespace

__global__ void k_gen_tables(uint8_t* __restrict__ center, int8_t* __restrict__ wt) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < uint64_t(kNC) * kD * kR) wt[t] = int8_t(int(H(6, t, 0) % 7) - 3);
    if (t < uint64_t(kNC) * kD) {
        const uint64_t c = t / kD, j = t % kD;
        const uint64_t h = H(1, c, j);
        center[t] = uint8_t(((h & 255) * ((h >> 8) & 255) * ((h >> 16) & 255)) >> 16);
    }
}

// Row i of the database, 16 bytes at a time into `out` (128 bytes).
__device__ void gen_row(const uint8_t* __restrict__ center, const int8_t* __restrict__ wt, uint64_t i,
                        uint8_t* __restrict__ out, const uint8_t* __restrict__ noise_q, bool as_query,
                        uint64_t qid) {
    const uint64_t cl = H(2, i, ~0ull) % kNC;
    int z[kR];
#pragma unroll
    for (int l = 0; l < kR; ++l) {
        const uint64_t h = H(7, i, l);
        z[l] = int(h & 15) + int((h >> 4) & 15) + int((h >> 8) & 15) + int((h >> 12) & 15) - 30;
    }
    (void)noise_q;
    for (int j0 = 0; j0 < kD; j0 += 16) {
        uint32_t packed[4] = {0, 0, 0, 0};
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const int j = j0 + jj;
            const int8_t* w = wt + (cl * kD + j) * kR;
            int acc = 0;
#pragma unroll
            for (int l = 0; l < kR; ++l) acc += int(__ldg(w + l)) * z[l];
            const uint64_t h = H(3, i, j);
            const int noise = int(h & 3) + int((h >> 2) & 3) - 3;
            int v = int(__ldg(center + cl * kD + j)) + (acc >> 3) + noise;
            v = v < 0 ? 0 : (v > 255 ? 255 : v);
            if (as_query) {
                const uint64_t hq = H(5, qid, j);
                v = v + int(hq & 15) + int((hq >> 4) & 15) - 15;
                v = v < 0 ? 0 : (v > 255 ? 255 : v);
            }
            packed[jj >> 2] |= uint32_t(v) << (8 * (jj & 3));
        }
        *reinterpret_cast<uint4*>(out + j0) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
}

__global__ void k_gen_rows(const uint8_t* __restrict__ center, const int8_t* __restrict__ wt, uint64_t first,
                           uint64_t stride, uint64_t count, uint8_t* __restrict__ out) {
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    gen_row(center, wt, first + r * stride, out + r * kD, nullptr, false, 0);
}

// Query q perturbs database row H(4, q, ~0) % n_db.
__global__ void k_gen_queries(const uint8_t* __restrict__ center, const int8_t* __restrict__ wt, uint64_t first,
                              uint64_t count, uint64_t n_db, uint8_t* __restrict__ out) {
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    const uint64_t q = first + r;
    gen_row(center, wt, H(4, q, ~0ull) % n_db, out + r * kD, nullptr, true, q);
}

namespace {
struct Tables {
    uint8_t* center = nullptr;
    int8_t* wt = nullptr;
};

hcg_status make_tables(Tables& t, cudaStream_t st) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&t.center), size_t(kNC) * kD, st) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&t.wt), size_t(kNC) * kD * kR, st) != cudaSuccess)
        return set_error(HCG_ENOMEM, "generator tables");
    const uint64_t total = uint64_t(kNC) * kD * kR;
    k_gen_tables<<<unsigned((total + 255) / 256), 256, 0, st>>>(t.center, t.wt);
    return check_launch("k_gen_tables");
}
void free_tables(Tables& t, cudaStream_t st) {
    if (t.center) cudaFreeAsync(t.center, st);
    if (t.wt) cudaFreeAsync(t.wt, st);
}
}  // namespace

hcg_status gen_rows(uint64_t first, uint64_t stride, uint64_t count, uint8_t* out, cudaStream_t st) {
    if (count == 0) return HCG_OK;
    Tables t;
    hcg_status rc = make_tables(t, st);
    if (rc == HCG_OK) {
        k_gen_rows<<<unsigned((count + 127) / 128), 128, 0, st>>>(t.center, t.wt, first, stride, count, out);
        rc = check_launch("k_gen_rows");
    }
    free_tables(t, st);
    return rc;
}

hcg_status gen_queries(uint64_t first, uint64_t count, uint64_t n_db, uint8_t* out, cudaStream_t st) {
    if (count == 0) return HCG_OK;
    if (n_db == 0) return set_error(HCG_EINVAL, "n_db must be >= 1");
    Tables t;
    hcg_status rc = make_tables(t, st);
    if (rc == HCG_OK) {
        k_gen_queries<<<unsigned((count + 127) / 128), 128, 0, st>>>(t.center, t.wt, first, count, n_db, out);
        rc = check_launch("k_gen_queries");
    }
    free_tables(t, st);
    return rc;
}

}  // namespace hcg
