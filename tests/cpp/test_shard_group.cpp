// hcb::ShardedIndex (include/hypercurves_b200.hpp) over libhcg's shard group on
// all GPUs of one process (G = device count, >= 2): per-shard sm_100a search,
// NCCL all-gather inside the library, K4 merge -- against the sharded CPU
// oracle (shard r holds ids r, r + G, ...; per-shard search
// at the per-shard depth; merge by (distance, id), truncated to k).
// Prints "shard group ok" and exits 0 on bit-identical NeighborLists.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <tuple>
#include <vector>

#include "hypercurves_b200.hpp"

extern "C" {
void* orc_build(uint32_t, uint32_t, uint32_t, uint32_t, const uint32_t*, const uint32_t*, const float*, uint64_t,
                const uint64_t*, int, int*);
int orc_default_scheme(uint32_t, uint32_t, uint32_t*, uint32_t*);
int orc_search(void*, const float*, uint64_t, uint64_t, uint64_t, uint64_t*, double*, uint32_t*, int);
void orc_gen_rows(uint64_t, uint64_t, uint8_t*, int);
void orc_gen_queries(uint64_t, uint64_t, uint64_t, uint8_t*, int);
void orc_free(void*);
}

int main() {
    int G = 0;
    cudaGetDeviceCount(&G);
    if (G < 2) {
        std::printf("needs >= 2 GPUs\n");
        return 2;
    }
    G = std::min(G, 8);
    const uint32_t n = 30001, nq = 200, d = 128, C = 8, m = 16;
    std::vector<uint8_t> rows(size_t(n) * d), qs(size_t(nq) * d);
    orc_gen_rows(0, n, rows.data(), 8);
    orc_gen_queries(0, nq, n, qs.data(), 8);
    std::vector<int> devs(G);
    for (int r = 0; r < G; ++r) devs[r] = r;
    const hcb::View view = hcb::View::lifted();
    hcb::ShardedIndex sharded(rows.data(), n, hcb::default_scheme(d, C, m, hcb::CurveKind::Hilbert, 0), view, devs);
    int bad = sharded.shards() == uint32_t(G) ? 0 : 1;

    std::vector<uint32_t> off(C + 1), asg(d);
    orc_default_scheme(d, C, off.data(), asg.data());
    std::vector<float> qf(size_t(nq) * d);
    for (size_t i = 0; i < qf.size(); ++i) qf[i] = 1.0f + float(qs[i]) / 256.0f;
    const uint64_t k = 10;
    for (size_t depth : {size_t(64), hcb::ShardedIndex::plan_depth(350, uint32_t(G)), size_t(5000)}) {
        // oracle: per-shard search, then the (distance, id) merge
        std::vector<std::vector<std::tuple<double, uint64_t>>> pool(nq);
        for (int r = 0; r < G; ++r) {
            std::vector<float> f;
            std::vector<uint64_t> ids;
            for (uint64_t i = r; i < n; i += G) {
                ids.push_back(i);
                for (uint32_t j = 0; j < d; ++j) f.push_back(1.0f + float(rows[i * d + j]) / 256.0f);
            }
            int err = 0;
            void* oi = orc_build(d, C, m, 1, off.data(), asg.data(), f.data(), ids.size(), ids.data(), 8, &err);
            std::vector<uint64_t> oids(nq * k);
            std::vector<double> od(nq * k);
            std::vector<uint32_t> ol(nq);
            orc_search(oi, qf.data(), nq, k, depth, oids.data(), od.data(), ol.data(), 8);
            orc_free(oi);
            for (uint32_t q = 0; q < nq; ++q)
                for (uint32_t i = 0; i < ol[q]; ++i) pool[q].emplace_back(od[q * k + i], oids[q * k + i]);
        }
        const auto got = sharded.search_bytes(qs.data(), nq, {k, depth});
        for (uint32_t q = 0; q < nq; ++q) {
            std::sort(pool[q].begin(), pool[q].end());
            if (pool[q].size() > k) pool[q].resize(k);
            if (got[q].size() != pool[q].size()) {
                ++bad;
                continue;
            }
            for (size_t i = 0; i < got[q].size(); ++i)
                if (got[q][i].id != std::get<1>(pool[q][i]) || got[q][i].distance != std::get<0>(pool[q][i])) ++bad;
        }
        // device-resident queries on the first GPU: the same lists
        uint8_t* dq = nullptr;
        cudaSetDevice(0);
        cudaMalloc(&dq, qs.size());
        cudaMemcpy(dq, qs.data(), qs.size(), cudaMemcpyHostToDevice);
        const auto got_d = sharded.search_bytes(dq, nq, {k, depth});
        cudaFree(dq);
        for (uint32_t q = 0; q < nq; ++q)
            if (!(got_d[q] == got[q])) ++bad;
        std::printf("G=%d depth=%zu mismatches so far %d\n", G, depth, bad);
    }
    try {  // reference error behaviour
        sharded.search_bytes(qs.data(), 1, {0, 10});
        ++bad;
    } catch (const std::invalid_argument&) {
    }
    std::printf(bad ? "shard group FAILED (%d)\n" : "shard group ok\n", bad);
    return bad ? 1 : 0;
}
