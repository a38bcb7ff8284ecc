// C++ drop-in test: hcb::MulticurvesIndex (include/hypercurves_b200.hpp) over
// libhcg.so against the CPU oracle (oracle/liboracle.so, test infrastructure).
// Prints "wrapper ok" and exits 0 on bit-identical NeighborLists.
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <cstdlib>
#include <limits>
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

struct Vec {
    std::uint64_t id;
    std::vector<float> components;
};
struct Data {
    std::uint32_t dims;
    std::vector<Vec> vectors;
};

int main() {
    const uint32_t n = 20000, nq = 50, d = 128, C = 8, m = 16;
    std::vector<uint8_t> rows(size_t(n) * d), qs(size_t(nq) * d);
    orc_gen_rows(0, n, rows.data(), 4);
    orc_gen_queries(0, nq, n, qs.data(), 4);
    const hcb::View view = hcb::View::lifted();
    Data ds{d, {}};
    std::vector<float> f(size_t(n) * d), qf(size_t(nq) * d);
    for (uint32_t i = 0; i < n; ++i) {
        Vec v{i, std::vector<float>(d)};
        for (uint32_t j = 0; j < d; ++j) v.components[j] = f[size_t(i) * d + j] = 1.0f + float(rows[size_t(i) * d + j]) / 256.0f;
        ds.vectors.push_back(std::move(v));
    }
    for (size_t i = 0; i < qf.size(); ++i) qf[i] = 1.0f + float(qs[i]) / 256.0f;

    hcb::MulticurvesIndex idx(ds, hcb::default_scheme(d, C, m, hcb::CurveKind::Hilbert, 0), view);
    std::vector<uint32_t> off(C + 1), asg(d);
    orc_default_scheme(d, C, off.data(), asg.data());
    int err = 0;
    void* oi = orc_build(d, C, m, 1, off.data(), asg.data(), f.data(), n, nullptr, 4, &err);
    const uint64_t k = 10, depth = 350;
    std::vector<uint64_t> oids(nq * k);
    std::vector<double> od(nq * k);
    std::vector<uint32_t> ol(nq);
    orc_search(oi, qf.data(), nq, k, depth, oids.data(), od.data(), ol.data(), 4);
    int bad = 0;
    for (uint32_t q = 0; q < nq; ++q) {
        Vec qv{q, std::vector<float>(qf.begin() + size_t(q) * d, qf.begin() + size_t(q + 1) * d)};
        const hcb::NeighborList nl = idx.search(qv, {k, depth});
        if (nl.size() != ol[q]) ++bad;
        for (size_t i = 0; i < nl.size() && i < ol[q]; ++i)
            if (nl[i].id != oids[q * k + i] || nl[i].distance != od[q * k + i]) ++bad;
        if (q == 0) {
            const auto cu = idx.candidate_union(qv, depth);
            if (cu.empty() || cu.size() > C * depth) ++bad;
        }
    }
    // reference error behaviour: invalid_argument on bad params / non-byte components
    try {
        Vec qv{0, std::vector<float>(d, 0.5f)};
        idx.search(qv, {k, depth});
        ++bad;
    } catch (const std::invalid_argument&) {
    }
    try {
        Vec qv{0, std::vector<float>(qf.begin(), qf.begin() + d)};
        idx.search(qv, {0, depth});
        ++bad;
    } catch (const std::invalid_argument&) {
    }
    orc_free(oi);

    // Float descriptors through the default view (HCG_F32): arbitrary signed
    // floats, ids and distances bit-identical to the oracle.
    {
        std::srand(7);
        auto rnd = [] { return (float(std::rand()) / float(RAND_MAX) - 0.5f) * 200.0f; };
        Data fd{d, {}};
        std::vector<float> ff(size_t(n) * d), fq(size_t(nq) * d);
        for (uint32_t i = 0; i < n; ++i) {
            Vec v{i, std::vector<float>(d)};
            for (uint32_t j = 0; j < d; ++j) v.components[j] = ff[size_t(i) * d + j] = rnd();
            fd.vectors.push_back(std::move(v));
        }
        for (auto& x : fq) x = rnd();
        hcb::MulticurvesIndex fidx(fd, hcb::default_scheme(d, C, m, hcb::CurveKind::Hilbert, 0));
        void* fo = orc_build(d, C, m, 1, off.data(), asg.data(), ff.data(), n, nullptr, 4, &err);
        orc_search(fo, fq.data(), nq, k, depth, oids.data(), od.data(), ol.data(), 4);
        for (uint32_t q = 0; q < nq; ++q) {
            Vec qv{q, std::vector<float>(fq.begin() + size_t(q) * d, fq.begin() + size_t(q + 1) * d)};
            const hcb::NeighborList nl = fidx.search(qv, {k, depth});
            if (nl.size() != ol[q]) ++bad;
            for (size_t i = 0; i < nl.size() && i < ol[q]; ++i)
                if (nl[i].id != oids[q * k + i] || nl[i].distance != od[q * k + i]) ++bad;
        }
        try {  // non-finite query component: invalid_argument (curve.cpp:167)
            Vec qv{0, std::vector<float>(d, 1.0f)};
            qv.components[3] = std::numeric_limits<float>::quiet_NaN();
            fidx.search(qv, {k, depth});
            ++bad;
        } catch (const std::invalid_argument&) {
        }
        // retrieve_candidates (one curve's window, key order) within the union
        {
            Vec qv{0, std::vector<float>(fq.begin(), fq.begin() + d)};
            const auto w0 = fidx.retrieve_candidates(qv, 0, 64);
            const auto un = fidx.candidate_union(qv, 64);
            if (w0.size() != 64) ++bad;
            for (auto id : w0)
                if (!std::binary_search(un.begin(), un.end(), id)) ++bad;
        }
        // save / load (scheme and view come back from the file) and insert
        {
            const std::string path = "/tmp/hcb_wrapper_test.hcg";
            fidx.save(path);
            hcb::MulticurvesIndex back = hcb::MulticurvesIndex::load(path);
            Vec qv{0, std::vector<float>(fq.begin(), fq.begin() + d)};
            if (back.search(qv, {k, depth}) != fidx.search(qv, {k, depth})) ++bad;
            if (back.size() != n || back.scheme().curves() != C) ++bad;
            Vec nv{n, std::vector<float>(fq.begin(), fq.begin() + d)};  // the query itself, id n
            back.insert(nv);
            const hcb::NeighborList nl = back.search(qv, {1, depth});
            if (back.size() != n + 1 || nl.empty() || nl[0].id != n || nl[0].distance != 0.0) ++bad;
            try {  // ids must continue densely
                Vec gap{n + 5, std::vector<float>(d, 1.0f)};
                back.insert(gap);
                ++bad;
            } catch (const std::invalid_argument&) {
            }
            std::remove(path.c_str());
        }
        orc_free(fo);
    }
    if (bad) {
        std::printf("wrapper FAILED: %d mismatches\n", bad);
        return 1;
    }
    std::printf("wrapper ok: %u queries identical to the oracle\n", nq);
    return 0;
}
