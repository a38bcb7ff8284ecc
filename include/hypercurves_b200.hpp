// hypercurves_b200.hpp -- header-only C++ mirror of the reference's index API
// (namespace hc, proj/include/hypercurves/{multicurves,vecio,curve}.hpp) over
// the C ABI in hcg.h.  A reference user swaps
//
//     hc::MulticurvesIndex idx(ds, hc::default_scheme(128, 8, 16, hc::CurveKind::Hilbert, 0));
//     hc::NeighborList nl = idx.search(q, {10, 350});
// for
//     hcb::MulticurvesIndex idx(ds, hcb::default_scheme(128, 8, 16, hcb::CurveKind::Hilbert, 0));
//     hcb::NeighborList nl = idx.search(q, {10, 350});
//
// and gets the same NeighborLists from the B200.  The default view keeps the
// float components as they are (HCG_F32: the reference's double squared
// distances bit for bit -- sequential sums in index order -- so the same ids,
// distances and tie order).  Byte-valued data can instead be stored as one byte per
// component through View::raw() (bvecs) or View::lifted() (1 + b/256): a 4x
// smaller row, exact integer distances, bit-identical NeighborLists.  The dataset and
// query types are templates: anything with hc::Dataset / hc::FeatureVector's
// shape (`.vectors[i].id`, `.vectors[i].components`, `.dims`) works, the
// reference's own types included.  Errors map back to the reference's
// exception types: std::invalid_argument for precondition / capacity /
// non-finite violations (curve.cpp:35-59,167; vecio.cpp:88,116),
// std::runtime_error for device failures.
//
// With a byte view, descriptors must be byte-valued in it (component ==
// offset + b * scale for an integral b in [0, 255]).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hcg.h"

namespace hcb {

enum class CurveKind : std::uint32_t { ZOrder = HCG_ZORDER, Hilbert = HCG_HILBERT };

struct Neighbor {  // vecio.hpp:27-32
    std::uint64_t id = 0;
    double distance = 0.0;
    friend bool operator==(const Neighbor&, const Neighbor&) = default;
};
using NeighborList = std::vector<Neighbor>;

struct SearchParams {  // multicurves.hpp:69-72
    std::size_t k = 1;
    std::size_t probe_depth = 1;
};

struct ProjectionScheme {  // multicurves.hpp:18-32
    std::uint32_t d_full = 0;
    std::uint32_t bits_per_dim = 8;
    CurveKind curve_kind = CurveKind::Hilbert;
    std::uint64_t seed = 0;
    std::vector<std::vector<std::uint32_t>> assignment;
    std::uint32_t curves() const { return static_cast<std::uint32_t>(assignment.size()); }
    std::uint32_t dims_of(std::uint32_t c) const { return static_cast<std::uint32_t>(assignment[c].size()); }
};

// How descriptors are stored: float components as-is (floats(), the
// reference's own representation), or one byte b per component that the
// reference sees as offset + b * scale.
struct View {
    float offset = 0.0f;
    float scale = 1.0f;
    bool f32 = false;
    static View floats() { return {0.0f, 1.0f, true}; }           // HCG_F32
    static View raw() { return {0.0f, 1.0f, false}; }             // bvecs widening, vecio.cpp:50-51
    static View lifted() { return {1.0f, 1.0f / 256.0f, false}; }  // 1 + b/256
};

namespace detail {
inline void check(hcg_status rc) {
    if (rc == HCG_OK) return;
    const std::string msg = hcg_last_error();
    if (rc == HCG_EINVAL || rc == HCG_ECAPACITY || rc == HCG_ENONFINITE) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline std::uint8_t to_byte(float x, const View& v) {
    if (!std::isfinite(x)) throw std::invalid_argument("non-finite component");
    const float b = (x - v.offset) / v.scale;
    const float r = std::nearbyint(b);
    if (!(r >= 0.0f && r <= 255.0f) || v.offset + r * v.scale != x)
        throw std::invalid_argument("component is not a byte value of the index view");
    return static_cast<std::uint8_t>(r);
}

template <class Vec>
void append_bytes(const Vec& v, std::uint32_t dims, const View& view, std::vector<std::uint8_t>& out) {
    if (v.components.size() != dims) throw std::invalid_argument("dimension mismatch");
    for (float x : v.components) out.push_back(to_byte(x, view));
}

template <class Vec>
void append_floats(const Vec& v, std::uint32_t dims, std::vector<float>& out) {
    if (v.components.size() != dims) throw std::invalid_argument("dimension mismatch");
    out.insert(out.end(), v.components.begin(), v.components.end());
}

// The hcg_scheme of a ProjectionScheme seen through a view (owns the assignment arrays).
struct CScheme {
    std::vector<std::uint32_t> off{0}, asg;
    hcg_scheme s{};
    CScheme(const ProjectionScheme& scheme, const View& view) {
        for (const auto& slots : scheme.assignment) {
            asg.insert(asg.end(), slots.begin(), slots.end());
            off.push_back(static_cast<std::uint32_t>(asg.size()));
        }
        s.d_full = scheme.d_full;
        s.curves = scheme.curves();
        s.bits_per_dim = scheme.bits_per_dim;
        s.curve_kind = static_cast<std::uint32_t>(scheme.curve_kind);
        s.assign_off = off.data();
        s.assign = asg.data();
        s.dist_scale = view.f32 ? 1.0 : view.scale;
        s.dtype = view.f32 ? HCG_F32 : HCG_U8;
        s.view_offset = view.f32 ? 0.0f : view.offset;
        if (!view.f32) check(hcg_make_lut(view.offset, view.scale, scheme.bits_per_dim, s.cell_lut));
    }
    CScheme(const CScheme&) = delete;
};

inline void check_params(const SearchParams& p) {
    if (p.k < 1 || p.probe_depth < 1) throw std::invalid_argument("invalid search params");
    if (p.k > HCG_MAX_K || p.probe_depth > 0xFFFFFFFFu) throw std::invalid_argument("k / probe_depth beyond capacity");
}
}  // namespace detail

// Round-robin assignment; a nonzero seed is unpinned by the
// reference and rejected.
inline ProjectionScheme default_scheme(std::uint32_t d_full, std::uint32_t curves, std::uint32_t bits_per_dim,
                                       CurveKind kind, std::uint64_t seed) {
    if (seed != 0) throw std::invalid_argument("seeded permutation is unpinned by the reference (SPEC.md:203)");
    std::vector<std::uint32_t> off(curves + 1), asg(d_full);
    detail::check(hcg_default_assignment(d_full, curves, off.data(), asg.data()));
    ProjectionScheme s;
    s.d_full = d_full;
    s.bits_per_dim = bits_per_dim;
    s.curve_kind = kind;
    s.seed = seed;
    for (std::uint32_t c = 0; c < curves; ++c) s.assignment.emplace_back(asg.begin() + off[c], asg.begin() + off[c + 1]);
    return s;
}

// hc::MulticurvesIndex on one B200.  Build copies the rows into HBM; search
// is const and may run concurrently from several threads.
class MulticurvesIndex {
  public:
    MulticurvesIndex() = default;

    template <class Dataset>
    MulticurvesIndex(const Dataset& ds, ProjectionScheme scheme, View view = View::floats(), int device = 0)
        : scheme_(std::move(scheme)), view_(view) {
        std::vector<std::uint8_t> rows;
        std::vector<float> frows;
        (view_.f32 ? frows.reserve(ds.vectors.size() * scheme_.d_full)
                   : rows.reserve(ds.vectors.size() * scheme_.d_full));
        for (std::size_t i = 0; i < ds.vectors.size(); ++i) {
            if (ds.vectors[i].id != i) throw std::invalid_argument("dataset ids must be 0..n-1 in order (vecio.hpp:22)");
            if (view_.f32)
                detail::append_floats(ds.vectors[i], scheme_.d_full, frows);
            else
                detail::append_bytes(ds.vectors[i], scheme_.d_full, view_, rows);
        }
        build(view_.f32 ? static_cast<const void*>(frows.data()) : rows.data(), ds.vectors.size(), device);
    }

    // Float rows (n x d_full, e.g. fvecs payloads), ids id_base + s * id_stride.
    MulticurvesIndex(const float* rows, std::uint64_t n, ProjectionScheme scheme, int device = 0,
                     std::uint64_t id_base = 0, std::uint64_t id_stride = 1)
        : scheme_(std::move(scheme)), view_(View::floats()) {
        build(rows, n, device, id_base, id_stride);
    }

    // Raw byte rows (bvecs payloads), ids id_base + s * id_stride.
    MulticurvesIndex(const std::uint8_t* rows, std::uint64_t n, ProjectionScheme scheme, View view, int device = 0,
                     std::uint64_t id_base = 0, std::uint64_t id_stride = 1)
        : scheme_(std::move(scheme)), view_(view) {
        if (view_.f32) throw std::invalid_argument("byte rows need a byte view");
        build(rows, n, device, id_base, id_stride);
    }

    MulticurvesIndex(const MulticurvesIndex&) = delete;
    MulticurvesIndex& operator=(const MulticurvesIndex&) = delete;
    MulticurvesIndex(MulticurvesIndex&& o) noexcept { *this = std::move(o); }
    MulticurvesIndex& operator=(MulticurvesIndex&& o) noexcept {
        std::swap(ix_, o.ix_);
        std::swap(scheme_, o.scheme_);
        std::swap(view_, o.view_);
        return *this;
    }
    ~MulticurvesIndex() {
        if (ix_) hcg_free(ix_);
    }

    std::size_t size() const { return ix_ ? hcg_size(ix_) : 0; }

    // multicurves.hpp:79.  Ids are dense here: v.id must be size() (the next id).
    template <class FeatureVector>
    void insert(const FeatureVector& v) {
        if (v.id != size()) throw std::invalid_argument("insert: ids must continue 0..n-1 in order");
        if (view_.f32) {
            std::vector<float> r;
            detail::append_floats(v, scheme_.d_full, r);
            detail::check(hcg_insert(ix_, reinterpret_cast<const std::uint8_t*>(r.data()), 1, nullptr));
        } else {
            std::vector<std::uint8_t> r;
            detail::append_bytes(v, scheme_.d_full, view_, r);
            detail::check(hcg_insert(ix_, r.data(), 1, nullptr));
        }
    }

    // multicurves.hpp:84: ids of the window of `depth` entries on curve c, in key order.
    template <class FeatureVector>
    std::vector<std::uint64_t> retrieve_candidates(const FeatureVector& q, std::uint32_t c, std::size_t depth) const {
        if (c >= scheme_.curves()) throw std::invalid_argument("curve out of range");
        const std::vector<std::uint8_t> qb = query_bytes(q);
        std::vector<std::uint64_t> rank(scheme_.curves()), begin(scheme_.curves()), end(scheme_.curves());
        detail::check(hcg_windows(ix_, qb.data(), 1, static_cast<std::uint32_t>(depth), rank.data(), begin.data(),
                                  end.data(), nullptr));
        std::vector<std::uint64_t> ids(end[c] - begin[c]);
        detail::check(hcg_sorted_range(ix_, c, begin[c], ids.size(), ids.data(), nullptr));
        return ids;
    }

    // multicurves.hpp:96-98: little-endian binary persistence, bit-exact round trip.
    void save(const std::string& path) const { detail::check(hcg_save(ix_, path.c_str())); }
    static MulticurvesIndex load(const std::string& path, int device = 0) {
        MulticurvesIndex idx;
        detail::check(hcg_load(path.c_str(), device, nullptr, &idx.ix_));
        hcg_scheme s{};
        std::uint32_t n_asg = 0;
        detail::check(hcg_describe(idx.ix_, &s, nullptr, nullptr, &n_asg));
        std::vector<std::uint32_t> off(s.curves + 1), asg(n_asg);
        detail::check(hcg_describe(idx.ix_, &s, off.data(), asg.data(), &n_asg));
        idx.scheme_.d_full = s.d_full;
        idx.scheme_.bits_per_dim = s.bits_per_dim;
        idx.scheme_.curve_kind = static_cast<CurveKind>(s.curve_kind);
        for (std::uint32_t c = 0; c < s.curves; ++c)
            idx.scheme_.assignment.emplace_back(asg.begin() + off[c], asg.begin() + off[c + 1]);
        idx.view_ = s.dtype == HCG_F32 ? View::floats()
                                        : View{s.view_offset, static_cast<float>(s.dist_scale), false};
        return idx;
    }
    const ProjectionScheme& scheme() const { return scheme_; }
    hcg_index* handle() const { return ix_; }

    // multicurves.hpp:81 for one query.
    template <class FeatureVector>
    NeighborList search(const FeatureVector& q, const SearchParams& p) const {
        if (view_.f32) {
            std::vector<float> qf;
            detail::append_floats(q, scheme_.d_full, qf);
            return search_floats(qf.data(), 1, p).front();
        }
        std::vector<std::uint8_t> qb;
        detail::append_bytes(q, scheme_.d_full, view_, qb);
        return search_bytes(qb.data(), 1, p).front();
    }

    // Batched search over float queries (nq x d_full) of a floats() index.
    std::vector<NeighborList> search_floats(const float* queries, std::uint32_t nq, const SearchParams& p,
                                            void* stream = nullptr) const {
        detail::check_params(p);
        const std::uint32_t k = static_cast<std::uint32_t>(p.k);
        std::vector<std::uint64_t> ids(std::size_t(nq) * k);
        std::vector<double> sq(std::size_t(nq) * k);
        std::vector<std::uint32_t> len(nq);
        detail::check(hcg_search_f32(ix_, queries, nq, k, static_cast<std::uint32_t>(p.probe_depth), ids.data(),
                                     sq.data(), len.data(), stream));
        std::vector<NeighborList> out(nq);
        for (std::uint32_t q = 0; q < nq; ++q) {
            out[q].resize(len[q]);
            for (std::uint32_t i = 0; i < len[q]; ++i)
                out[q][i] = {ids[std::size_t(q) * k + i], std::sqrt(sq[std::size_t(q) * k + i])};
        }
        return out;
    }

    // Batched search over byte queries (nq x d_full); one NeighborList each.
    std::vector<NeighborList> search_bytes(const std::uint8_t* queries, std::uint32_t nq, const SearchParams& p,
                                           void* stream = nullptr) const {
        detail::check_params(p);
        const std::uint32_t k = static_cast<std::uint32_t>(p.k);
        std::vector<std::uint64_t> ids(std::size_t(nq) * k);
        std::vector<std::uint32_t> sq(std::size_t(nq) * k), len(nq);
        detail::check(hcg_search(ix_, queries, nq, k, static_cast<std::uint32_t>(p.probe_depth), ids.data(),
                                 sq.data(), len.data(), stream));
        std::vector<NeighborList> out(nq);
        for (std::uint32_t q = 0; q < nq; ++q) {
            out[q].resize(len[q]);
            for (std::uint32_t i = 0; i < len[q]; ++i)
                out[q][i] = {ids[std::size_t(q) * k + i],
                             std::sqrt(double(sq[std::size_t(q) * k + i])) * double(view_.scale)};
        }
        return out;
    }

    // multicurves.hpp:87-89 (sorted ascending).
    template <class FeatureVector>
    std::vector<std::uint64_t> candidate_union(const FeatureVector& q, std::size_t depth) const {
        std::vector<std::uint8_t> qb;
        std::vector<float> qf;
        if (view_.f32)
            detail::append_floats(q, scheme_.d_full, qf);
        else
            detail::append_bytes(q, scheme_.d_full, view_, qb);
        const void* qp = view_.f32 ? static_cast<const void*>(qf.data()) : qb.data();
        const std::uint32_t cap = static_cast<std::uint32_t>(scheme_.curves() * std::min<std::size_t>(depth, size()));
        std::vector<std::uint64_t> ids(cap ? cap : 1);
        std::uint32_t cnt = 0;
        detail::check(hcg_candidates(ix_, static_cast<const std::uint8_t*>(qp), 1, static_cast<std::uint32_t>(depth),
                                     ids.data(), cap ? cap : 1, &cnt, nullptr));
        ids.resize(cnt);
        std::sort(ids.begin(), ids.end());
        return ids;
    }

  private:
    // One query as the index stores it (floats or view bytes), as raw bytes.
    template <class FeatureVector>
    std::vector<std::uint8_t> query_bytes(const FeatureVector& q) const {
        std::vector<std::uint8_t> out;
        if (view_.f32) {
            std::vector<float> f;
            detail::append_floats(q, scheme_.d_full, f);
            out.resize(f.size() * sizeof(float));
            std::memcpy(out.data(), f.data(), out.size());
        } else {
            detail::append_bytes(q, scheme_.d_full, view_, out);
        }
        return out;
    }

    void build(const void* rows, std::uint64_t n, int device, std::uint64_t id_base = 0,
               std::uint64_t id_stride = 1) {
        detail::CScheme cs(scheme_, view_);
        detail::check(hcg_build(&cs.s, static_cast<const std::uint8_t*>(rows), n, id_base, id_stride, device, nullptr,
                                &ix_));
    }

    hcg_index* ix_ = nullptr;
    ProjectionScheme scheme_;
    View view_;
};

// The hypershard module on the GPUs of one process: global
// id i lives on shard i mod G (devices[i mod G]) at local slot i / G; a search
// runs every shard at the per-shard probe depth, all-gathers the packed top-k
// lists with NCCL over NVLink and merges them by (distance, id), truncated to
// k (aggregate) -- the reference's per-shard
// MulticurvesIndex::search + aggregate, bit for bit.  Byte views only.
class ShardedIndex {
  public:
    ShardedIndex() = default;

    // n x d_full view bytes (host or device memory), shard r built on devices[r].
    ShardedIndex(const std::uint8_t* rows, std::uint64_t n, ProjectionScheme scheme, View view,
                 const std::vector<int>& devices)
        : scheme_(std::move(scheme)), view_(view) {
        if (view_.f32) throw std::invalid_argument("sharded indexes store byte views");
        detail::CScheme cs(scheme_, view_);
        detail::check(hcg_shard_group_build(&cs.s, rows, n, static_cast<std::uint32_t>(devices.size()),
                                            devices.data(), &g_));
    }

    template <class Dataset>
    ShardedIndex(const Dataset& ds, ProjectionScheme scheme, View view, const std::vector<int>& devices)
        : scheme_(std::move(scheme)), view_(view) {
        if (view_.f32) throw std::invalid_argument("sharded indexes store byte views");
        std::vector<std::uint8_t> rows;
        rows.reserve(ds.vectors.size() * scheme_.d_full);
        for (std::size_t i = 0; i < ds.vectors.size(); ++i) {
            if (ds.vectors[i].id != i) throw std::invalid_argument("dataset ids must be 0..n-1 in order (vecio.hpp:22)");
            detail::append_bytes(ds.vectors[i], scheme_.d_full, view_, rows);
        }
        detail::CScheme cs(scheme_, view_);
        detail::check(hcg_shard_group_build(&cs.s, rows.data(), ds.vectors.size(),
                                            static_cast<std::uint32_t>(devices.size()), devices.data(), &g_));
    }

    // One process per GPU: rank `rank` of G joins with its shard (built with
    // id_base rank, id_stride G); every rank calls this with the same id.
    static ShardedIndex join(const hcg_nccl_id& id, std::uint32_t rank, std::uint32_t G, MulticurvesIndex& local,
                             View view) {
        ShardedIndex s;
        s.scheme_ = local.scheme();
        s.view_ = view;
        detail::check(hcg_shard_group_join(&id, rank, G, local.handle(), &s.g_));
        return s;
    }

    ShardedIndex(const ShardedIndex&) = delete;
    ShardedIndex& operator=(const ShardedIndex&) = delete;
    ShardedIndex(ShardedIndex&& o) noexcept { *this = std::move(o); }
    ShardedIndex& operator=(ShardedIndex&& o) noexcept {
        std::swap(g_, o.g_);
        std::swap(scheme_, o.scheme_);
        std::swap(view_, o.view_);
        return *this;
    }
    ~ShardedIndex() {
        if (g_) hcg_shard_group_free(g_);
    }

    std::uint32_t shards() const { return g_ ? hcg_shard_group_shards(g_) : 0; }
    hcg_shard_group* handle() const { return g_; }

    // Per-shard probe depth 2 phi* for a sequential depth D: the smallest phi
    // with miss bound <= target for Phi = ceil(D / 2) (SPEC.md:286-329,
    // PAPER.md:883-907).
    static std::size_t plan_depth(std::size_t depth, std::uint32_t shards, double target = 0.02) {
        return 2 * std::size_t(hcg_plan_depth(static_cast<std::uint32_t>((depth + 1) / 2), shards, target));
    }

    // Batched search; p.probe_depth is the per-shard depth.
    std::vector<NeighborList> search_bytes(const std::uint8_t* queries, std::uint32_t nq, const SearchParams& p,
                                           void* stream = nullptr) const {
        detail::check_params(p);
        const std::uint32_t k = static_cast<std::uint32_t>(p.k);
        std::vector<std::uint64_t> ids(std::size_t(nq) * k);
        std::vector<std::uint32_t> sq(std::size_t(nq) * k), len(nq);
        detail::check(hcg_shard_group_search(g_, queries, nq, k, static_cast<std::uint32_t>(p.probe_depth),
                                             ids.data(), sq.data(), len.data(), stream));
        std::vector<NeighborList> out(nq);
        for (std::uint32_t q = 0; q < nq; ++q) {
            out[q].resize(len[q]);
            for (std::uint32_t i = 0; i < len[q]; ++i)
                out[q][i] = {ids[std::size_t(q) * k + i],
                             std::sqrt(double(sq[std::size_t(q) * k + i])) * double(view_.scale)};
        }
        return out;
    }

    template <class FeatureVector>
    NeighborList search(const FeatureVector& q, const SearchParams& p) const {
        std::vector<std::uint8_t> qb;
        detail::append_bytes(q, scheme_.d_full, view_, qb);
        return search_bytes(qb.data(), 1, p).front();
    }

  private:
    hcg_shard_group* g_ = nullptr;
    ProjectionScheme scheme_;
    View view_;
};

}  // namespace hcb
