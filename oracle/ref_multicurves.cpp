// ref_multicurves.cpp -- CPU ORACLE / CPU BASELINE glue (test infrastructure only).
//
// Compiled by oracle/Makefile together with the UNMODIFIED reference TUs
// /root/reference/proj/src/curve.cpp and vecio.cpp (read where they lie, never
// copied) into oracle/_ref/libhcref.so.  The reference ships the header
// proj/include/hypercurves/multicurves.hpp but not multicurves.cpp
// (proj/src/CMakeLists.txt:4), so this file supplies the missing member
// definitions, written against the header contract:
//   ProjectionScheme::validate / default_scheme ... multicurves.hpp:18-38
//   project ....................................... multicurves.hpp:40
//   SubIndex::bulk_load/insert (key, id order) ..... multicurves.hpp:47-52
//   SubIndex::rank_of (key-only lower_bound) ....... multicurves.hpp:57-58
//   SubIndex::window (floor below, ceil at/above) .. multicurves.hpp:60-63
//   MulticurvesIndex ctor/search/candidates ........ multicurves.hpp:74-107
// Everything on the arithmetic side (quantizer, curve keys, ExtendedKey order,
// squared_distance, select_top_k, brute_force_knn) is the reference's own code.
//
// It is used (a) to pin the independent restatement in hc_oracle.cpp and
// (b) as bench.py's reference CPU arm / cpu_baseline (kind "reference").
// The product path never links it.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include "hypercurves/curve.hpp"
#include "hypercurves/keys.hpp"
#include "hypercurves/multicurves.hpp"
#include "hypercurves/vecio.hpp"

namespace hc {

void ProjectionScheme::validate() const {
    if (assignment.empty()) throw std::invalid_argument("scheme needs at least one curve");
    std::vector<bool> covered(d_full, false);
    for (const auto& slots : assignment) {
        if (slots.empty()) throw std::invalid_argument("curve with no dimensions");
        if (std::uint64_t(slots.size()) * bits_per_dim > kMaxKeyBits)
            throw std::invalid_argument("key width exceeds capacity");
        for (auto a : slots) {
            if (a >= d_full) throw std::invalid_argument("assignment out of range");
            covered[a] = true;
        }
    }
    for (bool c : covered)
        if (!c) throw std::invalid_argument("input dimension not covered by any curve");
    if (bits_per_dim < 1 || bits_per_dim > 32) throw std::invalid_argument("bits_per_dim out of range");
}

ProjectionScheme default_scheme(std::uint32_t d_full, std::uint32_t curves,
                                std::uint32_t bits_per_dim, CurveKind kind, std::uint64_t seed) {
    if (curves < 1 || curves > d_full) throw std::invalid_argument("curves must be in [1, d_full]");
    if (seed != 0)
        throw std::invalid_argument("seeded permutation is unpinned by the reference (SPEC.md:203)");
    ProjectionScheme s;
    s.d_full = d_full;
    s.bits_per_dim = bits_per_dim;
    s.curve_kind = kind;
    s.seed = seed;
    s.assignment.assign(curves, {});
    for (std::uint32_t j = 0; j < d_full; ++j) s.assignment[j % curves].push_back(j);
    return s;
}

OrdinalPoint project(const FeatureVector& v, const ProjectionScheme& scheme, std::uint32_t c) {
    OrdinalPoint p;
    p.bits_per_dim = scheme.bits_per_dim;
    p.coords.reserve(scheme.dims_of(c));
    for (auto a : scheme.assignment[c]) p.coords.push_back(quantize_component(v.components[a], p.bits_per_dim));
    return p;
}

static bool entry_less(const SubIndexEntry& a, const SubIndexEntry& b) {
    const auto o = a.key <=> b.key;
    return o != 0 ? o < 0 : a.id < b.id;
}

void SubIndex::bulk_load(std::vector<SubIndexEntry>&& entries) {
    entries_ = std::move(entries);
    std::sort(entries_.begin(), entries_.end(), entry_less);
}

void SubIndex::insert(SubIndexEntry entry) {
    entries_.insert(std::upper_bound(entries_.begin(), entries_.end(), entry, entry_less), entry);
}

std::size_t SubIndex::rank_of(const ExtendedKey& key) const {
    return std::size_t(std::lower_bound(entries_.begin(), entries_.end(), key,
                                        [](const SubIndexEntry& e, const ExtendedKey& k) {
                                            return (e.key <=> k) < 0;
                                        }) -
                       entries_.begin());
}

std::pair<std::size_t, std::size_t> SubIndex::window(const ExtendedKey& key, std::size_t depth) const {
    const std::size_t n = entries_.size();
    const std::size_t take = std::min(depth, n);
    const std::size_t r = rank_of(key);
    const std::size_t below = take / 2;
    std::size_t begin = r >= below ? r - below : 0;
    std::size_t end = begin + take;
    if (end > n) {
        end = n;
        begin = n - take;
    }
    return {begin, end};
}

MulticurvesIndex::MulticurvesIndex(const Dataset& ds, ProjectionScheme scheme)
    : scheme_(std::move(scheme)), dataset_(ds) {
    scheme_.validate();
    std::uint64_t max_id = 0;
    for (const auto& v : dataset_.vectors) max_id = std::max(max_id, v.id);
    id_to_slot_.assign(dataset_.empty() ? 0 : max_id + 1, ~std::uint64_t{0});
    for (std::size_t s = 0; s < dataset_.size(); ++s) {
        if (dataset_[s].dims() != scheme_.d_full) throw std::invalid_argument("dimension mismatch");
        if (id_to_slot_[dataset_[s].id] != ~std::uint64_t{0}) throw std::invalid_argument("duplicate id");
        id_to_slot_[dataset_[s].id] = s;
    }
    subindexes_.resize(scheme_.curves());
    // One thread per curve (BASELINE.md §2 "Index build runs one thread per curve").
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(scheme_.curves());
    for (std::uint32_t c = 0; c < scheme_.curves(); ++c)
        pool.emplace_back([&, c] {
            try {
                std::vector<SubIndexEntry> entries;
                entries.reserve(dataset_.size());
                for (const auto& v : dataset_.vectors)
                    entries.push_back({curve_encode(scheme_.curve_kind, project(v, scheme_, c)), v.id});
                subindexes_[c].bulk_load(std::move(entries));
            } catch (...) {
                errs[c] = std::current_exception();
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

void MulticurvesIndex::insert(const FeatureVector& v) {
    if (v.id < id_to_slot_.size() && id_to_slot_[v.id] != ~std::uint64_t{0})
        throw std::invalid_argument("duplicate id");
    if (v.dims() != scheme_.d_full) throw std::invalid_argument("dimension mismatch");
    if (v.id >= id_to_slot_.size()) id_to_slot_.resize(v.id + 1, ~std::uint64_t{0});
    id_to_slot_[v.id] = dataset_.size();
    dataset_.vectors.push_back(v);
    for (std::uint32_t c = 0; c < scheme_.curves(); ++c)
        subindexes_[c].insert({curve_encode(scheme_.curve_kind, project(v, scheme_, c)), v.id});
}

std::vector<std::uint64_t> MulticurvesIndex::retrieve_candidates(const FeatureVector& query,
                                                                 std::uint32_t c,
                                                                 std::size_t depth) const {
    const auto key = curve_encode(scheme_.curve_kind, project(query, scheme_, c));
    const auto [b, e] = subindexes_[c].window(key, depth);
    std::vector<std::uint64_t> ids;
    ids.reserve(e - b);
    for (std::size_t p = b; p < e; ++p) ids.push_back(subindexes_[c].entries()[p].id);
    return ids;
}

std::vector<std::uint64_t> MulticurvesIndex::candidate_union(const FeatureVector& query,
                                                             std::size_t depth) const {
    std::vector<std::uint64_t> all;
    for (std::uint32_t c = 0; c < scheme_.curves(); ++c) {
        auto part = retrieve_candidates(query, c, depth);
        all.insert(all.end(), part.begin(), part.end());
    }
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    return all;
}

NeighborList MulticurvesIndex::search(const FeatureVector& query, const SearchParams& params) const {
    if (params.k < 1 || params.probe_depth < 1) throw std::invalid_argument("invalid search params");
    std::vector<Neighbor> sq;
    for (auto id : candidate_union(query, params.probe_depth))
        sq.push_back({id, squared_distance(query.components, dataset_[id_to_slot_[id]].components)});
    return select_top_k(std::move(sq), params.k);
}

}  // namespace hc

// ---------------------------------------------------------------------------
// C API for ctypes (tests + bench).  Same argument meaning as hc_oracle.cpp's
// orc_* functions; errors are caught here and returned as negative codes.
// ---------------------------------------------------------------------------
namespace {
thread_local std::string g_err;

float view_value(std::uint8_t b, int view) {
    return view == 1 ? 1.0f + float(b) / 256.0f : float(b);
}

hc::FeatureVector make_vec(const std::uint8_t* row, std::uint32_t dim, int view, std::uint64_t id) {
    hc::FeatureVector v;
    v.id = id;
    v.components.resize(dim);
    for (std::uint32_t j = 0; j < dim; ++j) v.components[j] = view_value(row[j], view);
    return v;
}

struct RefIndex {
    hc::MulticurvesIndex index;
    std::uint32_t dim;
    int view;
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -4;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint32_t ref_float_to_ordinal(float x, int* err) {
    std::uint32_t r = 0;
    *err = guard([&] { r = hc::float_to_ordinal(x); });
    return r;
}

int ref_quantize(float x, std::uint32_t m, std::uint64_t* out) {
    return guard([&] { *out = hc::quantize_component(x, m); });
}

int ref_curve_encode(std::uint32_t kind, std::uint32_t d, std::uint32_t m, const std::uint64_t* coords,
                     std::uint64_t* key16) {
    return guard([&] {
        hc::OrdinalPoint p;
        p.bits_per_dim = m;
        p.coords.assign(coords, coords + d);
        const auto k = hc::curve_encode(kind ? hc::CurveKind::Hilbert : hc::CurveKind::ZOrder, p);
        std::memcpy(key16, k.words.data(), 8 * hc::kKeyWords);
    });
}

int ref_curve_decode(std::uint32_t kind, std::uint32_t d, std::uint32_t m, const std::uint64_t* key16,
                     std::uint64_t* coords) {
    return guard([&] {
        hc::ExtendedKey k = hc::ExtendedKey::zero(d * m);
        std::memcpy(k.words.data(), key16, 8 * hc::kKeyWords);
        const auto p = kind ? hc::hilbert_decode(k, d, m) : hc::zorder_decode(k, d, m);
        std::memcpy(coords, p.coords.data(), 8 * d);
    });
}

// rows: n x dim bytes, viewed as floats by `view` (0 raw: float(b); 1 lifted: 1+b/256).
void* ref_build(std::uint32_t dim, std::uint32_t curves, std::uint32_t m, std::uint32_t kind,
                const std::uint8_t* rows, std::uint64_t n, int view, int* err) {
    RefIndex* out = nullptr;
    *err = guard([&] {
        hc::Dataset ds;
        ds.dims = dim;
        ds.vectors.resize(n);
        for (std::uint64_t i = 0; i < n; ++i) ds.vectors[i] = make_vec(rows + i * dim, dim, view, i);
        auto scheme = hc::default_scheme(dim, curves, m, kind ? hc::CurveKind::Hilbert : hc::CurveKind::ZOrder, 0);
        out = new RefIndex{hc::MulticurvesIndex(ds, scheme), dim, view};
    });
    return out;
}

// The same over one shard of an id mod G partition: row i
// carries the global id id_base + i * id_stride.
void* ref_build_ids(std::uint32_t dim, std::uint32_t curves, std::uint32_t m, std::uint32_t kind,
                    const std::uint8_t* rows, std::uint64_t n, int view, std::uint64_t id_base,
                    std::uint64_t id_stride, int* err) {
    RefIndex* out = nullptr;
    *err = guard([&] {
        hc::Dataset ds;
        ds.dims = dim;
        ds.vectors.resize(n);
        for (std::uint64_t i = 0; i < n; ++i)
            ds.vectors[i] = make_vec(rows + i * dim, dim, view, id_base + i * id_stride);
        auto scheme = hc::default_scheme(dim, curves, m, kind ? hc::CurveKind::Hilbert : hc::CurveKind::ZOrder, 0);
        out = new RefIndex{hc::MulticurvesIndex(ds, scheme), dim, view};
    });
    return out;
}

void ref_free(void* h) { delete static_cast<RefIndex*>(h); }

// keys_out: n x words (LS word first), ids_out: n.
void ref_sorted(void* h, std::uint32_t c, std::uint32_t words, std::uint64_t* keys_out, std::uint64_t* ids_out) {
    const auto& e = static_cast<RefIndex*>(h)->index.subindex(c).entries();
    for (std::size_t p = 0; p < e.size(); ++p) {
        if (keys_out) std::memcpy(keys_out + p * words, e[p].key.words.data(), 8 * words);
        if (ids_out) ids_out[p] = e[p].id;
    }
}

int ref_windows(void* h, const std::uint8_t* qs, std::uint64_t nq, std::uint64_t depth,
                std::uint64_t* rank_out, std::uint64_t* begin_out, std::uint64_t* end_out) {
    auto* r = static_cast<RefIndex*>(h);
    return guard([&] {
        const auto& sc = r->index.scheme();
        for (std::uint64_t q = 0; q < nq; ++q) {
            const auto v = make_vec(qs + q * r->dim, r->dim, r->view, q);
            for (std::uint32_t c = 0; c < sc.curves(); ++c) {
                const auto key = hc::curve_encode(sc.curve_kind, hc::project(v, sc, c));
                const auto o = q * sc.curves() + c;
                rank_out[o] = r->index.subindex(c).rank_of(key);
                const auto [b, e] = r->index.subindex(c).window(key, depth);
                begin_out[o] = b;
                end_out[o] = e;
            }
        }
    });
}

std::uint64_t ref_candidates(void* h, const std::uint8_t* q, std::uint64_t depth, std::uint64_t* out) {
    auto* r = static_cast<RefIndex*>(h);
    const auto ids = r->index.candidate_union(make_vec(q, r->dim, r->view, 0), depth);
    if (out) std::memcpy(out, ids.data(), 8 * ids.size());
    return ids.size();
}

// Query-parallel search over `threads` threads pulling from a shared counter.
int ref_search(void* h, const std::uint8_t* qs, std::uint64_t nq, std::uint64_t k, std::uint64_t depth,
               std::uint64_t* out_ids, double* out_dist, std::uint32_t* out_len, int threads) {
    auto* r = static_cast<RefIndex*>(h);
    std::atomic<std::uint64_t> next{0};
    std::atomic<int> rc{0};
    auto work = [&] {
        for (std::uint64_t q; (q = next.fetch_add(1)) < nq;) {
            const int e = guard([&] {
                const auto nl = r->index.search(make_vec(qs + q * r->dim, r->dim, r->view, q),
                                                hc::SearchParams{k, depth});
                out_len[q] = std::uint32_t(nl.size());
                for (std::size_t i = 0; i < nl.size(); ++i) {
                    out_ids[q * k + i] = nl[i].id;
                    out_dist[q * k + i] = nl[i].distance;
                }
            });
            if (e) rc = e;
        }
    };
    if (threads <= 1) {
        work();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work);
        for (auto& t : pool) t.join();
    }
    return rc;
}

int ref_brute_force(void* h, const std::uint8_t* qs, std::uint64_t nq, std::uint64_t k,
                    std::uint64_t* out_ids, double* out_dist, std::uint32_t* out_len, int threads) {
    auto* r = static_cast<RefIndex*>(h);
    std::atomic<std::uint64_t> next{0};
    std::atomic<int> rc{0};
    auto work = [&] {
        for (std::uint64_t q; (q = next.fetch_add(1)) < nq;) {
            const int e = guard([&] {
                const auto nl = hc::brute_force_knn(r->index.dataset(), make_vec(qs + q * r->dim, r->dim, r->view, q), k);
                out_len[q] = std::uint32_t(nl.size());
                for (std::size_t i = 0; i < nl.size(); ++i) {
                    out_ids[q * k + i] = nl[i].id;
                    out_dist[q * k + i] = nl[i].distance;
                }
            });
            if (e) rc = e;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    return rc;
}

int ref_select_top_k(const std::uint64_t* ids, const double* sq, std::uint64_t n, std::uint64_t k,
                     std::uint64_t* out_ids, double* out_dist) {
    std::vector<hc::Neighbor> v(n);
    for (std::uint64_t i = 0; i < n; ++i) v[i] = {ids[i], sq[i]};
    const auto nl = hc::select_top_k(std::move(v), k);
    for (std::size_t i = 0; i < nl.size(); ++i) {
        out_ids[i] = nl[i].id;
        out_dist[i] = nl[i].distance;
    }
    return int(nl.size());
}

}  // extern "C"

// ---- vecio round trip through the reference's own reader (vecio.cpp:18-61) ----
extern "C" int ref_read_vectors(const char* path, int bvecs, float* out, std::uint64_t cap, std::uint64_t* n,
                                std::uint32_t* dim) {
    return guard([&] {
        const auto ds = hc::read_vectors(path, bvecs ? hc::VectorFormat::bvecs : hc::VectorFormat::fvecs);
        *n = ds.size();
        *dim = ds.dims;
        std::uint64_t k = 0;
        for (const auto& v : ds.vectors)
            for (float x : v.components)
                if (k < cap) out[k++] = x;
    });
}
