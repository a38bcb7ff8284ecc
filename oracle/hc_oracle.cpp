// hc_oracle.cpp -- CPU ORACLE (test infrastructure only).
//
// An independent, plain restatement of the reference's approximate-kNN hot
// path, used ONLY by tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg as the checker.  The product path (paper_1209_0410_b200/)
// never links or calls this file.
//
// Each function cites the reference file:line it restates (paths relative to
// the reference repo root, /root/reference in the build container):
//   float_to_ordinal ........ proj/src/curve.cpp:166-170
//   quantize_component ...... proj/src/curve.cpp:172-174
//   interleave .............. proj/src/curve.cpp:62-75
//   axes_to_transpose ....... proj/src/curve.cpp:100-123 (Skilling 2004)
//   transpose_to_axes ....... proj/src/curve.cpp:125-145
//   hilbert/zorder encode ... proj/src/curve.cpp:90-93,147-164
//   validate_point .......... proj/src/curve.cpp:38-51
//   ExtendedKey compare ..... proj/include/hypercurves/keys.hpp:50-57
//   squared_distance ........ proj/src/vecio.cpp:87-95
//   select_top_k ............ proj/src/vecio.cpp:101-113
//   brute_force_knn ......... proj/src/vecio.cpp:115-122
//   default_scheme .......... multicurves.hpp:36-38 + SPEC.md:200-208 (seed 0)
//   project ................. multicurves.hpp:40 + SPEC.md:209-217
//   SubIndex order .......... multicurves.hpp:47-48 (key, then id)
//   rank_of ................. multicurves.hpp:57-58 (key-only lower_bound)
//   window .................. multicurves.hpp:60-63 (floor below / ceil at-or-above,
//                              boundary deficit spills to the other side)
//   candidate_union ......... multicurves.hpp:87-89 + SPEC.md:262 (dedup)
//   search .................. multicurves.hpp:81 + SPEC.md:245-253
//   synthetic generator ..... SURVEY.md §8(d) (counter-based, integer only)
//
// Parity pins: the SURVEY.md §A golden vectors (produced by running the shipped
// reference curve.cpp/vecio.cpp) and, when oracle/_ref was built, the reference
// TUs themselves (tests/test_oracle.py cross-checks both).

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

constexpr uint32_t kMaxWords = 16;  // 1024-bit capacity (keys.hpp:15-23)

enum : int { ORC_OK = 0, ORC_EINVAL = -1, ORC_ECAPACITY = -2, ORC_ENONFINITE = -3 };

inline uint32_t ordinal_of(float x) {
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    // sign set -> flip every bit; sign clear -> set the sign bit.
    return (bits >> 31) ? ~bits : (bits | 0x80000000u);
}

inline bool finite(float x) { return std::isfinite(x); }

// Skilling's "AxestoTranspose" on m-bit coordinates (in place).
void hilbert_transpose(uint64_t* x, uint32_t d, uint32_t m) {
    if (m == 0) return;
    const uint64_t top = uint64_t{1} << (m - 1);
    for (uint64_t q = top; q > 1; q >>= 1) {
        const uint64_t low = q - 1;
        for (uint32_t i = 0; i < d; ++i) {
            if (x[i] & q) {
                x[0] ^= low;
            } else {
                const uint64_t swap = (x[0] ^ x[i]) & low;
                x[0] ^= swap;
                x[i] ^= swap;
            }
        }
    }
    for (uint32_t i = 1; i < d; ++i) x[i] ^= x[i - 1];
    uint64_t fix = 0;
    for (uint64_t q = top; q > 1; q >>= 1)
        if (x[d - 1] & q) fix ^= q - 1;
    for (uint32_t i = 0; i < d; ++i) x[i] ^= fix;
}

// Inverse of hilbert_transpose.
void hilbert_untranspose(uint64_t* x, uint32_t d, uint32_t m) {
    const uint64_t limit = (m >= 64) ? 0 : (uint64_t{1} << m);
    const uint64_t t = x[d - 1] >> 1;
    for (uint32_t i = d - 1; i > 0; --i) x[i] ^= x[i - 1];
    x[0] ^= t;
    for (uint64_t q = 2; q != limit; q <<= 1) {
        const uint64_t low = q - 1;
        for (uint32_t i = d; i-- > 0;) {
            if (x[i] & q) {
                x[0] ^= low;
            } else {
                const uint64_t swap = (x[0] ^ x[i]) & low;
                x[0] ^= swap;
                x[i] ^= swap;
            }
        }
    }
}

// Plane j (0 = MSB plane) of coordinate i -> key bit (width-1-(j*d+i)).
void bits_interleave(const uint64_t* x, uint32_t d, uint32_t m, uint64_t* key) {
    const uint32_t width = d * m;
    std::memset(key, 0, kMaxWords * 8);
    uint32_t pos = width;  // next key bit to fill is pos-1
    for (uint32_t j = 0; j < m; ++j) {
        for (uint32_t i = 0; i < d; ++i) {
            --pos;
            if ((x[i] >> (m - 1 - j)) & 1u) key[pos >> 6] |= uint64_t{1} << (pos & 63);
        }
    }
}

void bits_deinterleave(const uint64_t* key, uint32_t d, uint32_t m, uint64_t* x) {
    const uint32_t width = d * m;
    for (uint32_t i = 0; i < d; ++i) x[i] = 0;
    uint32_t pos = width;
    for (uint32_t j = 0; j < m; ++j) {
        for (uint32_t i = 0; i < d; ++i) {
            --pos;
            if ((key[pos >> 6] >> (pos & 63)) & 1u) x[i] |= uint64_t{1} << (m - 1 - j);
        }
    }
}

int check_point(uint32_t d, uint32_t m, const uint64_t* coords) {
    if (d < 1 || m < 1 || m > 64) return ORC_EINVAL;
    if (uint64_t(d) * m > kMaxWords * 64) return ORC_ECAPACITY;
    if (m < 64)
        for (uint32_t i = 0; i < d; ++i)
            if (coords[i] >> m) return ORC_EINVAL;
    return ORC_OK;
}

// Value comparison from the most significant word (keys.hpp:50-57).
inline int key_cmp(const uint64_t* a, const uint64_t* b, uint32_t words) {
    for (uint32_t i = words; i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

struct Index {
    uint32_t d_full = 0, curves = 0, m = 0, kind = 1;
    std::vector<uint32_t> off, assign;  // per-curve slot -> input dim
    std::vector<float> rows;            // n * d_full, dataset copy (multicurves.hpp:102)
    std::vector<uint64_t> ids;
    uint64_t n = 0;
    // Per curve: sorted keys (n * W words, LS word first), ids and slots.
    std::vector<uint32_t> W;
    std::vector<std::vector<uint64_t>> keys;
    std::vector<std::vector<uint64_t>> sorted_id;
    std::vector<std::vector<uint64_t>> sorted_slot;

    uint32_t dims_of(uint32_t c) const { return off[c + 1] - off[c]; }
};

int project_key(const Index& ix, const float* v, uint32_t c, uint64_t* key) {
    uint64_t x[kMaxWords * 64];
    const uint32_t d = ix.dims_of(c);
    for (uint32_t s = 0; s < d; ++s) {
        const float comp = v[ix.assign[ix.off[c] + s]];
        if (!finite(comp)) return ORC_ENONFINITE;
        x[s] = uint64_t{ordinal_of(comp)} >> (32 - ix.m);
    }
    if (ix.kind == 1 && d > 1) hilbert_transpose(x, d, ix.m);
    bits_interleave(x, d, ix.m, key);
    return ORC_OK;
}

uint64_t rank_of(const Index& ix, uint32_t c, const uint64_t* key) {
    const uint32_t w = ix.W[c];
    const uint64_t* k = ix.keys[c].data();
    uint64_t lo = 0, hi = ix.n;  // first entry with key >= query
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (key_cmp(k + mid * w, key, w) < 0) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

void window_of(uint64_t n, uint64_t rank, uint64_t depth, uint64_t* b, uint64_t* e) {
    const uint64_t take = std::min(depth, n);
    const uint64_t below = take / 2;  // multicurves.hpp:60-62
    uint64_t begin = rank >= below ? rank - below : 0;
    uint64_t end = begin + take;
    if (end > n) {
        end = n;
        begin = n - take;
    }
    *b = begin;
    *e = end;
}

double sqdist(const float* a, const float* b, uint32_t d) {
    double acc = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
        const double t = double(a[i]) - double(b[i]);
        acc += t * t;
    }
    return acc;
}

struct Cand {
    double d;
    uint64_t id;
};
inline bool cand_less(const Cand& x, const Cand& y) {
    return x.d != y.d ? x.d < y.d : x.id < y.id;
}

uint32_t top_k(std::vector<Cand>& all, uint64_t k, uint64_t* ids, double* dist) {
    if (all.size() > k) {
        std::nth_element(all.begin(), all.begin() + k, all.end(), cand_less);
        all.resize(k);
    }
    std::sort(all.begin(), all.end(), cand_less);
    for (size_t i = 0; i < all.size(); ++i) {
        ids[i] = all[i].id;
        dist[i] = std::sqrt(all[i].d);
    }
    return uint32_t(all.size());
}

void union_of(const Index& ix, const float* q, uint64_t depth, std::vector<uint64_t>& slots) {
    slots.clear();
    uint64_t key[kMaxWords];
    for (uint32_t c = 0; c < ix.curves; ++c) {
        project_key(ix, q, c, key);
        uint64_t b, e;
        window_of(ix.n, rank_of(ix, c, key), depth, &b, &e);
        for (uint64_t p = b; p < e; ++p) slots.push_back(ix.sorted_slot[c][p]);
    }
    std::sort(slots.begin(), slots.end());
    slots.erase(std::unique(slots.begin(), slots.end()), slots.end());
}

template <class F>
void parallel_for(uint64_t count, int threads, F&& fn) {
    if (threads <= 1 || count < 2) {
        for (uint64_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (uint64_t i; (i = next.fetch_add(1)) < count;) fn(i);
        });
    for (auto& th : pool) th.join();
}

// ---- synthetic SIFT-like generator ----
inline uint64_t sm64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline uint64_t H(uint64_t s, uint64_t a, uint64_t b) {
    return sm64(s ^ sm64(a * 0x100000001b3ull ^ sm64(b)));
}
constexpr int kNC = 4096, kD = 128, kR = 12;

struct GenTables {
    std::vector<uint8_t> center;  // kNC * kD
    std::vector<int8_t> wt;       // kNC * kD * kR
    GenTables() : center(size_t(kNC) * kD), wt(size_t(kNC) * kD * kR) {
        for (int c = 0; c < kNC; ++c)
            for (int j = 0; j < kD; ++j) {
                const uint64_t h = H(1, c, j);
                center[size_t(c) * kD + j] =
                    uint8_t(((h & 255) * ((h >> 8) & 255) * ((h >> 16) & 255)) >> 16);
            }
        for (size_t t = 0; t < wt.size(); ++t) wt[t] = int8_t(int(H(6, t, 0) % 7) - 3);
    }
};
const GenTables& gen_tables() {
    static const GenTables t;
    return t;
}

void gen_row(const GenTables& g, uint64_t i, uint8_t* out) {
    const uint64_t cl = H(2, i, ~0ull) % kNC;
    int z[kR];
    for (int l = 0; l < kR; ++l) {
        const uint64_t h = H(7, i, l);
        z[l] = int(h & 15) + int((h >> 4) & 15) + int((h >> 8) & 15) + int((h >> 12) & 15) - 30;
    }
    for (int j = 0; j < kD; ++j) {
        int acc = 0;
        const int8_t* w = &g.wt[(cl * kD + j) * kR];
        for (int l = 0; l < kR; ++l) acc += w[l] * z[l];
        const uint64_t h = H(3, i, j);
        const int noise = int(h & 3) + int((h >> 2) & 3) - 3;
        const int v = int(g.center[cl * kD + j]) + (acc >> 3) + noise;
        out[j] = uint8_t(std::clamp(v, 0, 255));
    }
}

}  // namespace

extern "C" {

uint32_t orc_float_to_ordinal(float x) { return ordinal_of(x); }

int orc_quantize(float x, uint32_t m, uint64_t* out) {
    if (!finite(x)) return ORC_ENONFINITE;
    if (m < 1 || m > 32) return ORC_EINVAL;  // m>32 shifts by a negative count in curve.cpp:173
    *out = uint64_t{ordinal_of(x)} >> (32 - m);
    return ORC_OK;
}

// key: 16 words, LS word first (ExtendedKey::words layout, keys.hpp:26-27).
int orc_curve_encode(uint32_t kind, uint32_t d, uint32_t m, const uint64_t* coords, uint64_t* key) {
    const int rc = check_point(d, m, coords);
    if (rc) return rc;
    std::vector<uint64_t> x(coords, coords + d);
    if (kind == 1 && d > 1) hilbert_transpose(x.data(), d, m);
    bits_interleave(x.data(), d, m, key);
    return ORC_OK;
}

int orc_curve_decode(uint32_t kind, uint32_t d, uint32_t m, const uint64_t* key, uint64_t* coords) {
    if (d < 1 || m < 1 || m > 64) return ORC_EINVAL;
    if (uint64_t(d) * m > kMaxWords * 64) return ORC_ECAPACITY;
    bits_deinterleave(key, d, m, coords);
    if (kind == 1 && d > 1) hilbert_untranspose(coords, d, m);
    return ORC_OK;
}

// Round-robin assignment, seed 0: dim j -> curve j % C, slot j / C.
int orc_default_scheme(uint32_t d_full, uint32_t curves, uint32_t* off, uint32_t* assign) {
    if (curves < 1 || curves > d_full) return ORC_EINVAL;
    uint32_t pos = 0;
    for (uint32_t c = 0; c < curves; ++c) {
        off[c] = pos;
        for (uint32_t j = c; j < d_full; j += curves) assign[pos++] = j;
    }
    off[curves] = pos;
    return ORC_OK;
}

void* orc_build(uint32_t d_full, uint32_t curves, uint32_t m, uint32_t kind, const uint32_t* off,
                const uint32_t* assign, const float* rows, uint64_t n, const uint64_t* ids,
                int threads, int* err) {
    *err = ORC_OK;
    if (curves < 1 || m < 1 || m > 32 || kind > 1) {
        *err = ORC_EINVAL;
        return nullptr;
    }
    auto* ix = new Index;
    ix->d_full = d_full;
    ix->curves = curves;
    ix->m = m;
    ix->kind = kind;
    ix->off.assign(off, off + curves + 1);
    ix->assign.assign(assign, assign + off[curves]);
    for (uint32_t c = 0; c < curves; ++c) {
        const uint32_t d = ix->dims_of(c);
        if (d < 1 || uint64_t(d) * m > kMaxWords * 64) {
            *err = d < 1 ? ORC_EINVAL : ORC_ECAPACITY;
            delete ix;
            return nullptr;
        }
        for (uint32_t s = 0; s < d; ++s)
            if (ix->assign[ix->off[c] + s] >= d_full) {
                *err = ORC_EINVAL;
                delete ix;
                return nullptr;
            }
    }
    ix->n = n;
    ix->rows.assign(rows, rows + n * d_full);
    ix->ids.resize(n);
    for (uint64_t i = 0; i < n; ++i) ix->ids[i] = ids ? ids[i] : i;
    for (uint64_t i = 0; i < n * d_full; ++i)
        if (!finite(ix->rows[i])) {
            *err = ORC_ENONFINITE;
            delete ix;
            return nullptr;
        }
    ix->W.resize(curves);
    ix->keys.resize(curves);
    ix->sorted_id.resize(curves);
    ix->sorted_slot.resize(curves);
    parallel_for(curves, threads, [&](uint64_t cc) {
        const uint32_t c = uint32_t(cc);
        const uint32_t w = (ix->dims_of(c) * m + 63) / 64;
        ix->W[c] = w;
        std::vector<uint64_t> raw(n * w);
        uint64_t key[kMaxWords];
        for (uint64_t i = 0; i < n; ++i) {
            project_key(*ix, &ix->rows[i * d_full], c, key);
            std::memcpy(&raw[i * w], key, w * 8);
        }
        std::vector<uint64_t> perm(n);
        for (uint64_t i = 0; i < n; ++i) perm[i] = i;
        std::sort(perm.begin(), perm.end(), [&](uint64_t a, uint64_t b) {
            const int o = key_cmp(&raw[a * w], &raw[b * w], w);
            return o != 0 ? o < 0 : ix->ids[a] < ix->ids[b];
        });
        auto& K = ix->keys[c];
        K.resize(n * w);
        ix->sorted_id[c].resize(n);
        ix->sorted_slot[c].resize(n);
        for (uint64_t p = 0; p < n; ++p) {
            std::memcpy(&K[p * w], &raw[perm[p] * w], w * 8);
            ix->sorted_id[c][p] = ix->ids[perm[p]];
            ix->sorted_slot[c][p] = perm[p];
        }
    });
    return ix;
}

void orc_free(void* h) { delete static_cast<Index*>(h); }
uint64_t orc_size(void* h) { return static_cast<Index*>(h)->n; }
uint32_t orc_key_words(void* h, uint32_t c) { return static_cast<Index*>(h)->W[c]; }

void orc_sorted(void* h, uint32_t c, uint64_t* keys_out, uint64_t* ids_out) {
    const Index& ix = *static_cast<Index*>(h);
    if (keys_out) std::memcpy(keys_out, ix.keys[c].data(), ix.keys[c].size() * 8);
    if (ids_out) std::memcpy(ids_out, ix.sorted_id[c].data(), ix.n * 8);
}

int orc_query_key(void* h, const float* q, uint32_t c, uint64_t* key16) {
    return project_key(*static_cast<Index*>(h), q, c, key16);
}

uint64_t orc_rank(void* h, uint32_t c, const uint64_t* key) {
    return rank_of(*static_cast<Index*>(h), c, key);
}

// Per query x curve: rank, begin, end (queries row-major, nq x d_full).
int orc_windows(void* h, const float* qs, uint64_t nq, uint64_t depth, uint64_t* rank_out,
                uint64_t* begin_out, uint64_t* end_out) {
    const Index& ix = *static_cast<Index*>(h);
    uint64_t key[kMaxWords];
    for (uint64_t qi = 0; qi < nq; ++qi)
        for (uint32_t c = 0; c < ix.curves; ++c) {
            const int rc = project_key(ix, qs + qi * ix.d_full, c, key);
            if (rc) return rc;
            const uint64_t r = rank_of(ix, c, key);
            const uint64_t o = qi * ix.curves + c;
            rank_out[o] = r;
            window_of(ix.n, r, depth, &begin_out[o], &end_out[o]);
        }
    return ORC_OK;
}

// Sorted unique candidate ids of one query; returns the count.
uint64_t orc_candidates(void* h, const float* q, uint64_t depth, uint64_t* out) {
    const Index& ix = *static_cast<Index*>(h);
    std::vector<uint64_t> slots;
    union_of(ix, q, depth, slots);
    std::vector<uint64_t> ids(slots.size());
    for (size_t i = 0; i < slots.size(); ++i) ids[i] = ix.ids[slots[i]];
    std::sort(ids.begin(), ids.end());
    if (out) std::memcpy(out, ids.data(), ids.size() * 8);
    return ids.size();
}

int orc_search(void* h, const float* qs, uint64_t nq, uint64_t k, uint64_t depth,
               uint64_t* out_ids, double* out_dist, uint32_t* out_len, int threads) {
    const Index& ix = *static_cast<Index*>(h);
    if (k < 1 || depth < 1) return ORC_EINVAL;
    for (uint64_t i = 0; i < nq * ix.d_full; ++i)
        if (!finite(qs[i])) return ORC_ENONFINITE;
    parallel_for(nq, threads, [&](uint64_t qi) {
        const float* q = qs + qi * ix.d_full;
        std::vector<uint64_t> slots;
        union_of(ix, q, depth, slots);
        std::vector<Cand> all;
        all.reserve(slots.size());
        for (uint64_t s : slots) all.push_back({sqdist(q, &ix.rows[s * ix.d_full], ix.d_full), ix.ids[s]});
        out_len[qi] = top_k(all, k, out_ids + qi * k, out_dist + qi * k);
    });
    return ORC_OK;
}

int orc_brute_force(const float* rows, const uint64_t* ids, uint64_t n, uint32_t dim,
                    const float* qs, uint64_t nq, uint64_t k, uint64_t* out_ids, double* out_dist,
                    uint32_t* out_len, int threads) {
    if (k < 1) return ORC_EINVAL;
    parallel_for(nq, threads, [&](uint64_t qi) {
        std::vector<Cand> all(n);
        for (uint64_t i = 0; i < n; ++i)
            all[i] = {sqdist(qs + qi * dim, rows + i * dim, dim), ids ? ids[i] : i};
        out_len[qi] = top_k(all, k, out_ids + qi * k, out_dist + qi * k);
    });
    return ORC_OK;
}

void orc_gen_rows_strided(uint64_t first, uint64_t stride, uint64_t count, uint8_t* out, int threads) {
    const GenTables& g = gen_tables();
    const uint64_t chunk = 4096;
    parallel_for((count + chunk - 1) / chunk, threads, [&](uint64_t b) {
        const uint64_t e = std::min(count, (b + 1) * chunk);
        for (uint64_t i = b * chunk; i < e; ++i) gen_row(g, first + i * stride, out + i * kD);
    });
}

// Rows of arbitrary generator ids (the certificate checks of tools/certify.py
// regenerate exactly the rows a window touches).
void orc_gen_rows_ids(const uint64_t* ids, uint64_t count, uint8_t* out, int threads) {
    const GenTables& g = gen_tables();
    const uint64_t chunk = 1024;
    parallel_for((count + chunk - 1) / chunk, threads, [&](uint64_t b) {
        const uint64_t e = std::min(count, (b + 1) * chunk);
        for (uint64_t i = b * chunk; i < e; ++i) gen_row(g, ids[i], out + i * kD);
    });
}

// Full keys (W words, LS word first) of n arbitrary float rows on curve c of
// an index's scheme (curve.cpp:162-164 over multicurves.hpp:40's projection).
int orc_keys_batch(void* h, const float* rows, uint64_t n, uint32_t c, uint64_t* keys_out) {
    const Index& ix = *static_cast<Index*>(h);
    const uint32_t w = ix.W[c];
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t key[kMaxWords] = {};
        const int rc = project_key(ix, rows + i * ix.d_full, c, key);
        if (rc != ORC_OK) return rc;
        std::memcpy(keys_out + i * w, key, 8 * w);
    }
    return ORC_OK;
}

void orc_gen_rows(uint64_t i0, uint64_t count, uint8_t* out, int threads) {
    orc_gen_rows_strided(i0, 1, count, out, threads);
}

// Queries perturb database row H(4,q,~0) % n_db.
void orc_gen_queries(uint64_t q0, uint64_t count, uint64_t n_db, uint8_t* out, int threads) {
    const GenTables& g = gen_tables();
    parallel_for(count, threads, [&](uint64_t i) {
        const uint64_t q = q0 + i;
        uint8_t base[kD];
        gen_row(g, H(4, q, ~0ull) % n_db, base);
        for (int j = 0; j < kD; ++j) {
            const uint64_t h = H(5, q, j);
            const int v = int(base[j]) + int(h & 15) + int((h >> 4) & 15) - 15;
            out[i * kD + j] = uint8_t(std::clamp(v, 0, 255));
        }
    });
}

}  // extern "C"
