// api.cu -- host side of the C ABI declared in include/hcg.h.
//
// Owns device memory of an index, stages host buffers, validates the
// reference's preconditions and turns them into status codes (the C++ wrapper
// turns the codes back into the reference's exceptions).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hcg_host.hpp"
#include "hcg_internal.cuh"

struct hcg_index {
    int device = 0;
    uint32_t d_full = 0, pitch = 0, C = 0, m = 0, kind = 0;
    uint32_t dtype = HCG_U8, row_bytes = 0;  // row_bytes = d_full * element size
    double dist_scale = 1.0;
    float view_offset = 0.0f;
    uint64_t n = 0, id_base = 0, id_stride = 1;
    std::vector<uint32_t> off, assign;
    uint32_t lut[256] = {};
    int dmax = 8, wsmax = 1;
    uint8_t* rows = nullptr;
    uint32_t* idtab = nullptr;  // physical row -> id slot (rows stored in curve-0 order); null: identity
    uint32_t* d_lut = nullptr;
    uint16_t* d_assign = nullptr;
    std::vector<hcg::CurveDev> curves;
    hcg::CurveDev* d_curves = nullptr;
    std::vector<uint64_t*> keys;
    std::vector<uint32_t*> slots;
    std::vector<uint64_t*> samples;  // per curve: every kSampleStride-th key (locate's upper levels)
    std::vector<uint64_t> sample_bytes;
    uint32_t** d_slot_ptrs = nullptr;
    uint64_t bytes = 0;
    bool broken = false;  // a failed table upload after an insert: every call is refused
    bool dims16 = false;  // every curve has exactly 16 dims (the default scheme at d = 128, C = 8)
};

namespace hcg {

namespace {
thread_local std::string g_err;
}

hcg_status set_error(hcg_status code, const std::string& msg) {
    g_err = msg;
    return code;
}

namespace {
std::atomic<unsigned long long> g_launches{0};
}
void count_launches(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

hcg_status check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(HCG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return HCG_OK;
}

namespace {

#define HCG_TRY_CUDA(call)                                                                          \
    do {                                                                                            \
        const cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return set_error(HCG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define HCG_TRY(call)                       \
    do {                                    \
        const hcg_status r_ = (call);       \
        if (r_ != HCG_OK) return r_;        \
    } while (0)

// Keep stream-ordered scratch cached in the device's default pool: with the
// default release threshold (0) every synchronise hands the memory back and
// the next call re-maps it, which dominates small-batch latency.
void keep_pool(int dev) {
    static bool done[64] = {};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    done[dev] = true;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
        keep_pool(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Stream-ordered scratch, released (stream-ordered) when the call returns.
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

uint32_t round16(uint32_t x) { return (x + 15u) & ~15u; }

// Device copy of nrows x d_full bytes with row pitch `pitch` (zero padded).
hcg_status stage_rows(Scratch& sc, const uint8_t* src, uint64_t nrows, uint32_t d_full, uint32_t pitch,
                      const uint8_t** out) {
    if (nrows == 0) {
        *out = nullptr;
        return HCG_OK;
    }
    if (pitch == d_full && is_device_ptr(src) && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        *out = src;
        return HCG_OK;
    }
    uint8_t* d = sc.alloc<uint8_t>(size_t(nrows) * pitch);
    if (!d) return set_error(HCG_ENOMEM, "query staging buffer");
    if (pitch != d_full) HCG_TRY_CUDA(cudaMemsetAsync(d, 0, size_t(nrows) * pitch, sc.st));
    HCG_TRY_CUDA(cudaMemcpy2DAsync(d, pitch, src, d_full, d_full, nrows, cudaMemcpyDefault, sc.st));
    *out = d;
    return HCG_OK;
}

template <class T>
struct OutBuf {
    T* user = nullptr;
    T* dev = nullptr;
    size_t count = 0;
    bool host = false;
};

template <class T>
hcg_status stage_out(Scratch& sc, T* user, size_t count, OutBuf<T>* o) {
    o->user = user;
    o->count = count;
    o->host = user && !is_device_ptr(user);
    o->dev = o->host ? sc.alloc<T>(count) : user;
    if (user && !o->dev) return set_error(HCG_ENOMEM, "output staging buffer");
    return HCG_OK;
}

template <class T>
hcg_status finish_out(Scratch& sc, const OutBuf<T>& o) {
    if (o.host && o.count)
        HCG_TRY_CUDA(cudaMemcpyAsync(o.user, o.dev, o.count * sizeof(T), cudaMemcpyDeviceToHost, sc.st));
    return HCG_OK;
}

uint32_t ordinal_of(float x) {
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    return (bits >> 31) ? ~bits : (bits | 0x80000000u);
}

int pow2_bucket(uint32_t v, int lo, int hi) {
    int b = lo;
    while (b < int(v) && b < hi) b <<= 1;
    return b;
}

hcg_status check_index(const hcg_index* ix) {
    if (!ix) return set_error(HCG_EINVAL, "null index");
    if (ix->broken) return set_error(HCG_ECUDA, "index unusable after a failed device table upload");
    return HCG_OK;
}

void release(hcg_index* ix) {
    if (!ix) return;
    DeviceGuard g(ix->device);
    cudaFree(ix->rows);
    cudaFree(ix->idtab);
    cudaFree(ix->d_lut);
    cudaFree(ix->d_assign);
    cudaFree(ix->d_curves);
    cudaFree(ix->d_slot_ptrs);
    for (auto* p : ix->keys) cudaFree(p);
    for (auto* p : ix->slots) cudaFree(p);
    for (auto* p : ix->samples) cudaFree(p);
    delete ix;
}

template <class T>
hcg_status dev_alloc(T** p, size_t count, uint64_t* bytes) {
    const size_t b = std::max<size_t>(count, 1) * sizeof(T);
    if (cudaMalloc(reinterpret_cast<void**>(p), b) != cudaSuccess) {
        cudaGetLastError();
        return set_error(HCG_ENOMEM, "device allocation of " + std::to_string(b) + " bytes failed");
    }
    *bytes += b;
    return HCG_OK;
}

hcg_status validate_scheme(const hcg_scheme* s) {
    if (!s) return set_error(HCG_EINVAL, "null scheme");
    if (s->dtype > HCG_F32) return set_error(HCG_EINVAL, "unknown descriptor dtype");
    const uint32_t esize = s->dtype == HCG_F32 ? 4 : 1;
    if (s->d_full < 1 || uint64_t(s->d_full) * esize > HCG_MAX_ROW_BYTES)
        return set_error(HCG_ECAPACITY, "d_full must be in [1, " + std::to_string(HCG_MAX_ROW_BYTES / esize) + "]");
    if (s->curves < 1 || s->curves > s->d_full) return set_error(HCG_EINVAL, "curves must be in [1, d_full]");
    if (s->bits_per_dim < 1 || s->bits_per_dim > 32) return set_error(HCG_EINVAL, "bits_per_dim out of range [1,32]");
    if (s->curve_kind > 1) return set_error(HCG_EINVAL, "unknown curve kind");
    if (!s->assign_off || !s->assign) return set_error(HCG_EINVAL, "null assignment");
    if (!(s->dist_scale > 0.0) || !std::isfinite(s->dist_scale)) return set_error(HCG_EINVAL, "dist_scale must be > 0");
    std::vector<bool> covered(s->d_full, false);
    for (uint32_t c = 0; c < s->curves; ++c) {
        if (s->assign_off[c + 1] < s->assign_off[c]) return set_error(HCG_EINVAL, "assignment offsets not monotone");
        const uint32_t d = s->assign_off[c + 1] - s->assign_off[c];
        if (d < 1) return set_error(HCG_EINVAL, "curve with no dimensions");
        if (uint64_t(d) * s->bits_per_dim > HCG_MAX_KEY_BITS)
            return set_error(HCG_ECAPACITY, "key width " + std::to_string(uint64_t(d) * s->bits_per_dim) +
                                                " exceeds capacity " + std::to_string(HCG_MAX_KEY_BITS));
        if (d > HCG_MAX_CURVE_DIMS) return set_error(HCG_ECAPACITY, "more than 128 dimensions on one curve");
        for (uint32_t i = s->assign_off[c]; i < s->assign_off[c + 1]; ++i) {
            if (s->assign[i] >= s->d_full) return set_error(HCG_EINVAL, "assignment out of range");
            covered[s->assign[i]] = true;
        }
    }
    for (bool cv : covered)
        if (!cv) return set_error(HCG_EINVAL, "input dimension not covered by any curve");
    if (s->dtype == HCG_F32) return HCG_OK;  // cells computed on the device; the table is unused
    // A u8 index scores the integer S = sum (b1 - b2)^2 and reports
    // sqrt(S) * scale.  That equals the reference's sqrt of its double sum
    // (vecio.cpp:87-95) over the floats offset + b * scale exactly when those
    // floats are exact and scale is a power of two (then every term, partial
    // sum and the root scale without rounding).  Other views are rejected.
    int e2 = 0;
    if (std::frexp(s->dist_scale, &e2) != 0.5)
        return set_error(HCG_EINVAL, "u8 view: dist_scale must be a power of two (exact rooted distances)");
    const float voff = std::isfinite(s->view_offset) ? s->view_offset : 0.0f;
    for (int b = 0; b < 256; ++b) {
        const double v = double(voff) + double(b) * s->dist_scale;
        if (double(float(v)) != v)
            return set_error(HCG_EINVAL, "u8 view: offset + b * scale is not exact in float32 for b = " + std::to_string(b));
    }
    const uint64_t lim = s->bits_per_dim == 32 ? (1ull << 32) : (1ull << s->bits_per_dim);
    for (int b = 0; b < 256; ++b)
        if (s->cell_lut[b] >= lim) return set_error(HCG_EINVAL, "cell_lut entry exceeds 2^m");
    return HCG_OK;
}

hcg_status check_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_error(HCG_ENODEV, "no CUDA device");
    }
    if (device < 0 || device >= count) return set_error(HCG_ENODEV, "device ordinal out of range");
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major != 10) return set_error(HCG_ENODEV, "this build targets sm_100a (B200) only");
    return HCG_OK;
}

// Keys of `count` rows (K1) as SoA words plus their OR / AND over all rows.
hcg_status keygen_reduce(const hcg_index* ix, uint32_t c, const uint8_t* rows, uint64_t count, Scratch& sc,
                         uint64_t** soa, std::vector<uint64_t>& oa) {
    const uint32_t d = ix->off[c + 1] - ix->off[c];
    const uint32_t W = (d * ix->m + 63) / 64;
    *soa = sc.alloc<uint64_t>(size_t(W) * count);
    unsigned long long* or_and = sc.alloc<unsigned long long>(2 * W + 1);  // + the non-finite flag
    if (!*soa || !or_and) return set_error(HCG_ENOMEM, "key buffers");
    HCG_TRY_CUDA(cudaMemsetAsync(or_and, 0, W * 8, sc.st));
    HCG_TRY_CUDA(cudaMemsetAsync(or_and + W, 0xFF, W * 8, sc.st));
    HCG_TRY_CUDA(cudaMemsetAsync(or_and + 2 * W, 0, 8, sc.st));
    HCG_TRY(keygen_rows(rows, count, ix->pitch, ix->d_assign + ix->off[c], int(d), int(ix->m), int(ix->kind),
                        ix->d_lut, *soa, int(W), or_and, ix->dmax, int(ix->dtype),
                        reinterpret_cast<unsigned*>(or_and + 2 * W), sc.st));
    oa.assign(2 * W + 1, 0);
    HCG_TRY_CUDA(cudaMemcpyAsync(oa.data(), or_and, (2 * W + 1) * 8, cudaMemcpyDeviceToHost, sc.st));
    HCG_TRY_CUDA(cudaStreamSynchronize(sc.st));
    const bool bad = oa[2 * W] != 0;
    oa.resize(2 * W);
    if (bad) return set_error(HCG_ENONFINITE, "non-finite component");
    return HCG_OK;
}

// K2: stable LSD radix sort of `count` keys (SoA, W words) by their bits
// [0, hv] (only the 8-bit digits that vary over `oa`), then pack the sorted
// suffixes (AoS, ws words) into *keys_out and slot_base + position into
// *slots_out (both allocated here; their bytes are added to *bytes).
// init_order (optional): the sort's input sequence as positions into soa --
// the id order of a physically permuted index, so that equal keys stay in id
// order and the output holds physical positions.
hcg_status sort_suffix(uint64_t* bytes, const uint64_t* soa, uint64_t count, uint32_t W, const std::vector<uint64_t>& oa,
                       uint32_t hv, uint64_t slot_base, Scratch& sc, uint64_t** keys_out, uint32_t** slots_out,
                       const uint32_t* init_order = nullptr) {
    const int hw = int(hv >> 6), hb = int(hv & 63);
    const uint64_t below = hb == 63 ? ~0ull : ((2ull << hb) - 1);
    const uint32_t ws = uint32_t(hw + 1);
    cudaStream_t st = sc.st;
    uint64_t* kb = sc.alloc<uint64_t>(count);
    uint64_t* ka = sc.alloc<uint64_t>(count);
    uint32_t* va = sc.alloc<uint32_t>(count);
    uint32_t* vb = sc.alloc<uint32_t>(count);
    uint32_t* counts = reinterpret_cast<uint32_t*>(sc.alloc<uint8_t>(radix_counts_bytes(count)));
    if (!kb || !ka || !va || !vb || !counts) return set_error(HCG_ENOMEM, "sort buffers");
    uint32_t* totals = counts + (radix_counts_bytes(count) / 4 - 256);
    uint32_t* v = vb;
    uint32_t* v_alt = va;
    if (init_order)
        HCG_TRY_CUDA(cudaMemcpyAsync(v, init_order, count * 4, cudaMemcpyDeviceToDevice, st));
    else
        launch_iota(v, count, 0, st);
    for (uint32_t w = 0; w <= uint32_t(hw); ++w) {
        uint64_t vary = oa[w] ^ oa[W + w];
        if (int(w) == hw) vary &= below;
        uint32_t dmask = 0;
        for (int sft = 0; sft < 8; ++sft)
            if ((vary >> (8 * sft)) & 0xFF) dmask |= 1u << sft;
        if (!dmask) continue;
        launch_gather_word(soa + uint64_t(w) * count, v, kb, count, st);
        uint64_t* k = kb;
        uint64_t* k_alt = ka;
        HCG_TRY(radix_sort_pairs(&k, &v, &k_alt, &v_alt, count, dmask, counts, totals, st));
        kb = k;
        ka = k_alt;
    }
    HCG_TRY(dev_alloc(keys_out, size_t(count) * ws, bytes));
    HCG_TRY(dev_alloc(slots_out, count, bytes));
    launch_pack_suffix(soa, v, count, int(ws), below, *keys_out, st);
    launch_offset(v, *slots_out, count, uint32_t(slot_base), st);
    return check_launch("pack suffix");
}

void dev_free(void* p, size_t bytes, uint64_t* total) {
    if (p) {
        cudaFree(p);
        *total -= std::min<uint64_t>(*total, bytes);
    }
}

// A curve's sorted arrays under construction: nothing of the index changes
// until every curve of a build / insert succeeded (then commit_curve swaps
// them in); on failure drop() frees them.
struct CurveOut {
    uint64_t* keys = nullptr;
    uint32_t* slots = nullptr;
    CurveDev cv{};
    uint64_t n = 0;
    uint64_t bytes = 0;
    void drop() {
        dev_free(keys, size_t(n) * cv.ws * 8, &bytes);
        dev_free(slots, size_t(n) * 4, &bytes);
        keys = nullptr;
        slots = nullptr;
    }
};

// Curve c over `n` rows (`rows`, the index's pitch): K1 keys, common-prefix
// detection, K2 sort.
hcg_status build_curve_into(const hcg_index* ix, uint32_t c, const uint8_t* rows, uint64_t n, cudaStream_t st,
                            const uint32_t* init_order, CurveOut* out) {
    const uint32_t d = ix->off[c + 1] - ix->off[c];
    const uint32_t W = (d * ix->m + 63) / 64;
    CurveDev& cv = out->cv;
    std::memset(&cv, 0, sizeof(cv));
    cv.w = W;
    cv.dims = d;
    cv.off = ix->off[c];
    cv.ws = 1;
    out->n = n;
    if (n == 0) return HCG_OK;
    Scratch sc(st);
    uint64_t* soa = nullptr;
    std::vector<uint64_t> oa;
    HCG_TRY(keygen_reduce(ix, c, rows, n, sc, &soa, oa));
    int hv = 0;
    for (int w = int(W) - 1; w >= 0; --w) {
        const uint64_t vary = oa[w] ^ oa[W + w];
        if (vary) {
            hv = 64 * w + 63 - __builtin_clzll(vary);
            break;
        }
    }
    const int hw = hv >> 6, hb = hv & 63;
    const uint64_t above = hb == 63 ? 0ull : (~0ull << (hb + 1));
    cv.hv = uint32_t(hv);
    cv.ws = uint32_t(hw + 1);
    for (uint32_t w = 0; w < W; ++w)
        cv.prefix[w] = int(w) > hw ? oa[w] : (int(w) == hw ? (oa[w] & above) : 0ull);
    HCG_TRY(sort_suffix(&out->bytes, soa, n, W, oa, cv.hv, 0, sc, &out->keys, &out->slots, init_order));
    cv.keys = out->keys;
    cv.slots = out->slots;
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return HCG_OK;
}

// Swap a finished curve into the index (frees the curve's previous arrays).
void commit_curve(hcg_index* ix, uint32_t c, uint64_t n_prev, CurveOut& o) {
    dev_free(ix->keys[c], size_t(n_prev) * ix->curves[c].ws * 8, &ix->bytes);
    dev_free(ix->slots[c], size_t(n_prev) * 4, &ix->bytes);
    ix->keys[c] = o.keys;
    ix->slots[c] = o.slots;
    ix->curves[c] = o.cv;
    ix->bytes += o.bytes;
    o.keys = nullptr;
    o.slots = nullptr;
    o.bytes = 0;
}

hcg_status build_curve(hcg_index* ix, uint32_t c, cudaStream_t st) {
    CurveOut o;
    const hcg_status rc = build_curve_into(ix, c, ix->rows, ix->n, st, nullptr, &o);
    if (rc != HCG_OK) {
        cudaStreamSynchronize(st);
        o.drop();
        return rc;
    }
    commit_curve(ix, c, 0, o);
    return HCG_OK;
}

// Curve c after appending `nb` rows to the index's n_old: `rows` is the new
// n_old + nb row buffer, `idtab` the new id table (null: identity).  When the
// new keys share the curve's common prefix they are sorted on their own and
// rank-merged into the resident arrays (stable: resident entries first on
// equal keys, i.e. id order); otherwise the curve is rebuilt over all rows.
// The index itself is not modified.
hcg_status insert_curve_into(const hcg_index* ix, uint32_t c, const uint8_t* rows, uint64_t n_old, uint64_t nb,
                             const uint32_t* idtab, cudaStream_t st, CurveOut* out) {
    const uint64_t n_new = n_old + nb;
    if (n_old == 0) return build_curve_into(ix, c, rows, n_new, st, nullptr, out);
    const CurveDev& cv = ix->curves[c];
    const uint32_t W = cv.w;
    Scratch sc(st);
    uint64_t* soa = nullptr;
    std::vector<uint64_t> oa;
    HCG_TRY(keygen_reduce(ix, c, rows + uint64_t(n_old) * ix->pitch, nb, sc, &soa, oa));
    const int hw = int(cv.hv >> 6), hb = int(cv.hv & 63);
    const uint64_t above = hb == 63 ? 0ull : (~0ull << (hb + 1));
    bool compatible = true;
    for (uint32_t w = uint32_t(hw); w < W; ++w) {
        const uint64_t m = int(w) == hw ? above : ~0ull;
        if ((oa[w] & m) != cv.prefix[w] || (oa[W + w] & m) != cv.prefix[w]) compatible = false;
    }
    if (!compatible) {
        if (!idtab) return build_curve_into(ix, c, rows, n_new, st, nullptr, out);
        // permuted rows: sort in id order (inverse of idtab) so ties keep id order
        uint32_t* inv = sc.alloc<uint32_t>(n_new);
        if (!inv) return set_error(HCG_ENOMEM, "inverse permutation");
        launch_invert(idtab, n_new, inv, st);
        HCG_TRY(check_launch("invert"));
        return build_curve_into(ix, c, rows, n_new, st, inv, out);
    }
    uint64_t tmp_bytes = 0;
    uint64_t* nk = nullptr;
    uint32_t* ns = nullptr;
    hcg_status rc = sort_suffix(&tmp_bytes, soa, nb, W, oa, cv.hv, n_old, sc, &nk, &ns);
    out->cv = cv;
    out->n = n_new;
    if (rc == HCG_OK) rc = dev_alloc(&out->keys, size_t(n_new) * cv.ws, &out->bytes);
    if (rc == HCG_OK) rc = dev_alloc(&out->slots, n_new, &out->bytes);
    if (rc == HCG_OK) {
        launch_rank_merge(ix->keys[c], ix->slots[c], n_old, nk, ns, nb, int(cv.ws), out->keys, out->slots, st);
        rc = check_launch("rank merge");
    }
    if (rc == HCG_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = set_error(HCG_ECUDA, "rank merge");
    cudaStreamSynchronize(st);
    dev_free(nk, size_t(nb) * cv.ws * 8, &tmp_bytes);
    dev_free(ns, size_t(nb) * 4, &tmp_bytes);
    out->cv.keys = out->keys;
    out->cv.slots = out->slots;
    return rc;
}

// Upload the curve table and slot pointers (after build / insert / load).
// Store the descriptors in curve-0 key order: rows that are near on curve 0
// (and, through the data's clusters, on the other curves) become neighbours
// in HBM, so a query's candidate rows share DRAM pages and L2 lines
// (measured: gather 5.94 -> 5.05 ms at 10M).  Ids do not move: idtab maps a
// physical row to its id slot, the curves' slot arrays are remapped to
// physical rows (their (key, id) order is unchanged), and the search reads
// idtab only for candidates that can enter a top-k (tie order by id).
hcg_status reorder_rows(hcg_index* ix, cudaStream_t st) {
    static const bool off = knob("HCG_NO_REORDER") != nullptr;
    const uint64_t n = ix->n;
    if (off || n < 2 || ix->idtab) return HCG_OK;
    uint8_t* nr = nullptr;
    uint32_t* idt = nullptr;
    HCG_TRY(dev_alloc(&nr, size_t(n) * ix->pitch, &ix->bytes));
    if (dev_alloc(&idt, n, &ix->bytes) != HCG_OK) {
        dev_free(nr, size_t(n) * ix->pitch, &ix->bytes);
        return set_error(HCG_ENOMEM, "id table");
    }
    Scratch sc(st);
    uint32_t* inv = sc.alloc<uint32_t>(n);
    if (!inv) {
        dev_free(nr, size_t(n) * ix->pitch, &ix->bytes);
        dev_free(idt, size_t(n) * 4, &ix->bytes);
        return set_error(HCG_ENOMEM, "inverse permutation");
    }
    const uint32_t* perm = ix->slots[0];  // id slots in curve-0 order
    HCG_TRY_CUDA(cudaMemcpyAsync(idt, perm, n * 4, cudaMemcpyDeviceToDevice, st));
    launch_permute_rows(ix->rows, perm, n, ix->pitch, nr, st);
    launch_invert(perm, n, inv, st);
    for (uint32_t c = 0; c < ix->C; ++c) launch_map(ix->slots[c], n, inv, st);
    HCG_TRY(check_launch("reorder rows"));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    dev_free(ix->rows, size_t(n) * ix->pitch, &ix->bytes);
    ix->rows = nr;
    ix->idtab = idt;
    return HCG_OK;
}

hcg_status publish_tables(hcg_index* ix, cudaStream_t st) {
    // sampled keys for the two-level lower_bound (derived data, rebuilt here)
    ix->samples.resize(ix->C, nullptr);
    ix->sample_bytes.resize(ix->C, 0);
    for (uint32_t c = 0; c < ix->C; ++c) {
        CurveDev& cv = ix->curves[c];
        dev_free(ix->samples[c], ix->sample_bytes[c], &ix->bytes);
        ix->samples[c] = nullptr;
        ix->sample_bytes[c] = 0;
        cv.samples = nullptr;
        cv.n_samples = 0;
        static const uint32_t stride = knob("HCG_SAMPLE_STRIDE") ? uint32_t(atoi(knob("HCG_SAMPLE_STRIDE")))
                                                                   : kSampleStride;
        if (stride < 2 || ix->n < 4 * uint64_t(stride) || !ix->keys[c]) continue;
        const uint64_t ns = (ix->n + stride - 1) / stride;
        HCG_TRY(dev_alloc(&ix->samples[c], size_t(ns) * cv.ws, &ix->bytes));
        ix->sample_bytes[c] = size_t(ns) * cv.ws * 8;
        cv.sample_stride = stride;
        launch_sample(ix->keys[c], ns, cv.ws, stride, ix->samples[c], st);
        HCG_TRY(check_launch("key samples"));
        cv.samples = ix->samples[c];
        cv.n_samples = uint32_t(ns);
    }
    uint32_t maxws = 1;
    for (auto& cv : ix->curves) maxws = std::max(maxws, cv.ws);
    ix->wsmax = pow2_bucket(maxws, 1, 16);
    if (!ix->d_curves) HCG_TRY(dev_alloc(&ix->d_curves, ix->C, &ix->bytes));
    if (!ix->d_slot_ptrs) HCG_TRY(dev_alloc(&ix->d_slot_ptrs, ix->C, &ix->bytes));
    HCG_TRY_CUDA(cudaMemcpyAsync(ix->d_curves, ix->curves.data(), sizeof(CurveDev) * ix->C, cudaMemcpyHostToDevice, st));
    HCG_TRY_CUDA(cudaMemcpyAsync(ix->d_slot_ptrs, ix->slots.data(), sizeof(uint32_t*) * ix->C, cudaMemcpyHostToDevice,
                                 st));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return HCG_OK;
}

// Allocate an index for `s` with room for n rows (rows buffer allocated,
// scheme uploaded); curves are filled by the caller (build / load).
hcg_status new_index(const hcg_scheme* s, uint64_t n, uint64_t id_base, uint64_t id_stride, int device, cudaStream_t st,
                     hcg_index** out) {
    auto* ix = new hcg_index;
    ix->device = device;
    ix->d_full = s->d_full;
    ix->dtype = s->dtype;
    ix->row_bytes = s->d_full * (s->dtype == HCG_F32 ? 4 : 1);
    ix->pitch = round16(ix->row_bytes);
    ix->C = s->curves;
    ix->m = s->bits_per_dim;
    ix->kind = s->curve_kind;
    ix->dist_scale = s->dist_scale;
    ix->view_offset = std::isfinite(s->view_offset) ? s->view_offset : 0.0f;
    ix->n = n;
    ix->id_base = id_base;
    ix->id_stride = id_stride;
    ix->off.assign(s->assign_off, s->assign_off + s->curves + 1);
    ix->assign.assign(s->assign, s->assign + ix->off[s->curves]);
    std::memcpy(ix->lut, s->cell_lut, sizeof(ix->lut));
    uint32_t maxd = 1;
    for (uint32_t c = 0; c < ix->C; ++c) maxd = std::max(maxd, ix->off[c + 1] - ix->off[c]);
    ix->dmax = pow2_bucket(maxd, 8, 128);
    ix->dims16 = true;
    for (uint32_t c = 0; c < ix->C; ++c) ix->dims16 = ix->dims16 && ix->off[c + 1] - ix->off[c] == 16;
    ix->curves.resize(ix->C);
    for (uint32_t c = 0; c < ix->C; ++c) {
        CurveDev& cv = ix->curves[c];
        std::memset(&cv, 0, sizeof(cv));
        cv.dims = ix->off[c + 1] - ix->off[c];
        cv.w = (cv.dims * ix->m + 63) / 64;
        cv.ws = 1;
        cv.off = ix->off[c];
    }
    ix->keys.assign(ix->C, nullptr);
    ix->slots.assign(ix->C, nullptr);
    hcg_status rc = dev_alloc(&ix->rows, size_t(n) * ix->pitch, &ix->bytes);
    if (rc == HCG_OK) rc = dev_alloc(&ix->d_lut, 256, &ix->bytes);
    if (rc == HCG_OK) rc = dev_alloc(&ix->d_assign, ix->assign.size(), &ix->bytes);
    std::vector<uint16_t> asg16(ix->assign.begin(), ix->assign.end());
    if (rc == HCG_OK &&
        (cudaMemcpyAsync(ix->d_lut, ix->lut, sizeof(ix->lut), cudaMemcpyHostToDevice, st) != cudaSuccess ||
         cudaMemcpyAsync(ix->d_assign, asg16.data(), asg16.size() * 2, cudaMemcpyHostToDevice, st) != cudaSuccess ||
         cudaStreamSynchronize(st) != cudaSuccess))
        rc = set_error(HCG_ECUDA, "copy scheme");
    if (rc != HCG_OK) {
        release(ix);
        return rc;
    }
    *out = ix;
    return HCG_OK;
}

// +inf distances for empty f32 result lists.
hcg_status fill_inf(double* p, size_t count, cudaStream_t st) {
    if (!count) return HCG_OK;
    const std::vector<double> h(count, HUGE_VAL);
    HCG_TRY_CUDA(cudaMemcpyAsync(p, h.data(), count * 8, cudaMemcpyHostToDevice, st));
    return cudaStreamSynchronize(st) == cudaSuccess ? HCG_OK : set_error(HCG_ECUDA, "fill");
}

hcg_status check_search_args(const hcg_index* ix, uint32_t k, uint32_t depth) {
    HCG_TRY(check_index(ix));
    if (k < 1) return set_error(HCG_EINVAL, "k must be >= 1");
    if (k > HCG_MAX_K) return set_error(HCG_ECAPACITY, "k exceeds HCG_MAX_K");
    if (depth < 1) return set_error(HCG_EINVAL, "probe_depth must be >= 1");
    return HCG_OK;
}

// Non-finite query flag (f32 indexes): cleared before locate, checked by
// check_queries() after it (the reference throws on NaN / Inf components).
struct QueryFlag {
    unsigned* dev = nullptr;
};

hcg_status make_flag(const hcg_index* ix, Scratch& sc, QueryFlag* f) {
    if (ix->dtype != HCG_F32) return HCG_OK;
    f->dev = sc.alloc<unsigned>(1);
    if (!f->dev) return set_error(HCG_ENOMEM, "flag");
    HCG_TRY_CUDA(cudaMemsetAsync(f->dev, 0, 4, sc.st));
    return HCG_OK;
}

hcg_status check_flag(const QueryFlag& f, cudaStream_t st) {
    if (!f.dev) return HCG_OK;
    unsigned h = 0;
    HCG_TRY_CUDA(cudaMemcpyAsync(&h, f.dev, 4, cudaMemcpyDeviceToHost, st));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return h ? set_error(HCG_ENONFINITE, "non-finite query component") : HCG_OK;
}

LocateArgs locate_args(const hcg_index* ix, const uint8_t* dq, uint32_t nq, uint32_t depth, uint32_t* begins,
                       uint64_t* ranks, const QueryFlag& flag) {
    LocateArgs a{};
    a.dtype = int(ix->dtype);
    a.bad = flag.dev;
    a.queries = dq;
    a.nq = nq;
    a.pitch = ix->pitch;
    a.curves = ix->d_curves;
    a.C = ix->C;
    a.assign = ix->d_assign;
    a.lut = ix->d_lut;
    a.m = int(ix->m);
    a.kind = int(ix->kind);
    a.n = ix->n;
    a.depth = depth;
    a.out_begin = begins;
    a.out_rank = ranks;
    return a;
}

hcg_status locate(const hcg_index* ix, Scratch& sc, const uint8_t* dq, uint32_t nq, uint32_t depth,
                  uint32_t* begins, uint64_t* ranks, const QueryFlag& flag) {
    return launch_locate(locate_args(ix, dq, nq, depth, begins, ranks, flag), ix->dmax, ix->wsmax, sc.st);
}

RefineArgs refine_args(const hcg_index* ix, const uint8_t* dq, uint32_t nq, uint32_t depth, uint32_t k,
                       const uint32_t* begins) {
    RefineArgs a{};
    a.queries = dq;
    a.nq = nq;
    a.pitch = ix->pitch;
    a.d_full = ix->d_full;
    a.rows = ix->rows;
    a.slots = ix->d_slot_ptrs;
    a.C = ix->C;
    a.begins = begins;
    a.take = uint32_t(std::min<uint64_t>(depth, ix->n));
    a.k = k;
    a.id_base = ix->id_base;
    a.id_stride = ix->id_stride;
    a.n_rows = ix->n;
    a.dtype = int(ix->dtype);
    a.idtab = ix->idtab;
    static const bool no_list = knob("HCG_NO_UNION_LIST") != nullptr;
    a.union_list = !no_list;
    return a;
}

hcg_status run_refine(const hcg_index* ix, Scratch& sc, const RefineArgs& a_in) {
    RefineArgs a = a_in;
    size_t need = 0;
    HCG_TRY(launch_refine(a, nullptr, &need, ix->device, sc.st));
    void* scratch = need ? sc.alloc<uint8_t>(need) : reinterpret_cast<void*>(1);
    if (!scratch) return set_error(HCG_ENOMEM, "refine scratch");
    const hcg_status rc = launch_refine(a, need ? scratch : reinterpret_cast<void*>(1), &need, ix->device, sc.st);
    return rc;
}

// v holds each of 0 .. v.size()-1 exactly once.
bool is_permutation_of_n(const std::vector<uint32_t>& v) {
    std::vector<uint8_t> seen(v.size(), 0);
    for (uint32_t x : v) {
        if (x >= v.size() || seen[x]) return false;
        seen[x] = 1;
    }
    return true;
}

// Copy a host-side vector to a user buffer that may be host or device memory.
template <class T>
hcg_status deliver(T* user, const std::vector<T>& v) {
    if (v.empty()) return HCG_OK;
    if (is_device_ptr(user)) HCG_TRY_CUDA(cudaMemcpy(user, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    else std::memcpy(user, v.data(), v.size() * sizeof(T));
    return HCG_OK;
}

}  // namespace
}  // namespace hcg

using namespace hcg;

namespace {
constexpr char kMagic[8] = {'H', 'C', 'G', 'I', 'D', 'X', 0, 1};
constexpr char kTrailer[8] = {'H', 'C', 'G', 'E', 'N', 'D', 0, 0};
constexpr uint32_t kFormatVersion = 4;  // 2: + dtype; 3: + physical row order (id table); 4: + view offset

struct FileCloser {
    FILE* f = nullptr;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};
template <class T>
bool put(FILE* f, const T* p, size_t count) {
    return count == 0 || std::fwrite(p, sizeof(T), count, f) == count;
}
template <class T>
bool get(FILE* f, T* p, size_t count) {
    return count == 0 || std::fread(p, sizeof(T), count, f) == count;
}
}  // namespace

extern "C" {

const char* hcg_last_error(void) { return g_err.c_str(); }
const char* hcg_version(void) { return "hcg 0.1 (sm_100a)"; }

hcg_status hcg_make_lut(float offset, float scale, uint32_t m, uint32_t* lut) {
    if (!lut) return set_error(HCG_EINVAL, "null lut");
    if (m < 1 || m > 32) return set_error(HCG_EINVAL, "bits_per_dim out of range [1,32]");
    for (int b = 0; b < 256; ++b) {
        const float v = offset + float(b) * scale;
        if (!std::isfinite(v)) return set_error(HCG_ENONFINITE, "non-finite component");
        lut[b] = uint32_t(uint64_t(ordinal_of(v)) >> (32 - m));
    }
    return HCG_OK;
}

hcg_status hcg_default_assignment(uint32_t d_full, uint32_t curves, uint32_t* off, uint32_t* assign) {
    if (!off || !assign) return set_error(HCG_EINVAL, "null output");
    if (curves < 1 || curves > d_full) return set_error(HCG_EINVAL, "curves must be in [1, d_full]");
    uint32_t pos = 0;
    for (uint32_t c = 0; c < curves; ++c) {
        off[c] = pos;
        for (uint32_t j = c; j < d_full; j += curves) assign[pos++] = j;
    }
    off[curves] = pos;
    return HCG_OK;
}

hcg_status hcg_build(const hcg_scheme* s, const uint8_t* rows, uint64_t n, uint64_t id_base, uint64_t id_stride,
                     int device, void* stream, hcg_index** out) {
    if (!out) return set_error(HCG_EINVAL, "null output handle");
    *out = nullptr;
    HCG_TRY(validate_scheme(s));
    if (id_stride < 1) return set_error(HCG_EINVAL, "id_stride must be >= 1");
    if (n >= (1ull << 32)) return set_error(HCG_ECAPACITY, "more than 2^32-1 rows in one index");
    if (n && !rows) return set_error(HCG_EINVAL, "null rows");
    HCG_TRY(check_device(device));
    DeviceGuard g(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);

    hcg_index* ix = nullptr;
    HCG_TRY(new_index(s, n, id_base, id_stride, device, st, &ix));
    auto fail = [&](hcg_status rc) {
        cudaStreamSynchronize(st);
        release(ix);
        return rc;
    };
    hcg_status rc;
    if (n) {
        if (ix->pitch != ix->row_bytes && cudaMemsetAsync(ix->rows, 0, size_t(n) * ix->pitch, st) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "memset rows"));
        if (cudaMemcpy2DAsync(ix->rows, ix->pitch, rows, ix->row_bytes, ix->row_bytes, n, cudaMemcpyDefault, st) !=
            cudaSuccess)
            return fail(set_error(HCG_ECUDA, std::string("copy rows: ") + cudaGetErrorString(cudaGetLastError())));
    }
    for (uint32_t c = 0; c < ix->C; ++c)
        if ((rc = build_curve(ix, c, st)) != HCG_OK) return fail(rc);
    if ((rc = reorder_rows(ix, st)) != HCG_OK) return fail(rc);
    if ((rc = publish_tables(ix, st)) != HCG_OK) return fail(rc);
    *out = ix;
    return HCG_OK;
}

hcg_status hcg_free(hcg_index* ix) {
    release(ix);
    return HCG_OK;
}

uint64_t hcg_size(const hcg_index* ix) { return ix ? ix->n : 0; }
uint32_t hcg_curves(const hcg_index* ix) { return ix ? ix->C : 0; }
uint32_t hcg_key_words(const hcg_index* ix, uint32_t c) { return ix && c < ix->C ? ix->curves[c].w : 0; }
uint64_t hcg_device_bytes(const hcg_index* ix) { return ix ? ix->bytes : 0; }
uint64_t hcg_launch_count(void) { return hcg::g_launches.load(); }
uint32_t hcg_index_dtype(const hcg_index* ix) { return ix ? ix->dtype : 0; }
int hcg_index_device(const hcg_index* ix) { return ix ? ix->device : -1; }
uint32_t hcg_refine_unionless(const hcg_index* ix, uint32_t nq, uint32_t k, uint32_t depth) {
    if (!ix || k < 1 || k > HCG_MAX_K || depth < 1 || ix->n == 0) return 0;
    RefineArgs a = refine_args(ix, nullptr, nq, depth, k, nullptr);
    a.mode = kOutIds;
    return refine_unionless(a) ? 1u : 0u;
}
hcg_status hcg_index_ids(const hcg_index* ix, uint64_t* id_base, uint64_t* id_stride) {
    HCG_TRY(check_index(ix));
    if (id_base) *id_base = ix->id_base;
    if (id_stride) *id_stride = ix->id_stride;
    return HCG_OK;
}

hcg_status hcg_insert(hcg_index* ix, const uint8_t* rows, uint64_t nb, void* stream) {
    HCG_TRY(check_index(ix));
    if (nb == 0) return HCG_OK;
    if (!rows) return set_error(HCG_EINVAL, "null rows");
    const uint64_t n_old = ix->n, n_new = n_old + nb;
    if (n_new >= (1ull << 32)) return set_error(HCG_ECAPACITY, "more than 2^32-1 rows in one index");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // Stage everything (rows, id table, every curve) first; the index is
    // only touched once all of it succeeded, so a failure leaves it as it was.
    uint64_t staged = 0;
    uint8_t* nr = nullptr;
    uint32_t* nt = nullptr;
    std::vector<CurveOut> outs(ix->C);
    auto fail = [&](hcg_status rc) {
        cudaStreamSynchronize(st);
        for (auto& o : outs) o.drop();
        dev_free(nr, size_t(n_new) * ix->pitch, &staged);
        dev_free(nt, size_t(n_new) * 4, &staged);
        return rc;
    };
    if (dev_alloc(&nr, size_t(n_new) * ix->pitch, &staged) != HCG_OK) return fail(HCG_ENOMEM);
    if ((n_old && cudaMemcpyAsync(nr, ix->rows, size_t(n_old) * ix->pitch, cudaMemcpyDeviceToDevice, st) != cudaSuccess) ||
        (ix->pitch != ix->row_bytes &&
         cudaMemsetAsync(nr + size_t(n_old) * ix->pitch, 0, size_t(nb) * ix->pitch, st) != cudaSuccess) ||
        cudaMemcpy2DAsync(nr + size_t(n_old) * ix->pitch, ix->pitch, rows, ix->row_bytes, ix->row_bytes, nb,
                          cudaMemcpyDefault, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return fail(set_error(HCG_ECUDA, std::string("copy rows: ") + cudaGetErrorString(cudaGetLastError())));
    if (ix->dtype == HCG_F32) {  // reject NaN / Inf before the index changes (curve.cpp:167)
        Scratch sc(st);
        unsigned* bad = sc.alloc<unsigned>(1);
        unsigned h = 0;
        if (!bad) return fail(set_error(HCG_ENOMEM, "flag"));
        if (cudaMemsetAsync(bad, 0, 4, st) != cudaSuccess) return fail(set_error(HCG_ECUDA, "memset"));
        launch_check_finite(nr + size_t(n_old) * ix->pitch, nb, ix->pitch, ix->d_full, bad, st);
        if (cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "finite check"));
        if (h) return fail(set_error(HCG_ENONFINITE, "non-finite component"));
    }
    if (ix->idtab) {  // appended rows sit at physical = id slot
        if (dev_alloc(&nt, n_new, &staged) != HCG_OK) return fail(set_error(HCG_ENOMEM, "id table"));
        if (cudaMemcpyAsync(nt, ix->idtab, n_old * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "copy id table"));
        launch_iota(nt + n_old, nb, uint32_t(n_old), st);
        if (check_launch("iota") != HCG_OK || cudaStreamSynchronize(st) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "id table"));
    }
    for (uint32_t c = 0; c < ix->C; ++c) {
        const hcg_status rc = insert_curve_into(ix, c, nr, n_old, nb, nt, st, &outs[c]);
        if (rc != HCG_OK) return fail(rc);
    }
    // commit
    for (uint32_t c = 0; c < ix->C; ++c) commit_curve(ix, c, n_old, outs[c]);
    dev_free(ix->rows, size_t(std::max<uint64_t>(n_old, 1)) * ix->pitch, &ix->bytes);
    ix->rows = nr;
    if (nt) {
        dev_free(ix->idtab, size_t(n_old) * 4, &ix->bytes);
        ix->idtab = nt;
    }
    ix->bytes += staged;
    ix->n = n_new;
    const hcg_status rc = publish_tables(ix, st);
    if (rc != HCG_OK) ix->broken = true;  // device tables may be stale: refuse further use
    return rc;
}


hcg_status hcg_save(const hcg_index* ix, const char* path) {
    HCG_TRY(check_index(ix));
    if (!path) return set_error(HCG_EINVAL, "null path");
    DeviceGuard g(ix->device);
    FileCloser fc;
    fc.f = std::fopen(path, "wb");
    if (!fc.f) return set_error(HCG_EIO, std::string("cannot open ") + path + " for writing");
    FILE* f = fc.f;
    const uint32_t hdr[7] = {kFormatVersion, ix->d_full, ix->C, ix->m, ix->kind, uint32_t(ix->assign.size()),
                             ix->dtype};
    const uint64_t ids[3] = {ix->n, ix->id_base, ix->id_stride};
    bool ok = put(f, kMagic, 8) && put(f, hdr, 7) && put(f, &ix->dist_scale, 1) && put(f, &ix->view_offset, 1) &&
              put(f, ids, 3) &&
              put(f, ix->lut, 256) && put(f, ix->off.data(), ix->off.size()) &&
              put(f, ix->assign.data(), ix->assign.size());
    // rows, unpadded, in slices
    const uint64_t slice = 1 << 20;
    std::vector<uint8_t> buf;
    for (uint64_t r = 0; ok && r < ix->n; r += slice) {
        const uint64_t cnt = std::min(slice, ix->n - r);
        buf.resize(cnt * ix->row_bytes);
        HCG_TRY_CUDA(cudaMemcpy2D(buf.data(), ix->row_bytes, ix->rows + r * ix->pitch, ix->pitch, ix->row_bytes, cnt,
                                  cudaMemcpyDeviceToHost));
        ok = put(f, buf.data(), buf.size());
    }
    // rows are stored in their physical order; the id table (if any) follows
    const uint32_t has_idtab = ix->idtab && ix->n ? 1u : 0u;
    ok = ok && put(f, &has_idtab, 1);
    if (ok && has_idtab) {
        std::vector<uint32_t> idt(ix->n);
        HCG_TRY_CUDA(cudaMemcpy(idt.data(), ix->idtab, ix->n * 4, cudaMemcpyDeviceToHost));
        ok = put(f, idt.data(), idt.size());
    }
    for (uint32_t c = 0; ok && c < ix->C; ++c) {
        const CurveDev& cv = ix->curves[c];
        const uint32_t ch[5] = {cv.w, cv.ws, cv.hv, cv.dims, cv.off};
        ok = put(f, ch, 5) && put(f, cv.prefix, kMaxKeyWords);
        if (ix->n) {
            std::vector<uint64_t> k(size_t(ix->n) * cv.ws);
            std::vector<uint32_t> sl(ix->n);
            HCG_TRY_CUDA(cudaMemcpy(k.data(), ix->keys[c], k.size() * 8, cudaMemcpyDeviceToHost));
            HCG_TRY_CUDA(cudaMemcpy(sl.data(), ix->slots[c], sl.size() * 4, cudaMemcpyDeviceToHost));
            ok = ok && put(f, k.data(), k.size()) && put(f, sl.data(), sl.size());
        }
    }
    ok = ok && put(f, kTrailer, 8);
    if (!ok) return set_error(HCG_EIO, std::string("write failed: ") + path);
    return HCG_OK;
}

hcg_status hcg_load(const char* path, int device, void* stream, hcg_index** out) {
    if (!path || !out) return set_error(HCG_EINVAL, "null argument");
    *out = nullptr;
    FileCloser fc;
    fc.f = std::fopen(path, "rb");
    if (!fc.f) return set_error(HCG_EIO, std::string("cannot open ") + path);
    FILE* f = fc.f;
    char magic[8];
    uint32_t hdr[7];
    double scale = 0;
    uint64_t ids[3];
    if (!get(f, magic, 8) || std::memcmp(magic, kMagic, 8) != 0) return set_error(HCG_EIO, std::string(path) + ": not an hcg index");
    if (!get(f, hdr, 7) || hdr[0] != kFormatVersion) return set_error(HCG_EIO, std::string(path) + ": unsupported version");
    float voff = 0.0f;
    if (!get(f, &scale, 1) || !get(f, &voff, 1) || !get(f, ids, 3))
        return set_error(HCG_EIO, std::string(path) + ": truncated header");
    hcg_scheme s{};
    s.d_full = hdr[1];
    s.curves = hdr[2];
    s.bits_per_dim = hdr[3];
    s.curve_kind = hdr[4];
    s.dist_scale = scale;
    s.view_offset = voff;
    s.dtype = hdr[6];
    if (s.curves == 0 || s.curves > 4096 || hdr[5] > 1u << 20) return set_error(HCG_EIO, std::string(path) + ": corrupt header");
    std::vector<uint32_t> off(s.curves + 1), asg(hdr[5]);
    if (!get(f, s.cell_lut, 256) || !get(f, off.data(), off.size()) || !get(f, asg.data(), asg.size()))
        return set_error(HCG_EIO, std::string(path) + ": truncated scheme");
    s.assign_off = off.data();
    s.assign = asg.data();
    if (off[s.curves] != hdr[5]) return set_error(HCG_EIO, std::string(path) + ": corrupt scheme");
    HCG_TRY(validate_scheme(&s));
    HCG_TRY(check_device(device));
    DeviceGuard g(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    hcg_index* ix = nullptr;
    HCG_TRY(new_index(&s, ids[0], ids[1], ids[2], device, st, &ix));
    auto fail = [&](hcg_status rc) {
        cudaStreamSynchronize(st);
        release(ix);
        return rc;
    };
    const uint64_t slice = 1 << 20;
    std::vector<uint8_t> buf;
    for (uint64_t r = 0; r < ix->n; r += slice) {
        const uint64_t cnt = std::min(slice, ix->n - r);
        buf.resize(cnt * ix->row_bytes);
        if (!get(f, buf.data(), buf.size())) return fail(set_error(HCG_EIO, std::string(path) + ": truncated rows"));
        if (cudaMemcpy2D(ix->rows + r * ix->pitch, ix->pitch, buf.data(), ix->row_bytes, ix->row_bytes, cnt,
                         cudaMemcpyHostToDevice) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "upload rows"));
    }
    uint32_t has_idtab = 0;
    if (!get(f, &has_idtab, 1) || has_idtab > 1) return fail(set_error(HCG_EIO, std::string(path) + ": corrupt id table"));
    if (has_idtab && ix->n) {
        std::vector<uint32_t> idt(ix->n);
        if (!get(f, idt.data(), idt.size())) return fail(set_error(HCG_EIO, std::string(path) + ": truncated id table"));
        if (!is_permutation_of_n(idt)) return fail(set_error(HCG_EIO, std::string(path) + ": id table is not a permutation"));
        if (dev_alloc(&ix->idtab, ix->n, &ix->bytes) != HCG_OK ||
            cudaMemcpy(ix->idtab, idt.data(), ix->n * 4, cudaMemcpyHostToDevice) != cudaSuccess)
            return fail(set_error(HCG_ECUDA, "upload id table"));
    }
    for (uint32_t c = 0; c < ix->C; ++c) {
        CurveDev& cv = ix->curves[c];
        std::memset(&cv, 0, sizeof(cv));
        uint32_t ch[5];
        if (!get(f, ch, 5) || !get(f, cv.prefix, kMaxKeyWords))
            return fail(set_error(HCG_EIO, std::string(path) + ": truncated curve header"));
        cv.w = ch[0];
        cv.ws = ch[1];
        cv.hv = ch[2];
        cv.dims = ch[3];
        cv.off = ch[4];
        if (cv.ws < 1 || cv.ws > cv.w || cv.w > kMaxKeyWords || cv.off != off[c] || cv.dims != off[c + 1] - off[c])
            return fail(set_error(HCG_EIO, std::string(path) + ": corrupt curve header"));
        if (ix->n) {
            std::vector<uint64_t> k(size_t(ix->n) * cv.ws);
            std::vector<uint32_t> sl(ix->n);
            if (!get(f, k.data(), k.size()) || !get(f, sl.data(), sl.size()))
                return fail(set_error(HCG_EIO, std::string(path) + ": truncated curve arrays"));
            // every slot is a row of this index, each row once: a corrupt file
            // must not turn into out-of-bounds row gathers
            if (!is_permutation_of_n(sl)) return fail(set_error(HCG_EIO, std::string(path) + ": corrupt slot array"));
            hcg_status rc;
            if ((rc = dev_alloc(&ix->keys[c], k.size(), &ix->bytes)) != HCG_OK) return fail(rc);
            if ((rc = dev_alloc(&ix->slots[c], sl.size(), &ix->bytes)) != HCG_OK) return fail(rc);
            if (cudaMemcpy(ix->keys[c], k.data(), k.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(ix->slots[c], sl.data(), sl.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
                return fail(set_error(HCG_ECUDA, "upload curve"));
            cv.keys = ix->keys[c];
            cv.slots = ix->slots[c];
        }
    }
    char tr[8];
    if (!get(f, tr, 8) || std::memcmp(tr, kTrailer, 8) != 0) return fail(set_error(HCG_EIO, std::string(path) + ": missing trailer"));
    hcg_status rc = publish_tables(ix, st);
    if (rc != HCG_OK) return fail(rc);
    *out = ix;
    return HCG_OK;
}

static hcg_status search_impl(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint32_t depth,
                              uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, uint64_t* out_packed,
                              void* stream, float* ms_out = nullptr, double* out_sq64 = nullptr) {
    HCG_TRY(check_search_args(ix, k, depth));
    const bool f32 = ix->dtype == HCG_F32;
    if (f32 != (out_sq64 != nullptr))  // packed / timed searches are u8-only
        return set_error(HCG_EINVAL, f32 ? "index holds f32 descriptors: use hcg_search_f32"
                                         : "index holds u8 descriptors: use hcg_search");
    if (nq == 0) return HCG_OK;
    if (!queries) return set_error(HCG_EINVAL, "null queries");
    const bool packed = out_packed != nullptr;
    if (!packed && (!out_ids || !(f32 ? static_cast<void*>(out_sq64) : out_sqdist) || !out_len))
        return set_error(HCG_EINVAL, "null output");
    if (packed && ix->n && ix->id_base + (ix->n - 1) * ix->id_stride >= (1ull << 32))
        return set_error(HCG_ECAPACITY, "packed results need ids < 2^32");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    OutBuf<uint64_t> oi, op;
    OutBuf<uint32_t> os, ol;
    OutBuf<double> o64;
    QueryFlag flag;
    const size_t cnt = size_t(nq) * k;
    if (packed) {
        HCG_TRY(stage_out(sc, out_packed, cnt, &op));
    } else {
        HCG_TRY(stage_out(sc, out_ids, cnt, &oi));
        if (f32)
            HCG_TRY(stage_out(sc, out_sq64, cnt, &o64));
        else
            HCG_TRY(stage_out(sc, out_sqdist, cnt, &os));
        HCG_TRY(stage_out(sc, out_len, nq, &ol));
    }
    if (ix->n == 0) {  // empty index: every list is empty
        if (packed) {
            HCG_TRY_CUDA(cudaMemsetAsync(op.dev, 0xFF, cnt * 8, st));
        } else {
            HCG_TRY_CUDA(cudaMemsetAsync(oi.dev, 0xFF, cnt * 8, st));
            if (f32)
                HCG_TRY(fill_inf(o64.dev, cnt, st));
            else
                HCG_TRY_CUDA(cudaMemsetAsync(os.dev, 0xFF, cnt * 4, st));
            HCG_TRY_CUDA(cudaMemsetAsync(ol.dev, 0, size_t(nq) * 4, st));
        }
    } else {
        const uint8_t* dq = nullptr;
        HCG_TRY(stage_rows(sc, queries, nq, ix->row_bytes, ix->pitch, &dq));
        HCG_TRY(make_flag(ix, sc, &flag));
        // small batches: the whole search of a query in one CTA, one launch
        {
            RefineArgs a = refine_args(ix, dq, nq, depth, k, nullptr);
            a.mode = packed ? kOutPacked : kOutIds;
            a.out_packed = op.dev;
            a.out_ids = oi.dev;
            a.out_sqdist = os.dev;
            a.out_len = ol.dev;
            const LocateArgs la = locate_args(ix, dq, nq, depth, nullptr, nullptr, flag);
            if (!ms_out && small_eligible(la, a, ix->dims16, ix->wsmax, ix->device)) {
                static unsigned long long* prof = nullptr;  // phase stamps (tuning builds: HCG_SMALL_PROF)
                if (knob("HCG_SMALL_PROF")) {
                    if (!prof) cudaMalloc(&prof, 8 * 8);
                    a.prof = prof;
                }
                HCG_TRY(launch_search_small(la, a, ix->wsmax, ix->device, st));
                if (a.prof) {
                    unsigned long long h[5];
                    cudaMemcpyAsync(h, prof, 40, cudaMemcpyDeviceToHost, st);
                    cudaStreamSynchronize(st);
                    fprintf(stderr, "small-batch phases (ns): locate %llu union %llu gather %llu merge %llu\n",
                            h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3]);
                }
                goto finish;
            }
        }
        {
        uint32_t* begins = sc.alloc<uint32_t>(size_t(nq) * ix->C);
        if (!begins) return set_error(HCG_ENOMEM, "window buffer");
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
        if (ms_out) {
            for (auto& e : ev) HCG_TRY_CUDA(cudaEventCreate(&e));
            HCG_TRY_CUDA(cudaEventRecord(ev[0], st));
        }
        HCG_TRY(locate(ix, sc, dq, nq, depth, begins, nullptr, flag));
        if (ms_out) HCG_TRY_CUDA(cudaEventRecord(ev[1], st));
        RefineArgs a = refine_args(ix, dq, nq, depth, k, begins);
        if (ms_out) a.ev_mid = ev[2];
        if (packed) {
            a.mode = kOutPacked;
            a.out_packed = op.dev;
        } else {
            a.mode = kOutIds;
            a.out_ids = oi.dev;
            a.out_sqdist = os.dev;
            a.out_sqdist_f64 = o64.dev;
            a.out_len = ol.dev;
        }
        HCG_TRY(run_refine(ix, sc, a));
        if (ms_out) {
            HCG_TRY_CUDA(cudaEventRecord(ev[3], st));
            HCG_TRY_CUDA(cudaEventSynchronize(ev[3]));
            HCG_TRY_CUDA(cudaEventElapsedTime(&ms_out[0], ev[0], ev[1]));
            float mid = 0.0f;
            if (cudaEventQuery(ev[2]) == cudaSuccess && cudaEventElapsedTime(&mid, ev[1], ev[2]) == cudaSuccess) {
                ms_out[1] = mid;  // candidate union
                HCG_TRY_CUDA(cudaEventElapsedTime(&ms_out[2], ev[2], ev[3]));
            } else {  // single refine kernel
                cudaGetLastError();
                ms_out[1] = 0.0f;
                HCG_TRY_CUDA(cudaEventElapsedTime(&ms_out[2], ev[1], ev[3]));
            }
            for (auto& e : ev) cudaEventDestroy(e);
        }
        }
    }
finish:
    HCG_TRY(finish_out(sc, oi));
    HCG_TRY(finish_out(sc, os));
    HCG_TRY(finish_out(sc, o64));
    HCG_TRY(finish_out(sc, ol));
    HCG_TRY(finish_out(sc, op));
    HCG_TRY(check_flag(flag, st));
    if (oi.host || os.host || o64.host || ol.host || op.host) HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return HCG_OK;
}

hcg_status hcg_search(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint32_t depth,
                      uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, void* stream) {
    return search_impl(ix, queries, nq, k, depth, out_ids, out_sqdist, out_len, nullptr, stream);
}

hcg_status hcg_search_f32(const hcg_index* ix, const float* queries, uint32_t nq, uint32_t k, uint32_t depth,
                          uint64_t* out_ids, double* out_sqdist, uint32_t* out_len, void* stream) {
    if (!out_sqdist) return set_error(HCG_EINVAL, "null output");
    return search_impl(ix, reinterpret_cast<const uint8_t*>(queries), nq, k, depth, out_ids, nullptr, out_len,
                       nullptr, stream, nullptr, out_sqdist);
}

hcg_status hcg_search_timed(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint32_t depth,
                            uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, float* ms_out, void* stream) {
    if (!ms_out) return set_error(HCG_EINVAL, "null ms_out");
    ms_out[0] = ms_out[1] = ms_out[2] = 0.0f;
    return search_impl(ix, queries, nq, k, depth, out_ids, out_sqdist, out_len, nullptr, stream, ms_out);
}

hcg_status hcg_search_packed(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint32_t depth,
                             uint64_t* out_packed, void* stream) {
    if (!out_packed) return set_error(HCG_EINVAL, "null output");
    return search_impl(ix, queries, nq, k, depth, nullptr, nullptr, nullptr, out_packed, stream);
}

hcg_status hcg_merge_packed(const uint64_t* packed, uint32_t parts, uint32_t nq, uint32_t k, uint64_t* out_ids,
                            uint32_t* out_sqdist, uint32_t* out_len, int device, void* stream) {
    if (k < 1) return set_error(HCG_EINVAL, "k must be >= 1");
    if (k > HCG_MAX_K) return set_error(HCG_ECAPACITY, "k exceeds HCG_MAX_K");
    if (parts < 1) return set_error(HCG_EINVAL, "parts must be >= 1");
    if (nq == 0) return HCG_OK;
    if (!packed || !out_ids || !out_sqdist || !out_len) return set_error(HCG_EINVAL, "null buffer");
    HCG_TRY(check_device(device));
    DeviceGuard g(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    const size_t cnt = size_t(nq) * k;
    const uint64_t* dp = packed;
    if (!is_device_ptr(packed)) {
        uint64_t* d = sc.alloc<uint64_t>(cnt * parts);
        if (!d) return set_error(HCG_ENOMEM, "merge staging");
        HCG_TRY_CUDA(cudaMemcpyAsync(d, packed, cnt * parts * 8, cudaMemcpyHostToDevice, st));
        dp = d;
    }
    OutBuf<uint64_t> oi;
    OutBuf<uint32_t> os, ol;
    HCG_TRY(stage_out(sc, out_ids, cnt, &oi));
    HCG_TRY(stage_out(sc, out_sqdist, cnt, &os));
    HCG_TRY(stage_out(sc, out_len, nq, &ol));
    HCG_TRY(launch_merge(dp, parts, nq, k, oi.dev, os.dev, ol.dev, st));
    HCG_TRY(finish_out(sc, oi));
    HCG_TRY(finish_out(sc, os));
    HCG_TRY(finish_out(sc, ol));
    if (oi.host || os.host || ol.host) HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return HCG_OK;
}

hcg_status hcg_keys(const hcg_index* ix, const uint8_t* rows, uint64_t n, uint32_t curve, uint64_t* out_words,
                    void* stream) {
    HCG_TRY(check_index(ix));
    if (curve >= ix->C) return set_error(HCG_EINVAL, "curve out of range");
    if (n == 0) return HCG_OK;
    if (!rows || !out_words) return set_error(HCG_EINVAL, "null buffer");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    const uint8_t* dr = nullptr;
    HCG_TRY(stage_rows(sc, rows, n, ix->row_bytes, ix->pitch, &dr));
    const uint32_t W = ix->curves[curve].w;
    uint64_t* soa = sc.alloc<uint64_t>(size_t(W) * n);
    unsigned long long* oa = sc.alloc<unsigned long long>(2 * W + 1);
    if (!soa || !oa) return set_error(HCG_ENOMEM, "key buffers");
    HCG_TRY_CUDA(cudaMemsetAsync(oa + 2 * W, 0, 8, st));
    const uint32_t d = ix->off[curve + 1] - ix->off[curve];
    HCG_TRY(keygen_rows(dr, n, ix->pitch, ix->d_assign + ix->off[curve], int(d), int(ix->m), int(ix->kind),
                        ix->d_lut, soa, int(W), oa, ix->dmax, int(ix->dtype), reinterpret_cast<unsigned*>(oa + 2 * W),
                        st));
    std::vector<uint64_t> h(size_t(W) * n), t(size_t(W) * n);
    unsigned long long bad = 0;
    HCG_TRY_CUDA(cudaMemcpyAsync(h.data(), soa, h.size() * 8, cudaMemcpyDeviceToHost, st));
    HCG_TRY_CUDA(cudaMemcpyAsync(&bad, oa + 2 * W, 8, cudaMemcpyDeviceToHost, st));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    if (bad) return set_error(HCG_ENONFINITE, "non-finite component");
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t w = 0; w < W; ++w) t[i * W + w] = h[uint64_t(w) * n + i];
    return deliver(out_words, t);
}

hcg_status hcg_sorted(const hcg_index* ix, uint32_t curve, uint64_t* out_ids, uint64_t* out_words, void* stream) {
    HCG_TRY(check_index(ix));
    if (curve >= ix->C) return set_error(HCG_EINVAL, "curve out of range");
    if (ix->n == 0) return HCG_OK;
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    const uint64_t n = ix->n;
    const CurveDev& cv = ix->curves[curve];
    if (out_ids) {
        std::vector<uint32_t> s(n), idt;
        HCG_TRY_CUDA(cudaMemcpyAsync(s.data(), ix->slots[curve], n * 4, cudaMemcpyDeviceToHost, st));
        if (ix->idtab) {
            idt.resize(n);
            HCG_TRY_CUDA(cudaMemcpyAsync(idt.data(), ix->idtab, n * 4, cudaMemcpyDeviceToHost, st));
        }
        HCG_TRY_CUDA(cudaStreamSynchronize(st));
        std::vector<uint64_t> ids(n);
        for (uint64_t i = 0; i < n; ++i)
            ids[i] = ix->id_base + uint64_t(ix->idtab ? idt[s[i]] : s[i]) * ix->id_stride;
        HCG_TRY(deliver(out_ids, ids));
    }
    if (out_words) {
        uint64_t* full = sc.alloc<uint64_t>(size_t(n) * cv.w);
        if (!full) return set_error(HCG_ENOMEM, "key buffer");
        launch_expand_keys(ix->keys[curve], n, int(cv.ws), int(cv.w), cv, full, st);
        HCG_TRY(check_launch("expand keys"));
        std::vector<uint64_t> h(size_t(n) * cv.w);
        HCG_TRY_CUDA(cudaMemcpyAsync(h.data(), full, h.size() * 8, cudaMemcpyDeviceToHost, st));
        HCG_TRY_CUDA(cudaStreamSynchronize(st));
        HCG_TRY(deliver(out_words, h));
    }
    return HCG_OK;
}

hcg_status hcg_sorted_range(const hcg_index* ix, uint32_t curve, uint64_t begin, uint64_t count, uint64_t* out_ids,
                            void* stream) {
    HCG_TRY(check_index(ix));
    if (curve >= ix->C) return set_error(HCG_EINVAL, "curve out of range");
    if (begin > ix->n || count > ix->n - begin) return set_error(HCG_EINVAL, "range beyond the subindex");
    if (count == 0) return HCG_OK;
    if (!out_ids) return set_error(HCG_EINVAL, "null buffer");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    uint32_t* d = sc.alloc<uint32_t>(count);
    if (!d) return set_error(HCG_ENOMEM, "range buffer");
    HCG_TRY_CUDA(cudaMemcpyAsync(d, ix->slots[curve] + begin, count * 4, cudaMemcpyDeviceToDevice, st));
    if (ix->idtab) launch_map(d, count, ix->idtab, st);  // physical row -> id slot
    HCG_TRY(check_launch("id map"));
    std::vector<uint32_t> sl(count);
    HCG_TRY_CUDA(cudaMemcpyAsync(sl.data(), d, count * 4, cudaMemcpyDeviceToHost, st));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> ids(count);
    for (uint64_t i = 0; i < count; ++i) ids[i] = ix->id_base + uint64_t(sl[i]) * ix->id_stride;
    return deliver(out_ids, ids);
}

hcg_status hcg_describe(const hcg_index* ix, hcg_scheme* out, uint32_t* assign_off, uint32_t* assign,
                        uint32_t* assign_len) {
    HCG_TRY(check_index(ix));
    if (!out || !assign_len) return set_error(HCG_EINVAL, "null argument");
    *assign_len = uint32_t(ix->assign.size());
    std::memset(out, 0, sizeof(*out));
    out->d_full = ix->d_full;
    out->curves = ix->C;
    out->bits_per_dim = ix->m;
    out->curve_kind = ix->kind;
    std::memcpy(out->cell_lut, ix->lut, sizeof(ix->lut));
    out->dist_scale = ix->dist_scale;
    out->dtype = ix->dtype;
    out->view_offset = ix->view_offset;
    if (assign_off && assign) {
        std::memcpy(assign_off, ix->off.data(), ix->off.size() * 4);
        std::memcpy(assign, ix->assign.data(), ix->assign.size() * 4);
        out->assign_off = assign_off;
        out->assign = assign;
    }
    return HCG_OK;
}

hcg_status hcg_windows(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t depth, uint64_t* out_rank,
                       uint64_t* out_begin, uint64_t* out_end, void* stream) {
    HCG_TRY(check_search_args(ix, 1, depth));
    if (nq == 0) return HCG_OK;
    if (!queries || !out_rank || !out_begin || !out_end) return set_error(HCG_EINVAL, "null buffer");
    const size_t cnt = size_t(nq) * ix->C;
    std::vector<uint64_t> r(cnt, 0), b(cnt, 0), e(cnt, 0);
    if (ix->n) {
        DeviceGuard g(ix->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        Scratch sc(st);
        const uint8_t* dq = nullptr;
        HCG_TRY(stage_rows(sc, queries, nq, ix->row_bytes, ix->pitch, &dq));
        uint32_t* begins = sc.alloc<uint32_t>(cnt);
        uint64_t* ranks = sc.alloc<uint64_t>(cnt);
        if (!begins || !ranks) return set_error(HCG_ENOMEM, "window buffers");
        QueryFlag flag;
        HCG_TRY(make_flag(ix, sc, &flag));
        HCG_TRY(locate(ix, sc, dq, nq, depth, begins, ranks, flag));
        HCG_TRY(check_flag(flag, st));
        std::vector<uint32_t> hb(cnt);
        HCG_TRY_CUDA(cudaMemcpyAsync(hb.data(), begins, cnt * 4, cudaMemcpyDeviceToHost, st));
        HCG_TRY_CUDA(cudaMemcpyAsync(r.data(), ranks, cnt * 8, cudaMemcpyDeviceToHost, st));
        HCG_TRY_CUDA(cudaStreamSynchronize(st));
        const uint64_t take = std::min<uint64_t>(depth, ix->n);
        for (size_t i = 0; i < cnt; ++i) {
            b[i] = hb[i];
            e[i] = hb[i] + take;
        }
    }
    HCG_TRY(deliver(out_rank, r));
    HCG_TRY(deliver(out_begin, b));
    return deliver(out_end, e);
}

hcg_status hcg_candidates(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t depth, uint64_t* out_ids,
                          uint32_t cap, uint32_t* out_count, void* stream) {
    HCG_TRY(check_search_args(ix, 1, depth));
    if (nq == 0) return HCG_OK;
    if (!queries || !out_count || (!out_ids && cap)) return set_error(HCG_EINVAL, "null buffer");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    OutBuf<uint64_t> oi;
    OutBuf<uint32_t> oc;
    HCG_TRY(stage_out(sc, out_ids, size_t(nq) * cap, &oi));
    HCG_TRY(stage_out(sc, out_count, nq, &oc));
    if (ix->n == 0) {
        HCG_TRY_CUDA(cudaMemsetAsync(oc.dev, 0, size_t(nq) * 4, st));
    } else {
        const uint8_t* dq = nullptr;
        HCG_TRY(stage_rows(sc, queries, nq, ix->row_bytes, ix->pitch, &dq));
        uint32_t* begins = sc.alloc<uint32_t>(size_t(nq) * ix->C);
        if (!begins) return set_error(HCG_ENOMEM, "window buffer");
        QueryFlag flag;
        HCG_TRY(make_flag(ix, sc, &flag));
        HCG_TRY(locate(ix, sc, dq, nq, depth, begins, nullptr, flag));
        HCG_TRY(check_flag(flag, st));
        RefineArgs a = refine_args(ix, dq, nq, depth, 1, begins);
        a.mode = kOutCandidates;
        a.out_ids = oi.dev;
        a.out_len = oc.dev;
        a.cap = cap;
        HCG_TRY(run_refine(ix, sc, a));
    }
    HCG_TRY(finish_out(sc, oi));
    HCG_TRY(finish_out(sc, oc));
    HCG_TRY_CUDA(cudaStreamSynchronize(st));
    std::vector<uint32_t> counts(nq);
    if (oc.host) std::memcpy(counts.data(), out_count, nq * 4);
    else HCG_TRY_CUDA(cudaMemcpy(counts.data(), out_count, nq * 4, cudaMemcpyDeviceToHost));
    if (out_ids)
        for (uint32_t c : counts)
            if (c > cap) return set_error(HCG_ECAPACITY, "candidate set larger than cap");
    return HCG_OK;
}

static hcg_status brute_impl(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint64_t* out_ids,
                             uint32_t* out_sqdist, double* out_sq64, uint32_t* out_len, void* stream) {
    HCG_TRY(check_search_args(ix, k, 1));
    const bool f32 = ix->dtype == HCG_F32;
    if (f32 != (out_sq64 != nullptr))
        return set_error(HCG_EINVAL, f32 ? "index holds f32 descriptors: use hcg_brute_force_f32"
                                         : "index holds u8 descriptors: use hcg_brute_force");
    if (nq == 0) return HCG_OK;
    if (!queries || !out_ids || !(f32 ? static_cast<void*>(out_sq64) : out_sqdist) || !out_len)
        return set_error(HCG_EINVAL, "null buffer");
    if (!f32 && ix->n && ix->id_base + (ix->n - 1) * ix->id_stride >= (1ull << 32))
        return set_error(HCG_ECAPACITY, "brute force needs ids < 2^32");
    DeviceGuard g(ix->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    OutBuf<uint64_t> oi;
    OutBuf<uint32_t> os, ol;
    OutBuf<double> o64;
    const size_t cnt = size_t(nq) * k;
    HCG_TRY(stage_out(sc, out_ids, cnt, &oi));
    if (f32)
        HCG_TRY(stage_out(sc, out_sq64, cnt, &o64));
    else
        HCG_TRY(stage_out(sc, out_sqdist, cnt, &os));
    HCG_TRY(stage_out(sc, out_len, nq, &ol));
    if (ix->n == 0) {
        HCG_TRY_CUDA(cudaMemsetAsync(oi.dev, 0xFF, cnt * 8, st));
        if (f32)
            HCG_TRY(fill_inf(o64.dev, cnt, st));
        else
            HCG_TRY_CUDA(cudaMemsetAsync(os.dev, 0xFF, cnt * 4, st));
        HCG_TRY_CUDA(cudaMemsetAsync(ol.dev, 0, size_t(nq) * 4, st));
    } else {
        const uint8_t* dq = nullptr;
        HCG_TRY(stage_rows(sc, queries, nq, ix->row_bytes, ix->pitch, &dq));
        BruteArgs a{ix->rows, ix->n, ix->pitch, dq, nq, k, ix->id_base, ix->id_stride, int(ix->dtype), ix->idtab};
        uint64_t* part = sc.alloc<uint64_t>((brute_scratch_bytes(a) + 7) / 8);
        if (!part) return set_error(HCG_ENOMEM, "brute-force scratch");
        HCG_TRY(launch_brute(a, part, oi.dev, os.dev, ol.dev, o64.dev, st));
    }
    HCG_TRY(finish_out(sc, oi));
    HCG_TRY(finish_out(sc, os));
    HCG_TRY(finish_out(sc, o64));
    HCG_TRY(finish_out(sc, ol));
    if (oi.host || os.host || o64.host || ol.host) HCG_TRY_CUDA(cudaStreamSynchronize(st));
    return HCG_OK;
}

hcg_status hcg_brute_force(const hcg_index* ix, const uint8_t* queries, uint32_t nq, uint32_t k, uint64_t* out_ids,
                           uint32_t* out_sqdist, uint32_t* out_len, void* stream) {
    if (!out_sqdist && nq) return set_error(HCG_EINVAL, "null buffer");
    return brute_impl(ix, queries, nq, k, out_ids, out_sqdist, nullptr, out_len, stream);
}

hcg_status hcg_brute_force_f32(const hcg_index* ix, const float* queries, uint32_t nq, uint32_t k, uint64_t* out_ids,
                               double* out_sqdist, uint32_t* out_len, void* stream) {
    if (!out_sqdist && nq) return set_error(HCG_EINVAL, "null buffer");
    return brute_impl(ix, reinterpret_cast<const uint8_t*>(queries), nq, k, out_ids, nullptr, out_sqdist, out_len,
                      stream);
}

hcg_status hcg_gen_rows(uint64_t first, uint64_t stride, uint64_t count, uint8_t* out_dev, int device, void* stream) {
    if (count && !is_device_ptr(out_dev)) return set_error(HCG_EINVAL, "hcg_gen_rows needs a device buffer");
    HCG_TRY(check_device(device));
    DeviceGuard g(device);
    return gen_rows(first, stride, count, out_dev, static_cast<cudaStream_t>(stream));
}

hcg_status hcg_gen_queries(uint64_t first, uint64_t count, uint64_t n_db, uint8_t* out_dev, int device, void* stream) {
    if (count && !is_device_ptr(out_dev)) return set_error(HCG_EINVAL, "hcg_gen_queries needs a device buffer");
    HCG_TRY(check_device(device));
    DeviceGuard g(device);
    return gen_queries(first, count, n_db, out_dev, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
