// hcg_host.hpp -- host-side declarations shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>

#include "../../include/hcg.h"

#define HCG_RET_IF(x)                   \
    do {                                \
        const hcg_status r_ = (x);      \
        if (r_ != HCG_OK) return r_;    \
    } while (0)

namespace hcg {

// A/B switches of the measured alternatives (e.g.
// HCG_NO_UNIONLESS).  Read only in a library built with -DHCG_TUNING_KNOBS
// (tools/build_variant.py); the release library always runs the measured-best
// paths and ignores the environment.
inline const char* knob(const char* name) {
#ifdef HCG_TUNING_KNOBS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

struct CurveDev;

hcg_status set_error(hcg_status code, const std::string& msg);
hcg_status check_launch(const char* what);

// build.cu
hcg_status keygen_rows(const uint8_t* rows, uint64_t n, uint32_t pitch, const uint16_t* assign_c, int d, int m,
                       int kind, const uint32_t* lut, uint64_t* keys_soa, int W, unsigned long long* or_and,
                       int dmax, int dtype, unsigned* bad, cudaStream_t st);
// Kernel-launch counter behind hcg_launch_count (search-path launchers and the radix sort add to it).
void count_launches(unsigned n);
hcg_status radix_sort_pairs(uint64_t** k, uint32_t** v, uint64_t** k_alt, uint32_t** v_alt, uint64_t n,
                            uint32_t digit_mask, uint32_t* counts, uint32_t* totals, cudaStream_t st);
size_t radix_counts_bytes(uint64_t n);
void launch_check_finite(const uint8_t* rows, uint64_t n, uint32_t pitch, uint32_t d, unsigned* bad,
                         cudaStream_t st);
void launch_permute_rows(const uint8_t* src, const uint32_t* perm, uint64_t n, uint32_t pitch, uint8_t* dst,
                         cudaStream_t st);
void launch_invert(const uint32_t* perm, uint64_t n, uint32_t* inv, cudaStream_t st);
void launch_map(uint32_t* v, uint64_t n, const uint32_t* map, cudaStream_t st);
void launch_sample(const uint64_t* keys, uint64_t n_samples, uint32_t ws, uint32_t stride, uint64_t* out,
                   cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, uint32_t base, cudaStream_t st);
void launch_offset(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t base, cudaStream_t st);
void launch_rank_merge(const uint64_t* ak, const uint32_t* as, uint64_t na, const uint64_t* bk, const uint32_t* bs,
                       uint64_t nb, int ws, uint64_t* ck, uint32_t* cs, cudaStream_t st);
void launch_gather_word(const uint64_t* src, const uint32_t* perm, uint64_t* dst, uint64_t n, cudaStream_t st);
void launch_pack_suffix(const uint64_t* keys_soa, const uint32_t* perm, uint64_t n, int ws, uint64_t top_mask,
                        uint64_t* out, cudaStream_t st);
void launch_expand_keys(const uint64_t* suffix, uint64_t n, int ws, int w_full, const CurveDev& cv, uint64_t* out,
                        cudaStream_t st);

// search.cu
struct LocateArgs {
    const uint8_t* queries;
    uint32_t nq;
    uint32_t pitch;
    const CurveDev* curves;  // device array
    uint32_t C;
    const uint16_t* assign;  // device, whole table
    const uint32_t* lut;     // device, 256
    int m, kind;
    uint64_t n;
    uint32_t depth;
    uint32_t* out_begin;  // nq x C
    uint64_t* out_rank;   // nq x C or null
    int dtype;            // hcg_dtype of the queries
    unsigned* bad;        // raised when a query component is non-finite (f32)
};
hcg_status launch_locate(const LocateArgs& a, int dmax, int wsmax, cudaStream_t st);

enum OutMode : int { kOutIds = 0, kOutPacked = 1, kOutCandidates = 2 };
struct RefineArgs {
    const uint8_t* queries;
    uint32_t nq;
    uint32_t pitch;
    uint32_t d_full;
    const uint8_t* rows;
    const uint32_t* const* slots;  // device array of C pointers
    uint32_t C;
    const uint32_t* begins;  // nq x C
    uint32_t take;
    uint32_t k;
    uint64_t id_base, id_stride;
    int mode;
    uint64_t* out_ids;     // kOutIds: nq x k ids; kOutCandidates: nq x cap ids
    uint32_t* out_sqdist;  // kOutIds
    uint32_t* out_len;     // kOutIds: len; kOutCandidates: count
    uint64_t* out_packed;  // kOutPacked
    uint32_t cap;          // kOutCandidates
    unsigned long long* prof;  // k_search_small phase timestamps (tuning builds, HCG_SMALL_PROF); null otherwise
    cudaEvent_t ev_mid;        // optional: recorded between the union and gather launches
    uint64_t n_rows;           // rows in the index (bounds checks)
    int dtype;                 // hcg_dtype of rows and queries
    double* out_sqdist_f64;    // HCG_F32 + kOutIds: nq x k squared distances
    const uint32_t* idtab;     // physical row -> id slot (null: identity)
    const uint32_t* qorder;    // processing order: batch position -> query (null: identity)
    bool union_list;           // union rounds after the first over a compacted shared-memory list
};
// Scratch bytes the refine launch needs (global hash tables when the table
// does not fit in shared memory); query with scratch == nullptr first.
hcg_status launch_refine(const RefineArgs& a, void* scratch, size_t* scratch_bytes, int device,
                         cudaStream_t st);
// Small batches: the whole search of a query in one CTA (k_search_small).
bool small_eligible(const LocateArgs& la, const RefineArgs& a, bool dims16, int wsmax, int device);
hcg_status launch_search_small(const LocateArgs& la, const RefineArgs& a, int wsmax, int device, cudaStream_t st);
// Whether a search of nq queries at k takes the union-less K3c (k_gather_nu).
bool refine_unionless(const RefineArgs& a);

hcg_status launch_merge(const uint64_t* packed, uint32_t parts, uint32_t nq, uint32_t k, uint64_t* out_ids,
                        uint32_t* out_sqdist, uint32_t* out_len, cudaStream_t st);

struct BruteArgs {
    const uint8_t* rows;
    uint64_t n;
    uint32_t pitch;
    const uint8_t* queries;
    uint32_t nq;
    uint32_t k;
    uint64_t id_base, id_stride;
    int dtype;
    const uint32_t* idtab;  // physical row -> id slot (null: identity)
};
size_t brute_scratch_bytes(const BruteArgs& a);
// brute_tc.cu: the same on the tensor cores (u8 rows of 128 B, k <= 32)
bool brute_tc_eligible(const BruteArgs& a);
size_t brute_tc_scratch_bytes(const BruteArgs& a);
hcg_status launch_brute_tc(const BruteArgs& a, void* scratch, uint64_t* out_ids, uint32_t* out_sqdist,
                           uint32_t* out_len, cudaStream_t st);
hcg_status launch_brute(const BruteArgs& a, uint64_t* scratch, uint64_t* out_ids, uint32_t* out_sqdist,
                        uint32_t* out_len, double* out_sqdist_f64, cudaStream_t st);

// datagen.cu
hcg_status gen_rows(uint64_t first, uint64_t stride, uint64_t count, uint8_t* out, cudaStream_t st);
hcg_status gen_queries(uint64_t first, uint64_t count, uint64_t n_db, uint8_t* out, cudaStream_t st);

}  // namespace hcg
