/*
 * hcg.h -- C ABI of the B200-native Hypercurves/Multicurves kNN hot path.
 *
 * Plain C: no torch, no C++ types, no exceptions cross this boundary.  Every
 * entry point returns an hcg_status; on failure hcg_last_error() holds a
 * thread-local message.  The C++ wrapper in hypercurves_b200.hpp maps the codes
 * back to the reference's exception types (std::invalid_argument for
 * HCG_EINVAL / HCG_ECAPACITY / HCG_ENONFINITE, std::runtime_error otherwise),
 * as the reference throws them (curve.cpp:35-59,167; vecio.cpp:15,78,88,116).
 *
 * Which reference interface each entry point replaces (paths relative to the
 * reference root):
 *   hcg_make_lut       quantize_component over the 256 byte values of a view
 *                      (proj/src/curve.cpp:166-174; bvecs widening vecio.cpp:50-51)
 *   hcg_build          hc::MulticurvesIndex(const Dataset&, ProjectionScheme)
 *                      (proj/include/hypercurves/multicurves.hpp:77; Alg. 1)
 *   hcg_search         hc::MulticurvesIndex::search(q, SearchParams) batched
 *                      (multicurves.hpp:81; Alg. 2)
 *   hcg_keys           hc::curve_encode(kind, project(v, scheme, c))  (curve.cpp:162-164,
 *                      multicurves.hpp:40)
 *   hcg_sorted         hc::SubIndex::entries()            (multicurves.hpp:55)
 *   hcg_windows        hc::SubIndex::rank_of / window     (multicurves.hpp:57-63)
 *   hcg_candidates     hc::MulticurvesIndex::candidate_union (multicurves.hpp:87-89)
 *   hcg_brute_force    hc::brute_force_knn                (proj/src/vecio.cpp:115-122)
 *   hcg_search_packed  per-shard search of hypershard's IHLS stage
 *   hcg_merge_packed   hypershard aggregate: k-way merge by (distance, id)
 *
 *   hcg_miss_bound /   equivalence module: binomial_tail / miss_bound / plan_depth
 *   hcg_plan_depth
 *   hcg_insert         hc::MulticurvesIndex::insert, batched (multicurves.hpp:79)
 *   hcg_save/hcg_load  hc::MulticurvesIndex::save / load (multicurves.hpp:96-98)
 *   hcg_read_vectors / hc::read_vectors / write_vectors (proj/src/vecio.cpp:18-85)
 *   hcg_write_vectors
 *   hcg_gen_rows /     the counter-based synthetic SIFT-like generator of
 *   hcg_gen_queries    SURVEY.md §8(d) (bench/test data; bit-identical to the oracle)
 *   hcg_shard_group_*  hypershard module: partition / broadcast / IHLS / aggregate
 *                       over G GPUs with NCCL
 *   hcg_server_*       dtahe module: Alg. 3's buffer dispatch (
 *                      SPEC.md:421-510) as a GPU batch-size controller
 *
 * Data model.  Descriptors are byte vectors (bvecs).  The reference sees each
 * byte b through a "view" v(b) (raw: float(b); lifted: 1 + b/256).  The
 * quantizer only ever sees those 256 values, so the scheme carries the 256
 * quantized cells (hcg_make_lut computes them with the reference's
 * float_to_ordinal >> (32 - m) rule) and a distance scale: the reference's
 * squared distance is exactly sqdist_u32 * dist_scale^2 for affine views with a
 * power-of-two scale, so search results are bit-exact in both views.
 *
 * Pointers.  Every data pointer may be host memory (pageable or pinned) or
 * device memory of the index's device; the library stages host buffers itself
 * (cudaMemcpyAsync on `stream`) and synchronises `stream` before returning
 * whenever an output lives in host memory.  With all-device buffers the calls
 * are stream-ordered and asynchronous.  `stream` may be NULL (legacy default
 * stream).
 *
 * Threading.  One index lives on one device.  Concurrent searches on one index
 * from different streams/threads are allowed (search is const);
 * build and free are exclusive.
 */
#ifndef HCG_H
#define HCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hcg_status {
    HCG_OK = 0,
    HCG_EINVAL = -1,      /* precondition violated (reference: std::invalid_argument) */
    HCG_ECAPACITY = -2,   /* key width / k / depth beyond capacity (curve.cpp:43-45)  */
    HCG_ENONFINITE = -3,  /* NaN/Inf component (curve.cpp:167)                        */
    HCG_ENOMEM = -4,      /* device allocation failed                                  */
    HCG_ECUDA = -5,       /* CUDA runtime error                                        */
    HCG_ENODEV = -6,      /* no usable sm_100 device                                   */
    HCG_EIO = -7          /* file I/O or format error (reference: std::runtime_error)  */
} hcg_status;

typedef enum hcg_curve_kind { HCG_ZORDER = 0, HCG_HILBERT = 1 } hcg_curve_kind;

/* Element type of the descriptors.  HCG_U8: bytes (bvecs) seen through the
 * scheme's view (cell_lut, dist_scale), distances exact integers.  HCG_F32:
 * the reference's float components as-is (fvecs): quantized on the device by
 * float_to_ordinal >> (32 - m) (curve.cpp:166-174), squared distances
 * accumulated in double exactly as vecio.cpp:87-95 does (the same terms,
 * summed sequentially in index order: the same double, bit for bit), searched
 * with hcg_search_f32. */
typedef enum hcg_dtype { HCG_U8 = 0, HCG_F32 = 1 } hcg_dtype;

#define HCG_MAX_KEY_BITS 1024  /* HC_MAX_KEY_BITS, keys.hpp:15-23 */
#define HCG_MAX_CURVE_DIMS 128 /* dims feeding one curve          */
#define HCG_MAX_K 256          /* largest k of the warp top-k      */
#define HCG_MAX_ROW_BYTES 512  /* descriptor length (bytes): 512 u8 / 128 f32 */

/* ProjectionScheme (multicurves.hpp:18-32) plus the view of the bytes. */
typedef struct hcg_scheme {
    uint32_t d_full;            /* bytes per descriptor                            */
    uint32_t curves;            /* number of subindexes                            */
    uint32_t bits_per_dim;      /* m in [1, 32]                                    */
    uint32_t curve_kind;        /* hcg_curve_kind                                  */
    const uint32_t* assign_off; /* curves+1 offsets into assign                    */
    const uint32_t* assign;     /* assign[assign_off[c] + s] = input dim of slot s */
    uint32_t cell_lut[256];     /* HCG_U8: quantized cell of each byte value        */
    double dist_scale;          /* HCG_U8 view scale: distance = sqrt(sqdist)*scale */
    uint32_t dtype;             /* an hcg_dtype; 0 = HCG_U8                        */
    float view_offset;          /* HCG_U8: byte b is the float view_offset + b *   */
                                /* dist_scale (kept with the index for wrappers)   */
} hcg_scheme;

typedef struct hcg_index hcg_index;

const char* hcg_last_error(void);
const char* hcg_version(void);

/* Quantized cell of every byte value for the affine view v(b) = offset + b*scale
 * (computed in f32 exactly like the reference's widened components).  Fails
 * with HCG_ENONFINITE when a value is not finite and HCG_EINVAL for m outside
 * [1, 32]. */
hcg_status hcg_make_lut(float offset, float scale, uint32_t bits_per_dim, uint32_t* lut256);

/* Round-robin assignment, seed 0: dim j -> curve j % curves,
 * slot j / curves.  assign_off has curves+1 entries, assign has d_full. */
hcg_status hcg_default_assignment(uint32_t d_full, uint32_t curves, uint32_t* assign_off,
                                  uint32_t* assign);

/* Build an index over n descriptors (rows: n x d_full elements of the scheme's
 * dtype; every `rows` / `queries` pointer below is d_full elements per row).  The id of row s
 * is id_base + s * id_stride (the dataset's ids 0..n-1 are base 0, stride 1; a
 * shard of `id mod G` partitioning is base r, stride G).  The index copies the
 * rows into HBM and owns all device memory. */
hcg_status hcg_build(const hcg_scheme* scheme, const uint8_t* rows, uint64_t n, uint64_t id_base,
                     uint64_t id_stride, int device, void* stream, hcg_index** out);
hcg_status hcg_free(hcg_index* index);

uint64_t hcg_size(const hcg_index* index);
uint32_t hcg_curves(const hcg_index* index);
/* 64-bit words of the full key of curve c: ceil(dims_c * m / 64). */
uint32_t hcg_key_words(const hcg_index* index, uint32_t curve);
/* Device bytes owned by the index. */
uint64_t hcg_device_bytes(const hcg_index* index);
uint32_t hcg_index_dtype(const hcg_index* index); /* hcg_dtype of the rows */
/* Kernels this library has launched (searches, merges, sorts), for launch accounting. */
uint64_t hcg_launch_count(void);

/* Batched search: for each of nq queries (nq x d_full bytes) the top-k of the
 * deduplicated union of every curve's probe-depth window, ordered by
 * (squared distance, id).  out_ids / out_sqdist are nq x k; entries at or past
 * out_len[q] are id UINT64_MAX, sqdist UINT32_MAX.  The reference's rooted
 * distance is sqrt((double)sqdist) * dist_scale. */
hcg_status hcg_search(const hcg_index* index, const uint8_t* queries, uint32_t nq, uint32_t k,
                      uint32_t depth, uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len,
                      void* stream);

/* hcg_search with per-kernel device times: records CUDA events around the
 * launches on `stream` and synchronises it.  ms_out[0] = locate (keys +
 * lower_bound + windows), ms_out[1] = candidate union (dedup; 0 when fused
 * into the refine kernel), ms_out[2] = gather + exact L2 + top-k
 * (instrumentation for bench.py). */
hcg_status hcg_search_timed(const hcg_index* index, const uint8_t* queries, uint32_t nq, uint32_t k,
                            uint32_t depth, uint64_t* out_ids, uint32_t* out_sqdist,
                            uint32_t* out_len, float* ms_out, void* stream);

/* hcg_search for an HCG_F32 index: queries are nq x d_full floats, out_sqdist
 * are the reference's squared distances in double (distance = sqrt).  Fails
 * with HCG_ENONFINITE on a NaN/Inf query component (curve.cpp:167). */
hcg_status hcg_search_f32(const hcg_index* index, const float* queries, uint32_t nq, uint32_t k,
                          uint32_t depth, uint64_t* out_ids, double* out_sqdist, uint32_t* out_len,
                          void* stream);

/* Per-shard search writing packed (sqdist << 32 | id) u64 per result, nq x k,
 * padding UINT64_MAX; requires ids < 2^32.  Input to hcg_merge_packed. */
hcg_status hcg_search_packed(const hcg_index* index, const uint8_t* queries, uint32_t nq,
                             uint32_t k, uint32_t depth, uint64_t* out_packed, void* stream);

/* k-way merge of `parts` packed lists (parts x nq x k, each sorted ascending)
 * into the global top-k per query.  device = CUDA device of
 * the buffers. */
hcg_status hcg_merge_packed(const uint64_t* packed, uint32_t parts, uint32_t nq, uint32_t k,
                            uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, int device,
                            void* stream);

/* Append n rows (ids continue the affine sequence: id_base + s * id_stride for
 * s = size..size+n-1) and merge their keys into every curve.  The result is
 * identical to building over the union (SPEC.md:227-235 order independence).
 * Exclusive with searches on the same index. */
hcg_status hcg_insert(hcg_index* index, const uint8_t* rows, uint64_t n, void* stream);

/* Little-endian binary persistence (SPEC.md:268 leaves the layout open):
 * "HCGIDX" header with the scheme, n, ids and view, the descriptor rows, then
 * per curve its common key prefix and the sorted (suffix key, slot) arrays.
 * Round-trips bit-exactly (tests/test_gpu_formats.py). */
hcg_status hcg_save(const hcg_index* index, const char* path);
hcg_status hcg_load(const char* path, int device, void* stream, hcg_index** out);

/* ---- bvecs / fvecs records (vecio.cpp:18-85): u32 LE dim + payload ---- */
typedef enum hcg_vector_format { HCG_FVECS = 0, HCG_BVECS = 1, HCG_FVECS_F32 = 2 } hcg_vector_format;
/* *rows_out is malloc'ed; release with hcg_free_buffer.  HCG_BVECS / HCG_FVECS:
 * n x dim bytes, fvecs components must be byte values of the view
 * offset + b * scale.  HCG_FVECS_F32: n x dim floats as stored (offset and
 * scale unused), the rows of an HCG_F32 index. */
hcg_status hcg_read_vectors(const char* path, uint32_t format, float offset, float scale, uint8_t** rows_out,
                            uint64_t* n_out, uint32_t* dim_out);
hcg_status hcg_write_vectors(const char* path, uint32_t format, float offset, float scale, const uint8_t* rows,
                             uint64_t n, uint32_t dim);
void hcg_free_buffer(void* p);

/* ---- parity taps ---- */
/* Full-width keys (hcg_key_words words per key, least significant word first,
 * as ExtendedKey::words) of n arbitrary rows on curve c. */
hcg_status hcg_keys(const hcg_index* index, const uint8_t* rows, uint64_t n, uint32_t curve,
                    uint64_t* out_words, void* stream);
/* Sorted subindex c: ids (n) and, when out_words != NULL, full keys (n x words). */
hcg_status hcg_sorted(const hcg_index* index, uint32_t curve, uint64_t* out_ids,
                      uint64_t* out_words, void* stream);
/* Ids of positions [begin, begin + count) of sorted subindex c
 * (SubIndex::entries() slice; retrieve_candidates = hcg_windows + this). */
hcg_status hcg_sorted_range(const hcg_index* index, uint32_t curve, uint64_t begin, uint64_t count,
                            uint64_t* out_ids, void* stream);
/* The scheme an index was built with (hcg_load callers recover it here).
 * *assign_len receives the assignment length; with assign_off / assign NULL
 * only the sizes are reported, else out->assign_off / out->assign point at
 * the caller's arrays (curves + 1 and *assign_len entries). */
hcg_status hcg_describe(const hcg_index* index, hcg_scheme* out, uint32_t* assign_off, uint32_t* assign,
                        uint32_t* assign_len);
/* rank_of and window [begin, end) of every (query, curve), nq x curves each. */
hcg_status hcg_windows(const hcg_index* index, const uint8_t* queries, uint32_t nq, uint32_t depth,
                       uint64_t* out_rank, uint64_t* out_begin, uint64_t* out_end, void* stream);
/* Deduplicated candidate ids per query (set semantics, order unspecified):
 * out_ids is nq x cap, out_count[q] the number of unique candidates.  Fails
 * with HCG_ECAPACITY when a query has more than cap candidates.  With
 * out_ids == NULL and cap == 0 only the counts are produced. */
hcg_status hcg_candidates(const hcg_index* index, const uint8_t* queries, uint32_t nq,
                          uint32_t depth, uint64_t* out_ids, uint32_t cap, uint32_t* out_count,
                          void* stream);

/* Exact kNN over the index's rows (ground truth for recall, vecio.cpp:115-122). */
hcg_status hcg_brute_force(const hcg_index* index, const uint8_t* queries, uint32_t nq, uint32_t k,
                           uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len,
                           void* stream);
/* hcg_brute_force for an HCG_F32 index (double squared distances; +inf and
 * id UINT64_MAX pad lists shorter than k). */
hcg_status hcg_brute_force_f32(const hcg_index* index, const float* queries, uint32_t nq, uint32_t k,
                               uint64_t* out_ids, double* out_sqdist, uint32_t* out_len,
                               void* stream);

/* ---- sharded search over G GPUs: the hypershard module (
 * PAPER.md:743-822) ----
 * Global id i lives on shard i mod G at local slot i / G (partition,
 * SPEC.md:357-365).  A search gives every shard the whole query batch
 * (broadcast), runs each shard's search at the per-shard
 * probe depth (IHLS stage; depth from hcg_plan_depth), all-gathers
 * the packed (sqdist << 32 | id) top-k lists with NCCL over NVLink
 * (B x k x 8 bytes per shard) and merges them by (distance, id), truncated to
 * k (aggregate).  Results equal the reference's sharded
 * search: per-shard MulticurvesIndex::search then the aggregate merge.
 * u8 indexes only (ids < 2^32).  NCCL is loaded at run time (an already
 * loaded libnccl.so.2 first, then $HCG_NCCL_LIB, then the system's). */
typedef struct hcg_shard_group hcg_shard_group;
typedef struct hcg_nccl_id { char internal[128]; } hcg_nccl_id; /* an ncclUniqueId */

/* One process driving G GPUs: shard r is built on devices[r] from rows
 * r, r + G, ... of `rows` (n_total x d_full bytes, host or device memory);
 * communicators from ncclCommInitAll.  Results land on devices[0]. */
hcg_status hcg_shard_group_build(const hcg_scheme* scheme, const uint8_t* rows, uint64_t n_total, uint32_t G,
                                 const int* devices, hcg_shard_group** out);
/* The same over G already-built shards (shard r built with id_base r,
 * id_stride G, one per device); the group takes ownership on success. */
hcg_status hcg_shard_group_adopt(uint32_t G, hcg_index* const* shards, hcg_shard_group** out);
/* One process per GPU: rank `rank` of G joins with its local shard (id_base
 * rank, id_stride G; the caller keeps ownership) through the NCCL id rank 0
 * made with hcg_nccl_unique_id and shared with every rank.  Collective: all
 * G ranks call it together. */
hcg_status hcg_nccl_unique_id(hcg_nccl_id* out);
hcg_status hcg_shard_group_join(const hcg_nccl_id* id, uint32_t rank, uint32_t G, hcg_index* local,
                                hcg_shard_group** out);
hcg_status hcg_shard_group_free(hcg_shard_group* group);
uint32_t hcg_shard_group_shards(const hcg_shard_group* group);
/* Global top-k of nq queries (hcg_search's layout and padding).  queries and
 * outputs: host memory or device memory (of devices[0] / the rank's device;
 * queries may also sit on another GPU).  `stream` belongs to devices[0] (the
 * rank's device); the call is stream-ordered against it and synchronises only
 * when an output is host memory.  Per-process mode: collective, every rank
 * passes the same batch and receives the same result. */
hcg_status hcg_shard_group_search(hcg_shard_group* group, const uint8_t* queries, uint32_t nq, uint32_t k,
                                  uint32_t shard_depth, uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len,
                                  void* stream);

/* The aggregate routed to one aggregator per query (route_to_aggregator,
 * SPEC.md:375-383): in per-process mode rank p receives every shard's
 * partials of the query block [nq*p/G, nq*(p+1)/G) only (NCCL send / recv:
 * 1/G of an all-gather's bytes and of the merge) and writes those rows of the
 * outputs (nq-row buffers); *block_first / *block_count name the block.  In
 * one process (all shards local) it is hcg_shard_group_search (block = all).
 * Collective. */
hcg_status hcg_shard_group_search_routed(hcg_shard_group* group, const uint8_t* queries, uint32_t nq, uint32_t k,
                                         uint32_t shard_depth, uint64_t* out_ids, uint32_t* out_sqdist,
                                         uint32_t* out_len, void* stream, uint32_t* block_first,
                                         uint32_t* block_count);

/* CUDA device of the group's first local shard (where results land) and the
 * descriptor length. */
int hcg_shard_group_device(const hcg_shard_group* group);
/* Shards driven by this process: G for one process over G GPUs, 1 per rank. */
uint32_t hcg_shard_group_local_shards(const hcg_shard_group* group);
uint32_t hcg_shard_group_dims(const hcg_shard_group* group);

/* ---- GPU batch-size controller: DTAHE (Alg. 3, PAPER.md:1177-1191;
 * SPEC.md:421-510) with the CPU branch removed (CC = 0) ----
 * With a slot free (at most `slots` batches in flight: 2 = the double buffer,
 * SPEC.md:436), the server launches min(waiting, max_batch) queries when the
 * device is idle ("GPU idle"), when >= min_batch queries wait ("buffer
 * full"), or when the oldest waiting query has waited max_wait_s; otherwise
 * it keeps buffering.  FIFO dispatch, every query answered exactly once
 * (SPEC.md:491-493).  Serving one index, small batches (<= 512 queries: one
 * SM per query) run side by side on their slots' own streams while their
 * queries fit one CTA per SM and no large batch is in flight; together they
 * count as one of the `slots` stages, and a large batch runs after them.
 * A batch is H2D (host queries -> device) -> search (one index, or a shard
 * group) -> D2H (results -> host), with uploads and downloads overlapping the
 * neighbouring batches' searches; a query's response time runs from its
 * arrival to its results being in host memory. */
typedef struct hcg_server_policy {
    uint32_t max_batch;  /* buffer capacity B                      */
    uint32_t min_batch;  /* launch when this many queries wait      */
    double max_wait_s;   /* launch when the oldest waited this long */
    uint32_t slots;      /* pipeline stages in flight (1..8)         */
} hcg_server_policy;
typedef struct hcg_server hcg_server;

/* Serve exactly one of `index` (u8) / `group` (one process over all its GPUs;
 * a per-rank group is rejected: its searches are collective) with fixed k and
 * probe depth (per-shard depth for a group).  policy NULL: {8192, 1, 0, 2}. */
hcg_status hcg_server_create(const hcg_index* index, hcg_shard_group* group, uint32_t k, uint32_t depth,
                             const hcg_server_policy* policy, hcg_server** out);
hcg_status hcg_server_free(hcg_server* server);
/* Open-loop replay: query i (row i of `queries`, host memory) arrives
 * arrival_s[i] seconds after the start (non-decreasing).  Results (host,
 * nq x k, hcg_search's layout) and latency_s[i] = completion - arrival.
 * batch_sizes (optional, capacity nq) / n_batches: the launched batches. */
hcg_status hcg_server_replay(hcg_server* server, const uint8_t* queries, uint32_t nq, const double* arrival_s,
                             uint64_t* out_ids, uint32_t* out_sqdist, uint32_t* out_len, double* latency_s,
                             uint32_t* batch_sizes, uint32_t* n_batches);
/* Online serving: start a dispatcher thread with a pinned ring of `capacity`
 * queries; submit copies queries in and returns a ticket (it blocks while
 * `capacity` submitted queries await collection); wait blocks until the
 * ticket's queries are answered and copies their results (and response times)
 * out, freeing their ring space.  Thread-safe; a replay and an online session
 * do not run at the same time on one server. */
hcg_status hcg_server_start(hcg_server* server, uint64_t capacity);
hcg_status hcg_server_submit(hcg_server* server, const uint8_t* queries, uint32_t nq, uint64_t* ticket);
hcg_status hcg_server_wait(hcg_server* server, uint64_t ticket, uint64_t* out_ids, uint32_t* out_sqdist,
                           uint32_t* out_len, double* latency_s);

/* 1 when a search of nq queries at (k, depth) runs the union-less refine
 * kernel (k_gather_nu: window walk + gather + top-k with repeats dropped),
 * 0 when it runs the separate candidate union + gather (instrumentation for
 * the byte model of bench.py). */
uint32_t hcg_refine_unionless(const hcg_index* index, uint32_t nq, uint32_t k, uint32_t depth);

/* CUDA device of an index, and its id map (id of slot s = base + s * stride). */
int hcg_index_device(const hcg_index* index);
hcg_status hcg_index_ids(const hcg_index* index, uint64_t* id_base, uint64_t* id_stride);

/* ---- probe-depth planner (equivalence module, host math) ---- */
/* P[Bin(trials, p) > phi]. */
double hcg_binomial_tail(uint32_t trials, double p, uint32_t phi);
/* 1 - max(0, 1 - Phi * P[Bin(Phi, 1/shards) > phi])^2 clamped to [0,1]
 * (PAPER.md:895-896). */
double hcg_miss_bound(uint32_t Phi, uint32_t shards, uint32_t phi);
/* Smallest phi <= Phi with miss_bound <= target. */
uint32_t hcg_plan_depth(uint32_t Phi, uint32_t shards, double target);

/* ---- synthetic data; out is a device pointer ---- */
/* Row i of the output is generator row first + i * stride (128 bytes each). */
hcg_status hcg_gen_rows(uint64_t first, uint64_t stride, uint64_t count, uint8_t* out_dev,
                        int device, void* stream);
hcg_status hcg_gen_queries(uint64_t first, uint64_t count, uint64_t n_db, uint8_t* out_dev,
                           int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HCG_H */
