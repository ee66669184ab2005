/*
 * raster_gpu.h — C-ABI of the B200 (sm_100a) implementation of RASTER's
 * contraction + agglomeration hot path.
 *
 * The reference (/root/reference/proj/include/raster, header-only C++20) has
 * no FFI layer: its boundary is the C++ API that pipeline.hpp and user code
 * call. Each entry point below names the reference member/function it
 * replaces (file:line, paths relative to proj/include/raster/). A C++ adapter
 * that restores the exact reference signatures over the reference types sits
 * in include/raster_b200/gpu.hpp; other languages bind these symbols directly
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - Plain pointers and sizes only. Points are interleaved float64 (x, y)
 *     pairs: exactly the bytes of a std::span<const raster::Point>
 *     (core.hpp:14-19), i.e. `const double* xy` of length 2*n.
 *   - Tiles are (int64 tx, int64 ty) as raster::Tile (core.hpp:48-54).
 *   - rg_memkind says whether a buffer lives in host memory (pageable or
 *     pinned; the library stages it through HBM) or in device memory of the
 *     context's GPU (zero-copy).
 *   - One context = one accumulator = one CUDA stream. Calls on one context
 *     must not overlap; distinct contexts may be used concurrently
 *     (accumulator.hpp:106-108: "A single accumulator is single-writer").
 *   - Every call returns an rg_status; rg_last_error() gives the message.
 *     Status codes map onto the reference exception hierarchy
 *     (errors.hpp:9-48) — see rg_status.
 *   - There is no CPU fallback: without a usable sm_100 device rg_create
 *     fails with RG_ERR_CUDA.
 */
#ifndef RASTER_GPU_H_
#define RASTER_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RG_ABI_VERSION 1

/* Status codes. Reference exception each one maps onto in the adapter:   */
typedef enum rg_status {
    RG_OK = 0,
    RG_ERR_CONFIG = 1,      /* raster::ConfigError      errors.hpp:15-18   */
    RG_ERR_OOB = 2,         /* raster::OutOfBoundsError errors.hpp:39-42   */
    RG_ERR_CUDA = 3,        /* raster::Error            errors.hpp:9-12    */
    RG_ERR_OOM = 4,         /* raster::Error (device allocation failed)    */
    RG_ERR_STATE = 5,       /* raster::Error (call out of order)           */
    RG_ERR_ARG = 6,         /* raster::Error (null pointer / bad size)     */
    RG_ERR_UNSUPPORTED = 7  /* raster::ConfigError (feature not on GPU)    */
} rg_status;

typedef enum rg_memkind { RG_MEM_HOST = 0, RG_MEM_DEVICE = 1 } rg_memkind;

/* raster::Metric core.hpp:71 */
typedef enum rg_metric { RG_METRIC_CHEBYSHEV = 0, RG_METRIC_MANHATTAN = 1 } rg_metric;
/* raster::Mode core.hpp:74 */
typedef enum rg_mode { RG_MODE_COUNT_ONLY = 0, RG_MODE_RETAIN_POINTS = 1 } rg_mode;
/* raster::OobPolicy core.hpp:77 */
typedef enum rg_oob { RG_OOB_SKIP = 0, RG_OOB_STRICT = 1 } rg_oob;

/* raster::GridParams core.hpp:84-93 (same fields, same defaults), plus a
 * sizing hint for the device hash table (0 = automatic). */
typedef struct rg_params {
    double precision;          /* p: scale = pow(10, p)            default 3.5 */
    double x_min, x_max;       /* Bounds core.hpp:27-31     default -180, 180 */
    double y_min, y_max;       /*                           default  -90,  90 */
    uint64_t threshold;        /* tau                              default 5   */
    int32_t distance;          /* delta                            default 1   */
    int32_t metric;            /* rg_metric                        chebyshev   */
    uint64_t min_cluster_size; /* mu                               default 4   */
    int32_t mode;              /* rg_mode                          count_only  */
    int32_t oob_policy;        /* rg_oob                           skip        */
    int32_t dedupe_points;     /* retain mode: thresholds and cluster points on
                                  unique coordinates (accumulator.hpp:199-204) */
    int32_t reserved0;
    uint64_t capacity_hint;    /* expected distinct tiles; 0 = automatic       */
} rg_params;

/* raster::PipelineStats pipeline.hpp:64-72, with device-side phase times. */
typedef struct rg_stats {
    uint64_t n_points;                 /* ingested + skipped  pipeline.hpp:113 */
    uint64_t n_ingested;               /* accumulator.hpp:194                  */
    uint64_t n_skipped;                /* accumulator.hpp:197                  */
    uint64_t peak_accumulator_entries; /* distinct tiles D    pipeline.hpp:100 */
    uint64_t n_significant;            /* S                   pipeline.hpp:116 */
    uint64_t n_components;             /* components before the mu filter      */
    uint64_t n_clusters;               /* C                                    */
    uint64_t table_capacity;           /* device hash-table slots              */
    uint64_t table_grows;              /* rehashes performed so far            */
    double ms_contract;                /* device time of ingest kernels        */
    double ms_prune;                   /* device time of compaction            */
    double ms_agglomerate;             /* device time of CC + filter + relabel */
    double ms_label;                   /* device time of per-point labelling   */
} rg_stats;

typedef struct rg_ctx rg_ctx;

/* Library facts. */
int rg_abi_version(void);
const char* rg_status_string(rg_status s);
/* Number of usable sm_100 devices (0 when none; never fails). */
int rg_device_count(void);

/* GridParams{} defaults (core.hpp:84-93). */
void rg_params_default(rg_params* out);

/* GridParams::validate core.hpp:98-115 (plus the GPU key-packing limit:
 * columns and rows of the canvas must fit a 63-bit packed key). Usable
 * without a GPU. Writes the message into err (may be NULL). */
rg_status rg_params_validate(const rg_params* p, char* err, size_t err_len);

/* Host-side facts used for parity: GridParams::scale core.hpp:95,
 * min_column/max_column core.hpp:117-122, tile_bound core.hpp:126-131. */
double rg_params_scale(const rg_params* p);
int64_t rg_params_min_column(const rg_params* p);
int64_t rg_params_max_column(const rg_params* p);
double rg_params_tile_bound(const rg_params* p);

/* TileAccumulator(GridParams) accumulator.hpp:111-115: validates and
 * allocates the device accumulator on `device` (-1 = current device). */
rg_status rg_create(const rg_params* p, int device, rg_ctx** out);
void rg_destroy(rg_ctx* ctx);
/* Message of the last failed call on ctx (or of the last failed rg_create
 * when ctx is NULL). Never NULL. */
const char* rg_last_error(const rg_ctx* ctx);

/* Run the context's work on a caller stream (cudaStream_t as void*), e.g.
 * torch.cuda.current_stream().cuda_stream. NULL restores the private one;
 * pass cudaStreamLegacy ((void*)1) for the legacy default stream (handle 0
 * would mean "private"). */
rg_status rg_set_stream(rg_ctx* ctx, void* stream);
rg_status rg_synchronize(rg_ctx* ctx);

/* Empty the context into a fresh accumulator (as constructing a new
 * TileAccumulator, accumulator.hpp:111-115), keeping its device buffers for
 * reuse: counts, totals, significant set and clusters are discarded. */
rg_status rg_reset(rg_ctx* ctx);

/* TileAccumulator::ingest accumulator.hpp:117-134 (+ io.hpp:226-241).
 * Repeatable; chunks may come in any order and partition. Skip policy:
 * out-of-bounds points (closed canvas, NaN included) are counted in
 * n_skipped. Strict policy: returns RG_ERR_OOB naming the first
 * out-of-bounds point in input order; every point before it has been
 * ingested, none after it (as the reference's throwing loop). */
rg_status rg_ingest(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind);

/* Streaming ingest: what ingest_all (io.hpp:226-241) does with a chunked
 * PointSource (io.hpp:21-36), with the source's next read overlapped with
 * the previous chunk's host-to-device copy and contraction.
 *   rg_stream_begin(ctx, chunk)   two pinned host buffers of `chunk` points
 *                                 (0: 4 Mi points)
 *   rg_stream_buffer(ctx, &buf, &cap)  the next buffer to fill (waits until
 *                                 its previous copy has left it)
 *   rg_stream_submit(ctx, n)      ingest its first n points; returns at once
 *   rg_stream_end(ctx)            waits for every chunk; counters are final
 * The accumulator semantics are those of rg_ingest on each chunk in order
 * (strict policy: the first out-of-bounds point ends the stream with
 * RG_ERR_OOB after the points before it). */
rg_status rg_stream_begin(rg_ctx* ctx, uint64_t chunk_points);
rg_status rg_stream_buffer(rg_ctx* ctx, double** buf, uint64_t* capacity);
rg_status rg_stream_submit(rg_ctx* ctx, uint64_t n);
rg_status rg_stream_end(rg_ctx* ctx);

/* TileAccumulator::merge accumulator.hpp:137-154: folds src into dst (counts
 * add); src is left empty. Both must have equal params. */
rg_status rg_merge(rg_ctx* dst, rg_ctx* src);

/* Copy of an accumulator (the reference's TileAccumulator copy, e.g.
 * test_agglomerate.cpp:268): a new context with equal params holding the
 * same counts and totals. */
rg_status rg_clone(rg_ctx* src, rg_ctx** out);

/* Packed tile keys (see rg_device_view) of the accumulator's grid:
 * key = (tx - origin_x) << bits_y | (ty - origin_y). */
rg_status rg_key_packing(rg_ctx* ctx, int64_t* origin_x, int64_t* origin_y, uint32_t* bits_y);

/* Entries of the accumulator as (packed key, count) pairs, unsorted — the
 * for_each_count view (accumulator.hpp:188-191) in a form that can be
 * exchanged between accumulators (multi-GPU merge). *n_out = D; cap = 0
 * only queries D, 0 < cap < D is RG_ERR_ARG with nothing written. keys and
 * counts share `kind`. */
rg_status rg_export_entries(rg_ctx* ctx, uint64_t* keys, uint64_t* counts, uint64_t cap,
                            uint64_t* n_out, rg_memkind kind);

/* Multi-rank routing of exported pairs (device pointers): pair i goes to
 * part p = number of bin_splits[0 .. n_parts-2] <= bin, where
 * bin = ((key >> key_bits_y) - col_min) * 4096 / col_width (the column
 * histogram bins the ranks agreed on). out_keys / out_counts receive the
 * pairs grouped by part (part order; order inside a part unspecified);
 * part_counts[n_parts] (device) the pairs per part. n_parts <= 1024. */
rg_status rg_route_pairs(rg_ctx* ctx, const uint64_t* keys, const uint64_t* counts, uint64_t n,
                         int64_t col_min, uint64_t col_width, const uint32_t* bin_splits,
                         uint32_t n_parts, uint64_t* out_keys, uint64_t* out_counts,
                         uint64_t* part_counts);

/* Adds (packed key, count) pairs produced by rg_export_entries of an
 * accumulator with equal params: the counts-add half of
 * TileAccumulator::merge (accumulator.hpp:137-154) for pairs that arrive
 * over the network. total_ingested grows by the summed counts. Keys are
 * checked first: a key that is not a packed key of this context (all ones,
 * or bits above the column and row fields) fails the call with RG_ERR_ARG
 * and nothing is added. */
rg_status rg_ingest_counts(rg_ctx* ctx, const uint64_t* keys, const uint64_t* counts,
                           uint64_t n, rg_memkind kind);

/* Accessors (accumulator.hpp:176-197). */
rg_status rg_entry_count(rg_ctx* ctx, uint64_t* out);      /* :177 */
rg_status rg_total_ingested(rg_ctx* ctx, uint64_t* out);   /* :194 */
rg_status rg_skipped(rg_ctx* ctx, uint64_t* out);          /* :197 */
rg_status rg_count_of(rg_ctx* ctx, int64_t tx, int64_t ty, uint64_t* out); /* :179 */
/* for_each_count :188-191 as a snapshot, lexicographically sorted. Writes
 * min(cap, entry_count) rows; *n_out = entry_count. Buffers are host. */
rg_status rg_export_counts(rg_ctx* ctx, int64_t* tx, int64_t* ty, uint64_t* count,
                           uint64_t cap, uint64_t* n_out);

/* TileAccumulator::prune accumulator.hpp:156-174: keeps tiles with
 * count >= threshold on the device. The accumulator is consumed: the next
 * rg_ingest starts from an empty table, as after the reference's prune. */
rg_status rg_prune(rg_ctx* ctx, uint64_t* n_significant);

/* window_fix agglomerate.hpp:212-246, the alternative to rg_prune: an
 * occupied tile is significant when some 2x2 window containing it holds
 * >= threshold points (a superset of rg_prune's set). Consumes the
 * accumulator like rg_prune (the reference's window_fix takes a const
 * accumulator: run it on an rg_clone to keep the original). */
rg_status rg_window_fix(rg_ctx* ctx, uint64_t* n_significant);

/* agglomerate(SignificantTiles, params) agglomerate.hpp:196-201 entry with
 * caller-supplied tiles (any order, no duplicates). Replaces whatever the
 * context held. Counts may be NULL. */
rg_status rg_load_significant(rg_ctx* ctx, const int64_t* tx, const int64_t* ty,
                              const uint64_t* count, uint64_t n, rg_memkind kind);

/* agglomerate agglomerate.hpp:196-201 = connected_components :124-170 +
 * erase_if(size < mu) :198-199 + finalize_clusters :175-191, on the device.
 * Requires a pruned or loaded significant-tile set. */
rg_status rg_agglomerate(rg_ctx* ctx, uint64_t* n_clusters);

/* cluster_sequential pipeline.hpp:92-126 over one span of points:
 * ingest + prune + agglomerate. stats may be NULL. */
rg_status rg_cluster(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                     rg_stats* stats);

/* cluster_sequential with its options (pipeline.hpp:92-108): flags is a
 * bitwise OR of RG_CLUSTER_* (RG_CLUSTER_WINDOW_FIX = use_window_fix). */
#define RG_CLUSTER_WINDOW_FIX 1u
rg_status rg_cluster_ex(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                        uint32_t flags, rg_stats* stats);

/* The prune + agglomerate half of cluster_sequential (pipeline.hpp:103-108)
 * on what the context has accumulated so far (rg_ingest / rg_ingest_counts /
 * rg_merge), with one host synchronisation: the owner step of a multi-rank
 * run, whose counts arrive through rg_ingest_counts. flags as rg_cluster_ex;
 * stats may be NULL. */
rg_status rg_prune_agglomerate(rg_ctx* ctx, uint32_t flags, rg_stats* stats);

/* RASTER' output (Mode::retain_points: take_points agglomerate.hpp:70-76 and
 * the point sort of finalize_clusters :183): every in-bounds point of xy
 * whose tile belongs to a kept cluster, grouped by cluster id and ordered by
 * point_less (core.hpp:22-24) within a cluster; with dedupe_points, equal
 * points of a cluster appear once (TileAccumulator::dedupe
 * accumulator.hpp:199-204). Pass the points that were clustered. Results
 * stay in the context (*n_points = M, *n_clusters = C) until
 * rg_get_cluster_points copies them out. n < 2^32 - 1 per call. */
rg_status rg_cluster_points(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                            uint64_t* n_points, uint64_t* n_clusters);
/* Copies min(cap, M) points (x, y interleaved) and the C + 1 cluster offsets
 * (cluster k = points [offsets[k], offsets[k+1])). Either pointer may be
 * NULL; both are `kind` memory. */
rg_status rg_get_cluster_points(rg_ctx* ctx, double* xy, uint64_t cap, uint64_t* offsets,
                                rg_memkind kind);

/* Significant tiles after prune/agglomerate, sorted lexicographically by
 * tile (the canonical order of finalize_clusters), with counts and cluster
 * ids (-1: component dropped by the mu filter, or not agglomerated yet).
 * Writes min(cap, S) rows; any output pointer may be NULL. */
rg_status rg_get_significant(rg_ctx* ctx, int64_t* tx, int64_t* ty, uint64_t* count,
                             int64_t* cluster_id, uint64_t cap, rg_memkind kind);

/* Per-cluster facts in id order: number of tiles, number of points (sum of
 * tile counts), smallest tile (= Cluster::tiles.front()). Any pointer may be
 * NULL; writes min(cap, C) rows. */
rg_status rg_get_clusters(rg_ctx* ctx, uint64_t* n_tiles, uint64_t* n_points,
                          int64_t* first_tx, int64_t* first_ty, uint64_t cap,
                          rg_memkind kind);

/* Device-resident result views (owned by ctx; valid until the next
 * mutating call). Unsorted: entry i of key/count/cluster_id describe the
 * same tile; decode a key with rg_decode_key. */
typedef struct rg_device_view {
    const uint64_t* key;        /* packed tile keys, S entries            */
    const uint64_t* count;      /* point counts,    S entries             */
    const int32_t* cluster_id;  /* canonical id or -1, S entries          */
    uint64_t n_significant;
    uint64_t n_clusters;
    int64_t origin_x, origin_y; /* tile = origin + unpacked key           */
    uint32_t key_bits_y;        /* key = (tx-origin_x) << bits_y | (ty-origin_y) */
    uint32_t reserved;
} rg_device_view;
rg_status rg_device_result(rg_ctx* ctx, rg_device_view* out);
void rg_decode_key(const rg_device_view* v, uint64_t key, int64_t* tx, int64_t* ty);

/* Point-retaining variant (RASTER', Mode::retain_points): int32 cluster id
 * of every input point, -1 for out-of-bounds points and points whose tile
 * is not in a kept cluster. This is the input-order form of
 * Cluster::points (accumulator.hpp:131, agglomerate.hpp:70-76,183) and of
 * labeled_points metrics.hpp:78-83. xy and labels share `kind`. */
rg_status rg_label_points(rg_ctx* ctx, const double* xy, uint64_t n, int32_t* labels,
                          rg_memkind kind);

rg_status rg_get_stats(rg_ctx* ctx, rg_stats* out);

/* Number of device kernels this context has launched (for launch
 * accounting in benchmarks). */
uint64_t rg_kernel_launches(const rg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* RASTER_GPU_H_ */
