// internal.h — launch interfaces between the C-ABI layer (api.cu) and the
// kernel translation units. Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace rg {

struct ContractLaunch {
    const double* xy;
    u64 n;
    u64 rows_per_seg;
    u64 warps;
    Grid g;
    Table t;
    Counters* ctr;
    const Partial* partial_in;
    u64 n_partial_in;
    Partial* partial_out;
    u64 budget;
    bool narrow;  // canvas column/row indices fit int32
    bool claim128 = false;  // most evictions claim new keys: one 128-bit CAS per claim
};

int contract_max_warps(int n_sm);
int contract_batch_rows();
int contract_block_warps();
cudaError_t launch_contract(const ContractLaunch& L, cudaStream_t st);
cudaError_t launch_table_clear(Slot* slots, u64 n, int n_sm, cudaStream_t st);
cudaError_t launch_table_fold(const Slot* src, u64 n_src, Table dst, u64* claimed, int n_sm,
                              cudaStream_t st);
cudaError_t launch_pairs_fold(const u64* keys, const u64* cnts, u64 n, Table dst, u64* claimed,
                              u64* points, int n_sm, cudaStream_t st);
cudaError_t launch_export(const Slot* slots, u64 cap, u64* keys, u64* cnts, u64* n_out, int n_sm,
                          cudaStream_t st);
cudaError_t launch_first_oob(const double* xy, u64 n, Grid g, u64* first, int n_sm,
                             cudaStream_t st);
// lb_scratch (K2 look-back: cap / 2048 + 2 words) selects the one-pass K2;
// null selects the staged K2 (reservation atomics)
u64 compact_lb_words(u64 cap);
cudaError_t launch_compact_pairs(const uint4* units, const u32* dcnt, u32 n_units, const u64* pkey,
                                 const u32* pcnt, u64 tau, u64* sig_key, u64* sig_cnt,
                                 u32* col_cnt, u32 bits_y, Counters* ctr, int n_sm,
                                 cudaStream_t st);
cudaError_t launch_find_slots(Table t, const u64* sig_key, u64 n, u32* slot_of, int n_sm,
                              cudaStream_t st);
cudaError_t launch_compact(Table t, u64 cap, u64 tau, const u8* keep, u64* sig_key, u64* sig_cnt,
                           u32* parent, u32* size, u64* npts, u64* min_key, int* root_cid,
                           u32* col_cnt, u32* slot_of, Counters* ctr, int n_sm,
                           cudaStream_t st, u64* lb_scratch = nullptr);
cudaError_t launch_mark_sig(Table t, const u32* slot_of, const int* cid, u64 n, int n_sm,
                            cudaStream_t st);
cudaError_t launch_window_mark(Table t, u64 cap, u64 tau, u32 bits_x, u8* keep, int n_sm,
                               cudaStream_t st);

struct AggLaunch {
    const u64* sig_key;
    const u64* sig_cnt;
    const u64* n_sig_dev;  // device copy of S (&ctr->n_sig)
    u64 n_sig;             // host copy of S (for sizing)
    Table t;
    u32 bits_y, bits_x;
    const int2* offsets;
    int n_offsets;
    int cheb1;  // offsets are exactly Chebyshev delta 1
    u64 mu;
    u32* parent;
    u32* size;
    u64* npts;
    u64* min_key;
    int* root_cid;
    int* tile_cid;
    uint2* edges;     // deferred external edges of k_union: 128 slots per 32-tile window
    u32* edge_n;      // edges per window
    u64* root_key;
    u32* root_idx;
    u64* root_key_sorted;
    u32* root_idx_sorted;
    void* sort_temp;
    size_t sort_temp_bytes;
    Counters* ctr;
    int n_sm;
};

cudaError_t launch_agglomerate(const AggLaunch& A, cudaStream_t st);

// K3 over key-sorted tiles (agglomerate_sorted.cu), delta <= 2.
struct SortedLaunch {
    const u64* sig_key;   // bucket order (K2 output)
    const u64* sig_cnt;
    const u64* n_sig_dev;
    u64 n_sig;
    u32 bits_y, key_bits;
    int delta, manhattan;
    u64 mu;
    u32* iota;            // scratch, S
    u64* ktmp;            // scratch, S
    u32* col_cnt;         // column counting sort: 2^bits_x + 1 entries (or null)
    u32* col_off;
    u64* skey;            // sorted keys, S
    u32* perm;            // sorted position -> bucket index, S
    u32* parent;          // sorted space
    u32* size;
    u64* npts;
    u32* flag;
    u32* scan;
    int* tile_cid_b;      // cluster id per bucket index (labelling pass)
    int* cid_s;           // cluster id per sorted position (canonical output)
    u32* clu_root;        // sorted position of cluster k's root
    uint2* edges;
    u64 edge_cap;
    void* temp;
    size_t temp_bytes;
    Counters* ctr;
    Counters* host_ctr;   // pinned mirror: the exact count is read back once
    int n_sm;
    bool col_hist_ready;  // K2 already built col_cnt (prune_enqueue)
    bool* npts_deferred;  // out: per-cluster point totals left for launch_cluster_npts
    bool check_k1_stop = false;  // the host read also checks K1's stop flag (returns
                                 // cudaErrorNotReady, nothing launched after it, if set)
    int* launches;        // out: kernels launched
    bool speculate = false;      // no host read: size for the bound n_sig, assume the bucketed
                                 // path; the caller verifies max_col / K1's stop flag afterwards
    bool* speculated = nullptr;  // out: the launch really went without the host read
};
u64 sorted_bucket_max_column();
size_t sorted_temp_bytes(u64 n, int bits, u32 bits_x);
u64 sorted_columns(u32 bits_x);
cudaError_t launch_agglomerate_sorted(const SortedLaunch& L, cudaStream_t st);
cudaError_t launch_cluster_npts(const int* cid_s, const u32* perm, const u64* cnt_b, u64 n,
                                const u32* clu_root, u64 n_kept, u64* npts, int n_sm,
                                cudaStream_t st);
cudaError_t launch_order_and_label(const AggLaunch& A, u64 n_kept, cudaStream_t st);
size_t sort_pairs_temp_bytes(u64 n, int bits);
cudaError_t sort_pairs(void* temp, size_t temp_bytes, const u64* k_in, u64* k_out,
                       const u32* v_in, u32* v_out, u64 n, int bits, cudaStream_t st);
cudaError_t launch_load_tiles(const long long* tx, const long long* ty, const u64* cnt, u64 n,
                              long long ox, long long oy, u32 bits_y, Table t, u64* sig_key,
                              u64* sig_cnt, u32* parent, u32* size, u64* npts, u64* min_key,
                              int* root_cid, int n_sm, cudaStream_t st);
cudaError_t launch_tile_extents(const long long* tx, const long long* ty, u64 n, long long* out,
                                int n_sm, cudaStream_t st);

// dedupe_points (dedupe.cu)
cudaError_t launch_dedupe_ingest(const double* xy, u64 n, Grid g, PointSet ps, Table ut,
                                 u64* n_new, int n_sm, cudaStream_t st);
cudaError_t launch_ps_fold(const PtKey* src, u64 src_cap, Grid g, PointSet dst, Table ut,
                           u64* n_new, int n_sm, cudaStream_t st);
cudaError_t launch_ps_rehash(const PtKey* src, u64 src_cap, PointSet dst, int n_sm,
                             cudaStream_t st);
cudaError_t launch_dedupe_counts(Table t, u64 cap, Table ut, int n_sm, cudaStream_t st);

// contraction for unordered inputs (partition.cu)
struct PartitionLaunch {
    const double* xy;
    u64 n;
    Grid g;
    u32 key_bits;
    Counters* ctr;
    void* scratch;      // partition_scratch_bytes(n)
    size_t scan_temp;
    u64* pkey;          // n entries: (key, count) pairs, one slab per work unit
    u32* pcnt;
    int n_sm;
    bool narrow;        // canvas indices fit int32 (32-bit projection)
    int* stream_hint;   // caller-owned memo: 1 = the one-pass scatter fell back last time
};
u64 partition_res_entries(u64 n);
bool partition_ingest_supported(u32 key_bits, u64 n);
size_t partition_scratch_bytes(u64 n, size_t* scan_temp);
cudaError_t launch_order_probe(const double* xy, u64 n, Grid g, u64* out, int n_sm,
                               cudaStream_t st);
struct PartitionPlan {
    std::vector<uint4> units;   // (first, end, partition) of every KP2 work unit
    std::vector<u32> dcnt;      // distinct tiles per unit (0xffffffff: overflowed)
    std::vector<u64> pair_off;  // exclusive prefix of dcnt (overflowed units add 0)
                                // (pairs live in per-unit slabs at units[u].x)
    u64 raw_points = 0;         // points of overflowed units (added one by one)
    int launches = 0;           // kernels launched by launch_partition_count
    bool single_units = true;   // every partition is one work unit (its pairs are final counts)
    const uint4* units_dev = nullptr;  // device copies of units / dcnt (in the scratch)
    const u32* dcnt_dev = nullptr;
};
cudaError_t launch_partition_count(const PartitionLaunch& L, cudaStream_t st, PartitionPlan* plan);
cudaError_t launch_partition_insert(const PartitionLaunch& L, Table t, const PartitionPlan& plan,
                                    cudaStream_t st, int blocks_per_sm = 8);
u32 partition_count();

// RASTER' cluster points (points.cu)
struct PointsLaunch {
    const double* xy;
    const int* labels;
    u64 n;
    u64 n_clusters;
    int dedupe;
    u32 *idx_a, *idx_b;   // n entries each
    u64 *key_a, *key_b;   // n + 1 entries each
    u64* m_dev;
    u64* m_host;          // pinned
    void* temp;
    size_t temp_bytes;
    double* out_xy;       // 2 * M doubles
    u64* offsets;         // n_clusters + 1
    int n_sm;
};
size_t cluster_points_temp_bytes(u64 m);
cudaError_t launch_cluster_points(const PointsLaunch& L, cudaStream_t st);

// table_cids: significant count words hold SIG | (cluster id + 1) (else SIG |
// dense index into tile_cid)
struct PointsV2 {
    const double* xy;     // 16-byte aligned
    const int* labels;
    u64 n;
    u64 n_clusters;
    int dedupe;
    u64* cnt;             // C + 1 (counts, then scatter cursors)
    u64* off;             // C + 1 (cluster starts; the offsets without dedupe)
    double2* grp;         // M points grouped by cluster (the output without dedupe)
    u32* flag;            // M (dedupe)
    u32* pos;             // M (dedupe)
    double2* out;         // M (dedupe output)
    u64* out_off;         // C + 1 (dedupe offsets)
    u64* scratch;         // one u64
    void* temp;
    size_t temp_bytes;
    int n_sm;
};
size_t cluster_points_v2_temp_bytes(u64 n, u64 C);
u32 cluster_points_v2_cap();
cudaError_t launch_cluster_points_v2_count(const PointsV2& L, cudaStream_t st, u64* m_host,
                                           u64* max_host);
cudaError_t launch_cluster_points_v2(const PointsV2& L, u64 m, cudaStream_t st);

// K4' for inputs without spatial order: a cell table of the kept tiles
// (8 x 8-tile cells, 16-byte entries, L2-sized; label.cu)
u64 cell_buckets(u64 cells);
cudaError_t launch_cells_build(const u64* skey, const int* cid, const u64* n_dev, u64 n_bound,
                               ulonglong2* tab, u64 nb, u32 bits_y, u64* counters, int n_sm,
                               cudaStream_t st);
cudaError_t launch_cells_mixed(const u64* skey, const int* cid, const u64* n_dev, u64 n_bound,
                               ulonglong2* tab, u64 nb, u32 bits_y, u64* counters, int* ids,
                               int n_sm, cudaStream_t st);
cudaError_t launch_label_cells(const double* xy, u64 n, Grid g, const ulonglong2* tab, u64 nb,
                               const int* ids, int* labels, int n_sm, cudaStream_t st);

cudaError_t launch_label_points(const double* xy, u64 n, Grid g, Table t, const int* tile_cid,
                                bool table_cids, int* labels, bool narrow, int n_sm,
                                cudaStream_t st);

// small utility kernels (api.cu)
cudaError_t launch_iota(u32* out, u64 n, int n_sm, cudaStream_t st);
cudaError_t launch_gather_sorted(const u32* order, const u64* key, const u64* cnt,
                                 const int* cid, u64 n, Grid res, long long* tx, long long* ty,
                                 u64* cnt_out, long long* cid_out, int n_sm, cudaStream_t st);

}  // namespace rg
