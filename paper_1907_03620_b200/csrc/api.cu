// api.cu — the C-ABI (include/raster_gpu.h): context lifetime, the
// accumulator state machine of TileAccumulator (accumulator.hpp:109-214), the
// composed pipeline of cluster_sequential (pipeline.hpp:92-126), host<->device
// staging, and small utility kernels. No CPU fallback anywhere: every
// computational entry point runs on the device or fails.
#include <algorithm>
#include <cstddef>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/raster_gpu.h"
#include "common.cuh"
#include "internal.h"

using namespace rg;

namespace {

thread_local std::string g_create_error;
const bool g_debug = std::getenv("RG_DEBUG") != nullptr;

constexpr double kMaxLoad = 0.7;  // TileCounts grows at 70% load (accumulator.hpp:34)
constexpr u64 kStagePoints = 1ull << 24;  // 256 MB per staging buffer

u64 next_pow2(u64 v) {
    u64 p = 1;
    while (p < v) p <<= 1;
    return p;
}

u32 bits_for(double count) {  // smallest b with 2^b >= count, at least 1
    u32 b = 1;
    while (b < 64 && std::ldexp(1.0, (int)b) < count) ++b;
    return b;
}

u32 log2u(u64 v) {
    u32 b = 0;
    while ((1ull << b) < v) ++b;
    return b;
}

// Count-table capacity for a slot target: the next power of two. (Tables
// sized exactly to the load target, with a multiply-high bucket map, were
// measured: config 4 at 55 % load instead of 37 % made K1's claims probe
// further, K1 1.59 -> 1.75 ms, more than K2 and the clear gained.)
u64 table_cap(u64 want) { return next_pow2(std::max<u64>(want, 1024)); }

// Forward half of neighbor_offsets (agglomerate.hpp:38-50): the delta-ball of
// the metric minus the centre, restricted to dx > 0 or (dx == 0 and dy > 0).
std::vector<int2> forward_offsets(const rg_params& p) {
    std::vector<int2> out;
    const int d = p.distance;
    for (int dx = -d; dx <= d; ++dx)
        for (int dy = -d; dy <= d; ++dy) {
            if (dx == 0 && dy == 0) continue;
            if (p.metric == RG_METRIC_MANHATTAN && std::abs(dx) + std::abs(dy) > d) continue;
            if (dx > 0 || (dx == 0 && dy > 0)) out.push_back(make_int2(dx, dy));
        }
    return out;
}

struct DevGuard {
    int prev = -1;
    bool changed = false;
    explicit DevGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) {
            changed = cudaSetDevice(d) == cudaSuccess;
        }
    }
    ~DevGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

// Accumulator counters from the host (no host round trip: the values travel
// as kernel arguments); K1's scheduling fields start from zero.
__global__ void k_set_counters(Counters* c, u64 used, u64 ingested, u64 skipped) {
    c->used = used;
    c->ingested = ingested;
    c->skipped = skipped;
    c->ticket = 0;
    c->n_partial = 0;
    c->partial_ticket = 0;
    c->stopped = 0;
}

// K1's scheduling fields before a launch (a resumed round keeps the ticket).
__global__ void k_reset_k1(Counters* c, bool fresh) {
    if (fresh) c->ticket = 0;
    c->n_partial = 0;
    c->partial_ticket = 0;
    c->stopped = 0;
}

// Fingerprint of a point buffer: a hash of 64 sampled points' bits. The
// order probe's verdict is remembered per (buffer, length, fingerprint).
__global__ void k_fingerprint(const double* xy, u64 n, u64* out) {
    const int lane = threadIdx.x;
    u64 h = 0;
    for (int k = lane; k < 64; k += 32) {
        const u64 i = n > 64 ? (u64)k * (n / 64) + (u64)k % (n / 64) : (u64)k % n;
        u64 a = (u64)__double_as_longlong(xy[2 * i]) * 0x9E3779B97F4A7C15ull;
        a ^= (u64)__double_as_longlong(xy[2 * i + 1]) + 0xBF58476D1CE4E5B9ull * (u64)(k + 1);
        a ^= a >> 31;
        a *= 0x94D049BB133111EBull;
        h ^= a ^ (a >> 29);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(kFull, h, o);
    if (lane == 0) *out = h;
}

// Packed keys handed in by a caller (rg_ingest_counts): every key must be a
// key of this context's packing (not the EMPTY word, no bits above the
// column and row fields). Counts the offenders.
__global__ void k_check_keys(const u64* keys, u64 n, u32 key_bits, u64* bad) {
    u32 b = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 k = keys[i];
        b += (k == kEmpty || (key_bits < 64 && (k >> key_bits) != 0)) ? 1u : 0u;
    }
    b = __reduce_add_sync(kFull, b);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, (u64)b);
}

__global__ void k_iota(u32* out, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        out[i] = (u32)i;
}

__global__ void k_gather_sorted(const u32* order, const u64* key, const u64* cnt, const int* cid,
                                u64 n, Grid res, long long* tx, long long* ty, u64* cnt_out,
                                long long* cid_out) {
    const u64 ymask = (1ull << res.bits_y) - 1;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u32 j = order[i];
        const u64 k = key[j];
        if (tx) tx[i] = res.origin_x + (long long)(k >> res.bits_y);
        if (ty) ty[i] = res.origin_y + (long long)(k & ymask);
        if (cnt_out) cnt_out[i] = cnt[j];
        if (cid_out) cid_out[i] = cid ? (long long)cid[j] : -1ll;
    }
}

// Cluster id per K2 index from the sorted ids (deferred by the sorted K3).
__global__ void k_scatter_cid(const u32* perm, const int* cid_s, u64 n, int* tile_cid) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        tile_cid[perm[i]] = cid_s[i];
}

// Canonical output of the sorted path: keys and ids are already in sorted
// order; only the counts are gathered through the permutation.
__global__ void k_gather_sorted_keys(const u64* skey, const u32* perm, const u64* cnt,
                                     const int* cid_s, u64 n, Grid res, long long* tx,
                                     long long* ty, u64* cnt_out, long long* cid_out) {
    const u64 ymask = (1ull << res.bits_y) - 1;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 k = skey[i];
        if (tx) tx[i] = res.origin_x + (long long)(k >> res.bits_y);
        if (ty) ty[i] = res.origin_y + (long long)(k & ymask);
        if (cnt_out) cnt_out[i] = cnt[perm[i]];
        if (cid_out) cid_out[i] = (long long)cid_s[i];
    }
}

__global__ void k_cluster_facts(const u64* root_key_sorted, const u32* root_idx_sorted,
                                const u32* clu_root, u64 n, const u32* size, const u64* npts,
                                Grid res, u64* n_tiles, u64* n_points, long long* fx,
                                long long* fy) {
    const u64 ymask = (1ull << res.bits_y) - 1;
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < n;
         k += (u64)gridDim.x * blockDim.x) {
        // hash path: k-th kept root and its smallest key; sorted path: the
        // root's sorted position, whose key is the smallest of its cluster
        const u32 r = clu_root ? clu_root[k] : root_idx_sorted[k];
        const u64 key = root_key_sorted[clu_root ? r : k];
        if (n_tiles) n_tiles[k] = size[r];
        if (n_points) n_points[k] = npts[r];
        if (fx) fx[k] = res.origin_x + (long long)(key >> res.bits_y);
        if (fy) fy[k] = res.origin_y + (long long)(key & ymask);
    }
}

__global__ void k_count_of(Table t, u64 key, u64* out) {
    const u64 v = table_find(t, key);
    *out = (v == kEmpty) ? 0 : v;
}

// Multi-rank routing (rg_route_pairs): part of a pair from its column bin.
__device__ __forceinline__ u32 route_part(u64 key, u32 bits_y, long long col_min, u64 width,
                                          const u32* splits, u32 n_splits) {
    const u64 bin = (((key >> bits_y) - (u64)col_min) * 4096ull) / width;
    u32 lo = 0, hi = n_splits;  // number of splits <= bin
    while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (splits[mid] <= bin) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_route_count(const u64* keys, u64 n, u32 bits_y, long long col_min, u64 width,
                              const u32* splits, u32 n_parts, u64* part_counts) {
    __shared__ u32 cnt[1024];
    for (u32 i = threadIdx.x; i < n_parts; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x)
        atomicAdd(&cnt[route_part(keys[i], bits_y, col_min, width, splits, n_parts - 1)], 1u);
    __syncthreads();
    for (u32 i = threadIdx.x; i < n_parts; i += blockDim.x)
        if (cnt[i]) atomicAdd(part_counts + i, (u64)cnt[i]);
}

__global__ void k_route_offsets(const u64* part_counts, u32 n_parts, u64* cursor) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        u64 s = 0;
        for (u32 i = 0; i < n_parts; ++i) {
            cursor[i] = s;
            s += part_counts[i];
        }
    }
}

__global__ void k_route_scatter(const u64* keys, const u64* counts, u64 n, u32 bits_y,
                                long long col_min, u64 width, const u32* splits, u32 n_parts,
                                u64* cursor, u64* out_keys, u64* out_counts) {
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const bool v = i < n;
        const u64 k = v ? keys[i] : 0;
        const u32 p = v ? route_part(k, bits_y, col_min, width, splits, n_parts - 1) : 0xffffffffu;
        const u32 peers = __match_any_sync(kFull, p);
        const int leader = __ffs(peers) - 1;
        u64 base = 0;
        if (v && lane == leader) base = atomicAdd(cursor + p, (u64)__popc(peers));
        base = __shfl_sync(kFull, base, leader);
        if (v) {
            const u64 at = base + __popc(peers & ((1u << lane) - 1));
            out_keys[at] = k;
            out_counts[at] = counts[i];
        }
    }
}

int grid_for(u64 n, int n_sm, int per_sm = 8) {
    const u64 want = (n + 255) / 256;
    const u64 cap = (u64)n_sm * per_sm;
    return (int)(want == 0 ? 1 : (want < cap ? want : cap));
}

}  // namespace

namespace rg {
cudaError_t launch_iota(u32* out, u64 n, int n_sm, cudaStream_t st) {
    k_iota<<<grid_for(n, n_sm), 256, 0, st>>>(out, n);
    return cudaGetLastError();
}
cudaError_t launch_gather_sorted(const u32* order, const u64* key, const u64* cnt,
                                 const int* cid, u64 n, Grid res, long long* tx, long long* ty,
                                 u64* cnt_out, long long* cid_out, int n_sm, cudaStream_t st) {
    k_gather_sorted<<<grid_for(n, n_sm), 256, 0, st>>>(order, key, cnt, cid, n, res, tx, ty,
                                                        cnt_out, cid_out);
    return cudaGetLastError();
}
}  // namespace rg

struct rg_ctx {
    rg_params p{};
    Grid grid{};  // canvas packing (ingest)
    Grid res{};   // packing of the current significant set
    bool res_is_canvas = true;
    bool narrow = false;  // canvas column/row indices fit int32 (K1 32-bit path)
    int device = 0;
    int n_sm = 148;
    int max_warps = 0;
    cudaStream_t own = nullptr, st = nullptr, copy_st = nullptr;
    // Double-buffered table: the idle table is cleared on aux_st while the
    // current step's K3 runs, so the next ingest starts on a clean table.
    cudaStream_t aux_st = nullptr;
    cudaEvent_t ev_alt = nullptr;  // recorded on aux_st after the idle table's clear
    Slot* slots_alt = nullptr;
    u64 cap_alt = 0;
    bool alt_dirty = false;  // the idle table holds a previous step's entries
    bool alt_ready = false;  // the idle table's clear is enqueued (ev_alt)
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaEvent_t ev_k2 = nullptr, ev_k3 = nullptr, ev_end = nullptr;  // fused prune + agglomerate
    cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;  // K1 interval (resolved at the next host wait)
    bool contract_pending = false;
    // K1 rounds of the current ingest: launched, counters not yet read back
    // when `active` (rg_cluster defers the stop check to K3's one host read)
    struct K1Run {
        const double* xy = nullptr;
        u64 n = 0, rps = 0, W = 0, n_partial_in = 0;
        int pin = 0, round = 0;
        bool active = false;
    } k1;
    cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};

    Slot* slots = nullptr;
    u64 cap = 0;
    Counters* ctr = nullptr;
    Counters* hctr = nullptr;  // pinned mirror
    Partial* part[2] = {nullptr, nullptr};
    u64* scratch = nullptr;  // device scratch words
    // RASTER' cluster points (rg_cluster_points): 2*cp_n doubles, cp_c+1 offsets
    double* cp_xy = nullptr;
    u64* cp_off = nullptr;
    u64 cp_n = 0, cp_c = 0;
    bool cp_valid = false;
    // dedupe_points (retain mode): point set + unique counts per tile
    PtKey* ps = nullptr;
    u64 ps_cap = 0, ps_used = 0;
    Slot* ut = nullptr;
    u64 ut_cap = 0;
    u8* wf_keep = nullptr;   // window_fix flags, one per table slot
    u64 wf_cap = 0;

    u64 used = 0, ingested = 0, skipped = 0, grows = 0;
    enum State { kAccum, kSig, kAgg } state = kAccum;
    bool table_dirty = false;  // holds pruned marks: clear before the next ingest

    // significant set + agglomeration scratch, capacity sig_cap
    u64 n_sig = 0, sig_cap = 0;
    u64 *sig_key = nullptr, *sig_cnt = nullptr, *npts = nullptr, *min_key = nullptr;
    u32 *parent = nullptr, *size = nullptr;
    int *tile_cid = nullptr, *root_cid = nullptr;
    u64 *root_key = nullptr, *root_key_sorted = nullptr;
    u32 *root_idx = nullptr, *root_idx_sorted = nullptr;
    uint2* edges = nullptr;  // K3 deferred edges: 128 slots per 32-tile window
    u32* edge_n = nullptr;   // edges per window
    // key-sorted K3 (agglomerate_sorted.cu)
    bool sorted = false;     // current result came from the sorted path
    u32 *s_flag = nullptr, *s_scan = nullptr, *s_clu_root = nullptr;
    int* s_cid = nullptr;
    uint2* s_edges = nullptr;
    u64 s_cap = 0, s_edge_cap = 0;
    u32 *s_col_cnt = nullptr, *s_col_off = nullptr;
    u64 s_cols = 0;
    bool col_hist_ready = false;  // s_col_cnt holds the histogram of the current sig set (K2)
    bool npts_pending = false;    // sorted K3 left per-cluster point totals to rg_get_clusters
    u32* slot_of = nullptr;       // sorted path: table slot of significant tile pos (K2)
    bool sig_deferred = false;    // K2 left the table's SIG marks to mark_table()
    bool table_cids = false;      // table count words hold SIG | (cluster id + 1)
    bool tile_cid_pending = false;  // sorted K3 left tile_cid (K2 order) to ensure_tile_cid()
    // contraction of unordered inputs (partition.cu)
    void* part_scratch = nullptr;
    size_t part_scratch_bytes = 0;
    u64* pair_key = nullptr;
    u32* pair_cnt = nullptr;
    u64 pair_cap = 0;
    int part_stream_hint = 0;  // 1: the one-pass scatter fell back for the probed buffer
    // K2 from the partitioned contraction's pairs (rg_cluster of one device
    // span into an empty table): the pairs are final counts, so prune filters
    // them while their insertion into the table (KP3) runs on aux_st.
    bool allow_pairs_k2 = false;   // set by rg_cluster_ex around its ingest
    bool pairs_k2 = false;         // the pair slabs below describe the whole accumulator
    const uint4* pk_units = nullptr;
    const u32* pk_dcnt = nullptr;
    u32 pk_n_units = 0;
    bool insert_pending = false;   // KP3 in flight on aux_st (ev_kp3)
    cudaEvent_t ev_kp3 = nullptr;
    bool slot_of_valid = true;     // K2 recorded the table slots of the significant tiles
    bool k3_speculated = false;    // the last sorted K3 ran without its sizing read (verify max_col)
    bool k3_no_spec = false;       // redo after a failed verification: with the sizing read
    u64 order_probe[3] = {0, 0, 0};
    u64 probe_fp = 0;       // fingerprint of the probed buffer's content
    u64* k2_lb = nullptr;   // K2's look-back status words
    u64 k2_lb_words = 0;
    // K4' cell table of the kept tiles (labels of unordered inputs)
    ulonglong2* lk_tab = nullptr;
    int* lk_ids = nullptr;
    u64 lk_cap = 0, lk_nb = 0, lk_ids_cap = 0;
    bool lk_valid = false;
    bool fp_check = false;  // a fingerprint of the reused buffer is in ctr->pad2[0]
    int chunk_verdict = -1;  // host-span ingest: the first chunk's verdict for the rest
    const double* probe_ptr = nullptr;  // last probed buffer and its verdict
    u64 probe_n = 0;
    bool probe_unordered = false;
    float probe_new_ratio = 0.f;  // share of the probed points that opened a new tile
    void* sort_temp = nullptr;
    size_t sort_temp_bytes = 0;
    u64 n_roots = 0, n_kept = 0;

    int2* offsets = nullptr;
    int n_offsets = 0;

    double* stage[2] = {nullptr, nullptr};
    int* lstage[2] = {nullptr, nullptr};
    u64 stage_pts = 0;
    // streaming ingest (rg_stream_*): pinned host buffers the source fills
    double* pin[2] = {nullptr, nullptr};
    cudaEvent_t pin_free[2] = {nullptr, nullptr};  // its H2D copy has finished
    u64 pin_pts = 0;
    int pin_next = 0, pin_held = -1;
    u64 stream_chunks = 0;
    bool streaming = false;

    double ms_contract = 0, ms_prune = 0, ms_agg = 0, ms_label = 0;
    u64 launches = 0;
    std::string err;
};

namespace {

rg_status set_err(rg_ctx* c, rg_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c)
        c->err = buf;
    else
        g_create_error = buf;
    return s;
}

rg_status cuda_err(rg_ctx* c, cudaError_t e, const char* what) {
    return set_err(c, e == cudaErrorMemoryAllocation ? RG_ERR_OOM : RG_ERR_CUDA,
                   "CUDA error in %s: %s", what, cudaGetErrorString(e));
}

#define CK(call)                                                         \
    do {                                                                 \
        cudaError_t e_ = (call);                                         \
        if (e_ != cudaSuccess) return cuda_err(ctx, e_, #call);          \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, u64 count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMalloc((void**)p, count * sizeof(T));
}

// Stream-ordered temporaries (pooled by the device's default memory pool,
// whose release threshold rg_create raises, so per-call scratch does not pay
// cudaMalloc/cudaFree).
template <typename T>
cudaError_t salloc(T** p, u64 count, cudaStream_t st) {
    *p = nullptr;
    return cudaMallocAsync((void**)p, (size_t)std::max<u64>(count, 1) * sizeof(T), st);
}
template <typename T>
void sfree(T*& p, cudaStream_t st) {
    if (p) cudaFreeAsync((void*)p, st);
    p = nullptr;
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

rg_status validate(const rg_params* p, std::string& msg) {
    // GridParams::validate core.hpp:98-115, same checks, same order, same text.
    const double s = std::pow(10.0, p->precision);
    if (!std::isfinite(s) || s <= 0.0) {
        msg = "precision yields a non-finite or zero scale factor";
        return RG_ERR_CONFIG;
    }
    if (!std::isfinite(p->x_min) || !std::isfinite(p->x_max) || !std::isfinite(p->y_min) ||
        !std::isfinite(p->y_max)) {
        msg = "canvas bounds must be finite";
        return RG_ERR_CONFIG;
    }
    if (p->x_min >= p->x_max || p->y_min >= p->y_max) {
        msg = "canvas bounds must satisfy x_min < x_max and y_min < y_max";
        return RG_ERR_CONFIG;
    }
    const double limit = 4.6e18;
    if (std::abs(p->x_min) * s > limit || std::abs(p->x_max) * s > limit ||
        std::abs(p->y_min) * s > limit || std::abs(p->y_max) * s > limit) {
        msg = "precision too high for the canvas extent (tile index overflow)";
        return RG_ERR_CONFIG;
    }
    if (p->threshold < 1) {
        msg = "threshold must be >= 1";
        return RG_ERR_CONFIG;
    }
    if (p->distance < 1) {
        msg = "distance must be >= 1";
        return RG_ERR_CONFIG;
    }
    if (p->min_cluster_size < 1) {
        msg = "min cluster size must be >= 1";
        return RG_ERR_CONFIG;
    }
    if (p->metric != RG_METRIC_CHEBYSHEV && p->metric != RG_METRIC_MANHATTAN) {
        msg = "unknown metric";
        return RG_ERR_CONFIG;
    }
    if (p->mode != RG_MODE_COUNT_ONLY && p->mode != RG_MODE_RETAIN_POINTS) {
        msg = "unknown mode";
        return RG_ERR_CONFIG;
    }
    if (p->oob_policy != RG_OOB_SKIP && p->oob_policy != RG_OOB_STRICT) {
        msg = "unknown out-of-bounds policy";
        return RG_ERR_CONFIG;
    }
    // GPU-path limits.
    if (p->distance > 64) {
        msg = "distance > 64 is not supported on the GPU path";
        return RG_ERR_UNSUPPORTED;
    }
    const double cols = std::floor(p->x_max * s) - std::floor(p->x_min * s) + 1.0;
    const double rows = std::floor(p->y_max * s) - std::floor(p->y_min * s) + 1.0;
    if (bits_for(cols) + std::max<u32>(kBlockBits, bits_for(rows)) > 63) {
        msg = "canvas has too many tiles for a 63-bit packed tile key on the GPU path";
        return RG_ERR_UNSUPPORTED;
    }
    return RG_OK;
}

Grid make_grid(const rg_params& p) {
    Grid g{};
    g.scale = std::pow(10.0, p.precision);  // GridParams::scale core.hpp:95
    g.x_min = p.x_min;
    g.x_max = p.x_max;
    g.y_min = p.y_min;
    g.y_max = p.y_max;
    g.origin_x = (long long)std::floor(p.x_min * g.scale);  // min_column core.hpp:117-119
    g.origin_y = (long long)std::floor(p.y_min * g.scale);
    g.ox32 = (int)g.origin_x;
    g.oy32 = (int)g.origin_y;
    const double cols = std::floor(p.x_max * g.scale) - std::floor(p.x_min * g.scale) + 1.0;
    const double rows = std::floor(p.y_max * g.scale) - std::floor(p.y_min * g.scale) + 1.0;
    g.bits_x = bits_for(cols);
    g.bits_y = std::max<u32>(kBlockBits, bits_for(rows));  // table blocks need >= 2 row bits
    return g;
}

Table make_table(Slot* slots, u64 cap, u32 bits_y) {
    Table t;
    t.slots = slots;
    t.bmask = cap / kBucketSlots - 1;
    t.shift = 64 - log2u(cap / kBucketSlots);
    t.bits_y = bits_y;
    return t;
}

Table table_of(const rg_ctx* c) { return make_table(c->slots, c->cap, c->res.bits_y); }

rg_status alloc_table(rg_ctx* ctx, u64 cap, Slot** out) {
    CK(dalloc(out, cap));
    cudaError_t e = launch_table_clear(*out, cap, ctx->n_sm, ctx->st);
    ++ctx->launches;
    if (e != cudaSuccess) {
        dfree(*out);
        return cuda_err(ctx, e, "table clear");
    }
    return RG_OK;
}

// TileCounts::grow accumulator.hpp:84-94: allocate a larger table and fold the
// old one into it.
rg_status grow_table(rg_ctx* ctx, u64 new_cap) {
    Slot* ns = nullptr;
    rg_status s = alloc_table(ctx, new_cap, &ns);
    if (s != RG_OK) return s;
    if (ctx->slots) {
        const Table nt = make_table(ns, new_cap, ctx->res.bits_y);
        CK(launch_table_fold(ctx->slots, ctx->cap, nt, ctx->scratch, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaStreamSynchronize(ctx->st));
        dfree(ctx->slots);
        ++ctx->grows;
    }
    ctx->slots = ns;
    ctx->cap = new_cap;
    return RG_OK;
}

void zero_field(rg_ctx* ctx, u64* f) { cudaMemsetAsync(f, 0, sizeof(u64), ctx->st); }

// After a host read of the whole Counters block: a reused buffer whose
// content fingerprint changed loses its order verdict.
void check_fingerprint(rg_ctx* ctx) {
    if (!ctx->fp_check) return;
    ctx->fp_check = false;
    if (ctx->hctr->pad2[0] != ctx->probe_fp) ctx->probe_ptr = nullptr;
}

rg_status pull_counters(rg_ctx* ctx) {
    CK(cudaMemcpyAsync(ctx->hctr, ctx->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    check_fingerprint(ctx);
    ctx->used = ctx->hctr->used;
    ctx->ingested = ctx->hctr->ingested;
    ctx->skipped = ctx->hctr->skipped;
    return RG_OK;
}

// Asynchronous (stream-ordered): callers that hand the context's buffers to
// another stream synchronise themselves.
rg_status push_counters(rg_ctx* ctx) {
    k_set_counters<<<1, 1, 0, ctx->st>>>(ctx->ctr, ctx->used, ctx->ingested, ctx->skipped);
    ++ctx->launches;
    CK(cudaGetLastError());
    return RG_OK;
}

rg_status k1_finish(rg_ctx* ctx);

// Returns the accumulator to "fresh" after a prune consumed it
// (accumulator.hpp:171-173: counts_.clear()). ingested/skipped are kept, as in
// the reference.
rg_status reopen_accumulator(rg_ctx* ctx) {
    ctx->lk_valid = false;
    if (ctx->k1.active) {  // an ingest whose stop check never ran: finish it
        rg_status s = k1_finish(ctx);
        if (s != RG_OK) return s;
    }
    if (ctx->state == rg_ctx::kAccum && !ctx->table_dirty) return RG_OK;
    if (ctx->slots) {
        if (ctx->alt_ready && ctx->slots_alt && ctx->cap_alt == ctx->cap) {
            // the idle table was cleared behind the previous step's K3
            std::swap(ctx->slots, ctx->slots_alt);
            CK(cudaStreamWaitEvent(ctx->st, ctx->ev_alt, 0));
            ctx->alt_ready = false;
            ctx->alt_dirty = true;
        } else {
            CK(launch_table_clear(ctx->slots, ctx->cap, ctx->n_sm, ctx->st));
            ++ctx->launches;
            if (ctx->slots_alt && ctx->cap_alt != ctx->cap) {
                CK(cudaStreamSynchronize(ctx->aux_st));
                dfree(ctx->slots_alt);
                ctx->slots_alt = nullptr;
                ctx->cap_alt = 0;
                ctx->alt_ready = ctx->alt_dirty = false;
            }
            if (!ctx->slots_alt && ctx->cap * sizeof(Slot) <= (8ull << 30)) {
                // second table (best effort: without it every step clears inline)
                Slot* a = nullptr;
                if (cudaMalloc(&a, ctx->cap * sizeof(Slot)) == cudaSuccess) {
                    ctx->slots_alt = a;
                    ctx->cap_alt = ctx->cap;
                    ctx->alt_dirty = true;
                    ctx->alt_ready = false;
                } else {
                    cudaGetLastError();
                }
            }
        }
    }
    if (ctx->ps && ctx->ps_used) {
        CK(cudaMemsetAsync(ctx->ps, 0xff, ctx->ps_cap * sizeof(PtKey), ctx->st));
        CK(launch_table_clear(ctx->ut, ctx->ut_cap, ctx->n_sm, ctx->st));
        ctx->launches += 1;
    }
    ctx->ps_used = 0;
    ctx->used = 0;
    ctx->col_hist_ready = false;
    ctx->sig_deferred = false;
    ctx->table_cids = false;
    ctx->tile_cid_pending = false;
    ctx->table_dirty = false;
    ctx->state = rg_ctx::kAccum;
    ctx->n_sig = 0;
    ctx->n_roots = ctx->n_kept = 0;
    ctx->res = ctx->grid;
    ctx->res_is_canvas = true;
    return push_counters(ctx);
}

struct PhaseTimer {
    rg_ctx* c;
    double* acc;
    PhaseTimer(rg_ctx* c_, double* a) : c(c_), acc(a) { cudaEventRecord(c->t0, c->st); }
    void stop() {
        if (!acc) return;
        cudaEventRecord(c->t1, c->st);
        cudaEventSynchronize(c->t1);
        float ms = 0;
        cudaEventElapsedTime(&ms, c->t0, c->t1);
        *acc += ms;
        acc = nullptr;
    }
    ~PhaseTimer() { stop(); }
};

// Adds the pending K1 interval to ms_contract (cheap once the host has
// waited for the stream anyway).
void resolve_contract_timer(rg_ctx* ctx) {
    if (!ctx->contract_pending) return;
    float ms = 0;
    if (cudaEventSynchronize(ctx->ev_c1) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->ev_c0, ctx->ev_c1) == cudaSuccess)
        ctx->ms_contract += ms;
    ctx->contract_pending = false;
}

// K1 driver over a device-resident span (TileAccumulator::ingest
// accumulator.hpp:120-134). Handles budget stops, growth and resumption.
// Inputs without spatial order take the partitioned contraction
// (partition.cu). RG_INGEST=k1 / =part forces a path; otherwise a probe of
// 64 windows of 2,048 consecutive points decides: when more than 60 % of a
// window's points open a new tile, K1's per-warp cache cannot help.
bool buffer_unordered(rg_ctx* ctx, const double* xy, u64 n);

bool use_partition_ingest(rg_ctx* ctx, const double* xy, u64 n) {
    static const int forced = [] {
        const char* v = std::getenv("RG_INGEST");
        return v ? (std::strcmp(v, "k1") == 0 ? 1 : (std::strcmp(v, "part") == 0 ? 2 : 0)) : 0;
    }();
    const u32 bits = ctx->grid.bits_x + ctx->grid.bits_y;
    // the partitioned kernels read points as 16-byte double2
    if (forced == 1 || !partition_ingest_supported(bits, n) || ((uintptr_t)xy & 15)) return false;
    if (forced == 2) return true;
    if (n < (1ull << 22)) return false;
    if (ctx->chunk_verdict >= 0) return ctx->chunk_verdict != 0;
    return buffer_unordered(ctx, xy, n);
}

// The order probe (memoised per buffer, see below): true when consecutive
// points rarely share tiles.
bool buffer_unordered(rg_ctx* ctx, const double* xy, u64 n) {
    // The same buffer clustered again (a serving loop, the bench) reuses the
    // verdict without a host round trip. Its content is still fingerprinted
    // on the device; the fingerprint comes back with the counters at the
    // next host read, and a mismatch (the buffer was refilled) drops the
    // verdict so the next call probes again. (The path choice only affects
    // speed: both contractions give identical counts.)
    if (ctx->probe_ptr == xy && ctx->probe_n == n) {
        k_fingerprint<<<1, 32, 0, ctx->st>>>(xy, n, &ctx->ctr->pad2[0]);
        ++ctx->launches;
        ctx->fp_check = true;
        return ctx->probe_unordered;
    }
    if (launch_order_probe(xy, n, ctx->grid, ctx->scratch, ctx->n_sm, ctx->st) != cudaSuccess)
        return false;
    k_fingerprint<<<1, 32, 0, ctx->st>>>(xy, n, ctx->scratch + 2);
    ctx->launches += 2;
    if (cudaMemcpyAsync(ctx->order_probe, ctx->scratch, 3 * sizeof(u64), cudaMemcpyDeviceToHost,
                        ctx->st) != cudaSuccess ||
        cudaStreamSynchronize(ctx->st) != cudaSuccess)
        return false;
    const u64 distinct = ctx->order_probe[0], valid = ctx->order_probe[1] & 0xffffffffull,
              near = ctx->order_probe[1] >> 32;
    ctx->probe_ptr = xy;
    ctx->probe_n = n;
    ctx->probe_fp = ctx->order_probe[2];
    // Without spatial order: more than 60 % of the points open a new tile in
    // their window; or more than 35 % do and fewer than 40 % lie within 8
    // tiles of their successor. The second rule tells a shuffled input with a
    // hot spot (config 5 shuffled: 50 % new tiles, 25 % near: the partitions
    // take 10.5 ms against K1's 15.6 ms) from an ordered one with few points
    // per tile (config 5 as generated: 30 % new, ~75 % near: K1 3.1 ms).
    ctx->probe_unordered = valid > 0 && (distinct * 5 > valid * 3 ||
                                         (distinct * 20 > valid * 7 && near * 5 < valid * 2));
    ctx->probe_new_ratio = valid ? (float)((double)distinct / (double)valid) : 0.f;
    if (g_debug)
        std::fprintf(stderr,
                     "[rg] order probe n=%llu: %llu of %llu sampled points open a tile, %llu near "
                     "their successor -> %s\n",
                     (unsigned long long)n, (unsigned long long)distinct,
                     (unsigned long long)valid, (unsigned long long)near,
                     ctx->probe_unordered ? "partitioned" : "K1");
    return ctx->probe_unordered;
}

bool dedupe_active(const rg_ctx* ctx);

// The table is complete again once the main stream has waited for a KP3
// that was left running on aux_st.
rg_status settle_insert(rg_ctx* ctx) {
    if (ctx->insert_pending) {
        CK(cudaStreamWaitEvent(ctx->st, ctx->ev_kp3, 0));
        ctx->insert_pending = false;
    }
    return RG_OK;
}

rg_status ingest_partitioned(rg_ctx* ctx, const double* xy, u64 n) {
    size_t scan_temp = 0;
    const size_t need = partition_scratch_bytes(n, &scan_temp);
    if (ctx->part_scratch_bytes < need) {
        if (ctx->part_scratch) cudaFree(ctx->part_scratch);
        ctx->part_scratch = nullptr;
        ctx->part_scratch_bytes = 0;
        CK(cudaMalloc(&ctx->part_scratch, need));
        ctx->part_scratch_bytes = need;
    }
    // one pair slot per residual entry: per-unit slabs never overlap
    const u64 pair_need = partition_res_entries(n);
    if (ctx->pair_cap < pair_need) {
        dfree(ctx->pair_key);
        dfree(ctx->pair_cnt);
        ctx->pair_cap = 0;
        CK(dalloc(&ctx->pair_key, pair_need));
        CK(dalloc(&ctx->pair_cnt, pair_need));
        ctx->pair_cap = pair_need;
    }
    PartitionPlan plan;
    PhaseTimer timer(ctx, &ctx->ms_contract);
    const u64 used_before = ctx->used;
    ctx->pairs_k2 = false;
    PartitionLaunch L;
    L.xy = xy;
    L.n = n;
    L.g = ctx->grid;
    L.key_bits = ctx->grid.bits_x + ctx->grid.bits_y;
    L.ctr = ctx->ctr;
    L.scratch = ctx->part_scratch;
    L.scan_temp = scan_temp;
    L.pkey = ctx->pair_key;
    L.pcnt = ctx->pair_cnt;
    L.n_sm = ctx->n_sm;
    L.narrow = ctx->narrow;
    // the one-pass scatter's fallback is remembered with the order verdict
    if (!(ctx->probe_ptr == xy && ctx->probe_n == n)) ctx->part_stream_hint = 0;
    L.stream_hint = &ctx->part_stream_hint;
    CK(launch_partition_count(L, ctx->st, &plan));
    ctx->launches += plan.launches;
    const u64 pairs = plan.pair_off.back();
    // the table must hold every key KP3 can claim below the load target
    while ((double)(ctx->used + pairs + plan.raw_points) >= kMaxLoad * (double)ctx->cap) {
        rg_status s = grow_table(ctx, ctx->cap * 2);
        if (s != RG_OK) return s;
    }
    // rg_cluster of one device span into an empty table, every partition one
    // work unit: the pairs are the final counts. K2 then filters the pairs
    // (prune_enqueue) and KP3 fills the table on aux_st beside K2 and K3.
    static const bool pairs_off = [] {
        const char* v = std::getenv("RG_PAIRS_K2");
        return v && std::strcmp(v, "0") == 0;
    }();
    const bool defer = ctx->allow_pairs_k2 && !pairs_off && used_before == 0 && pairs > 0 &&
                       plan.raw_points == 0 && plan.single_units && !dedupe_active(ctx);
    if (defer) {
        CK(cudaEventRecord(ctx->ev_kp3, ctx->st));
        CK(cudaStreamWaitEvent(ctx->aux_st, ctx->ev_kp3, 0));
        static const int side_bps = [] {
            const char* v = std::getenv("RG_KP3_SIDE_BPS");
            const int b = v ? std::atoi(v) : 0;
            return b >= 1 && b <= 64 ? b : 16;
        }();
        CK(launch_partition_insert(L, table_of(ctx), plan, ctx->aux_st, side_bps));
        CK(cudaEventRecord(ctx->ev_kp3, ctx->aux_st));
        ctx->launches += 1;
        ctx->insert_pending = true;
        ctx->pairs_k2 = true;
        ctx->pk_units = plan.units_dev;
        ctx->pk_dcnt = plan.dcnt_dev;
        ctx->pk_n_units = (u32)plan.units.size();
        rg_status s = pull_counters(ctx);  // ingested / skipped (KP3 is still adding to `used`)
        ctx->used = pairs;                 // one claim per pair into the empty table
        return s;
    }
    CK(launch_partition_insert(L, table_of(ctx), plan, ctx->st));
    ctx->launches += 1 + (plan.raw_points ? 1 : 0);
    return pull_counters(ctx);
}

// One K1 round of ctx->k1 (growing the table first when the round's
// budget would not fit under the load target).
rg_status k1_launch_round(rg_ctx* ctx) {
    rg_ctx::K1Run& r = ctx->k1;
    u64 soft = (u64)(kMaxLoad * (double)ctx->cap);
    while (ctx->used + 64 * r.W >= soft) {
        rg_status s = grow_table(ctx, ctx->cap * 2);
        if (s != RG_OK) return s;
        soft = (u64)(kMaxLoad * (double)ctx->cap);
    }
    ContractLaunch L;
    L.xy = r.xy;
    L.n = r.n;
    L.rows_per_seg = r.rps;
    L.warps = r.W;
    L.g = ctx->grid;
    L.t = table_of(ctx);
    L.ctr = ctx->ctr;
    L.partial_in = ctx->part[r.pin];
    L.n_partial_in = r.n_partial_in;
    L.partial_out = ctx->part[1 - r.pin];
    L.budget = (soft - ctx->used) / r.W;
    L.narrow = ctx->narrow;
    // An input whose evictions mostly claim NEW keys (config 5: 60M noise and
    // chain tiles, ~30 % of the probed points open a tile) installs key and
    // count with one 128-bit CAS: K1 3.52 -> 3.17 ms; for config 4 (2 %) the
    // 64-bit claim + RED is faster (1.55 against 1.59 ms).
    static const int c128_mode = [] {  // RG_K1_CLAIM128=0 / =1 forces it (A/B)
        const char* v = std::getenv("RG_K1_CLAIM128");
        return v ? (std::strcmp(v, "0") == 0 ? 0 : 1) : -1;
    }();
    L.claim128 = c128_mode >= 0 ? c128_mode != 0
                                : (ctx->probe_ptr == r.xy && ctx->probe_n == r.n &&
                                   ctx->probe_new_ratio >= 0.2f);
    CK(launch_contract(L, ctx->st));
    ++ctx->launches;
    CK(cudaEventRecord(ctx->ev_c1, ctx->st));
    if (g_debug)
        std::fprintf(stderr, "[rg] K1 round %d: n=%llu W=%llu rps=%llu cap=%llu used=%llu budget=%llu\n",
                     r.round, (unsigned long long)r.n, (unsigned long long)r.W,
                     (unsigned long long)r.rps, (unsigned long long)ctx->cap,
                     (unsigned long long)ctx->used, (unsigned long long)L.budget);
    return RG_OK;
}

// Reads K1's counters back; while warps ran out of budget, resumes their
// partial segments (and the untouched tickets) after growing the table if
// it is filling up. Partial segments of the previous round that no warp
// reached before every warp stopped are carried over behind the new ones.
rg_status k1_finish(rg_ctx* ctx) {
    rg_ctx::K1Run& r = ctx->k1;
    while (true) {
        rg_status s = pull_counters(ctx);
        if (s != RG_OK) return s;
        if (g_debug)
            std::fprintf(stderr, "[rg] K1 round %d done: used=%llu stopped=%llu partial=%llu "
                         "ticket=%llu ingested=%llu\n", r.round, (unsigned long long)ctx->used,
                         (unsigned long long)ctx->hctr->stopped,
                         (unsigned long long)ctx->hctr->n_partial,
                         (unsigned long long)ctx->hctr->ticket, (unsigned long long)ctx->ingested);
        if (ctx->hctr->stopped == 0) break;
        const u64 taken = std::min<u64>(ctx->hctr->partial_ticket, r.n_partial_in);
        u64 n_next = ctx->hctr->n_partial;
        if (taken < r.n_partial_in) {
            CK(cudaMemcpyAsync(ctx->part[1 - r.pin] + n_next, ctx->part[r.pin] + taken,
                               (r.n_partial_in - taken) * sizeof(Partial),
                               cudaMemcpyDeviceToDevice, ctx->st));
            n_next += r.n_partial_in - taken;
        }
        r.n_partial_in = n_next;
        r.pin = 1 - r.pin;
        k_reset_k1<<<1, 1, 0, ctx->st>>>(ctx->ctr, false);  // the ticket keeps counting
        if (ctx->used >= (u64)(0.85 * kMaxLoad * (double)ctx->cap)) {
            s = grow_table(ctx, ctx->cap * 2);
            if (s != RG_OK) return s;
        }
        if (++r.round > 64) return set_err(ctx, RG_ERR_CUDA, "contraction failed to make progress");
        s = k1_launch_round(ctx);
        if (s != RG_OK) return s;
    }
    r.active = false;
    resolve_contract_timer(ctx);
    return RG_OK;
}

// Upper bound of the table's keys while a deferred K1 round is in flight:
// the round's budget keeps it under the load target plus one batch per warp.
u64 k1_used_bound(const rg_ctx* ctx) {
    const u64 soft = (u64)(kMaxLoad * (double)ctx->cap);
    return std::min<u64>(ctx->cap, soft + ctx->k1.W * (u64)contract_batch_rows() * 32);
}

rg_status ingest_device(rg_ctx* ctx, const double* xy, u64 n, bool defer = false) {
    if (n == 0) return RG_OK;
    const u64 rows = (n + 31) / 32;
    const u64 w0 = (u64)ctx->max_warps;
    const u64 batch = (u64)contract_batch_rows();
    u64 rps = rows / (8 * w0);
    rps = std::max<u64>(batch, std::min<u64>(256, rps)) / batch * batch;
    const u64 n_seg = (rows + rps - 1) / rps;
    const u64 bw = (u64)contract_block_warps();
    const u64 W = (std::min(w0, n_seg) + bw - 1) / bw * bw;  // whole blocks (w0 is a multiple)
    // A warp checks its budget once per batch of rows, so it can overshoot
    // by batch*32 - 1 keys: the table must hold soft + W*batch*32 keys, i.e.
    // (1 - kMaxLoad) * cap > W * batch * 32.
    const u64 cap_min = table_cap((u64)((double)(W * batch * 32) / (1.0 - kMaxLoad)) + 1024);

    if (!ctx->slots) {
        u64 want;
        if (ctx->p.capacity_hint) {
            want = (u64)((double)ctx->p.capacity_hint / kMaxLoad) + 1;
        } else {
            const double tb = rg_params_tile_bound(&ctx->p);
            double est = std::min((double)(n / 32), tb);
            want = (u64)(est / kMaxLoad) + 1;
        }
        want = std::max<u64>(std::max<u64>(want, cap_min), 1024);
        rg_status s = grow_table(ctx, table_cap(want));
        if (s != RG_OK) return s;
    } else if (ctx->cap < cap_min) {
        rg_status s = grow_table(ctx, cap_min);
        if (s != RG_OK) return s;
    }

    if (use_partition_ingest(ctx, xy, n)) return ingest_partitioned(ctx, xy, n);

    resolve_contract_timer(ctx);  // a previous chunk's interval
    CK(cudaEventRecord(ctx->ev_c0, ctx->st));
    ctx->contract_pending = true;
    k_reset_k1<<<1, 1, 0, ctx->st>>>(ctx->ctr, true);
    ctx->k1 = rg_ctx::K1Run{xy, n, rps, W, 0, 0, 0, true};
    rg_status s = k1_launch_round(ctx);
    if (s != RG_OK) return s;
    return defer ? RG_OK : k1_finish(ctx);
}

rg_status ensure_stage(rg_ctx* ctx, u64 pts, bool labels) {
    const u64 want = std::min<u64>(pts, kStagePoints);
    if (ctx->stage_pts < want) {
        for (int b = 0; b < 2; ++b) {
            dfree(ctx->stage[b]);
            dfree(ctx->lstage[b]);
        }
        ctx->stage_pts = 0;
        for (int b = 0; b < 2; ++b) CK(dalloc(&ctx->stage[b], 2 * want));
        ctx->stage_pts = want;
    }
    if (labels && !ctx->lstage[0]) {
        for (int b = 0; b < 2; ++b) CK(dalloc(&ctx->lstage[b], ctx->stage_pts));
    }
    return RG_OK;
}

// Strict policy: index of the first out-of-bounds point, or n.
rg_status first_oob(rg_ctx* ctx, const double* dxy, u64 n, u64* first) {
    CK(cudaMemsetAsync(&ctx->ctr->first_oob, 0xff, sizeof(u64), ctx->st));
    CK(launch_first_oob(dxy, n, ctx->grid, &ctx->ctr->first_oob, ctx->n_sm, ctx->st));
    ++ctx->launches;
    u64 f = 0;
    CK(cudaMemcpyAsync(&ctx->hctr->first_oob, &ctx->ctr->first_oob, sizeof(u64),
                       cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    f = ctx->hctr->first_oob;
    *first = f < n ? f : n;
    return RG_OK;
}

rg_status oob_error(rg_ctx* ctx, double x, double y) {
    // accumulator.hpp:123-125: "point (" + to_string(x) + ", " + to_string(y) + ") ..."
    // std::to_string(double) formats with "%f".
    return set_err(ctx, RG_ERR_OOB, "point (%f, %f) outside canvas bounds", x, y);
}

// ---- dedupe_points (retain mode): see dedupe.cu
bool dedupe_active(const rg_ctx* ctx) {
    return ctx->p.dedupe_points && ctx->p.mode == RG_MODE_RETAIN_POINTS;
}

PointSet point_set(const rg_ctx* c) { return PointSet{c->ps, c->ps_cap - 1}; }
Table ut_table(const rg_ctx* c) { return make_table(c->ut, c->ut_cap, c->res.bits_y); }

// The unique-count table follows the capacity of the count table (its keys
// are a subset of the count table's).
rg_status ensure_ut(rg_ctx* ctx) {
    if (ctx->ut && ctx->ut_cap >= ctx->cap) return RG_OK;
    Slot* nu = nullptr;
    const u64 nc = std::max<u64>(ctx->cap, 1024);
    rg_status s = alloc_table(ctx, nc, &nu);
    if (s != RG_OK) return s;
    if (ctx->ut) {
        CK(launch_table_fold(ctx->ut, ctx->ut_cap, make_table(nu, nc, ctx->res.bits_y),
                             ctx->scratch, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaStreamSynchronize(ctx->st));
        dfree(ctx->ut);
    }
    ctx->ut = nu;
    ctx->ut_cap = nc;
    return RG_OK;
}

// Point set at <= 50% load after `add` more distinct points.
rg_status ensure_ps(rg_ctx* ctx, u64 add) {
    const u64 need = ctx->ps_used + add;
    if (ctx->ps && 2 * need <= ctx->ps_cap) return RG_OK;
    const u64 nc = next_pow2(std::max<u64>(2 * need, 1024));
    PtKey* np = nullptr;
    CK(dalloc(&np, nc));
    CK(cudaMemsetAsync(np, 0xff, nc * sizeof(PtKey), ctx->st));
    if (ctx->ps) {
        CK(launch_ps_rehash(ctx->ps, ctx->ps_cap, PointSet{np, nc - 1}, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaStreamSynchronize(ctx->st));
        dfree(ctx->ps);
    }
    ctx->ps = np;
    ctx->ps_cap = nc;
    return RG_OK;
}

rg_status dedupe_ingest(rg_ctx* ctx, const double* dxy, u64 n) {
    if (n == 0) return RG_OK;
    rg_status s = ensure_ut(ctx);
    if (s != RG_OK) return s;
    s = ensure_ps(ctx, n);
    if (s != RG_OK) return s;
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(u64), ctx->st));
    CK(launch_dedupe_ingest(dxy, n, ctx->grid, point_set(ctx), ut_table(ctx), ctx->scratch,
                            ctx->n_sm, ctx->st));
    ++ctx->launches;
    CK(cudaMemcpyAsync(&ctx->hctr->pad0[0], ctx->scratch, sizeof(u64), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->ps_used += ctx->hctr->pad0[0];
    return RG_OK;
}

rg_status ingest_counted(rg_ctx* ctx, const double* dxy, u64 n, bool defer = false) {
    rg_status s = ingest_device(ctx, dxy, n, defer && !dedupe_active(ctx));
    if (s == RG_OK && dedupe_active(ctx)) s = dedupe_ingest(ctx, dxy, n);
    return s;
}

rg_status ingest_span(rg_ctx* ctx, const double* dxy, u64 n, bool* hit_oob, double* ox,
                      double* oy, bool defer = false) {
    *hit_oob = false;
    if (ctx->p.oob_policy == RG_OOB_STRICT) {
        u64 f = n;
        rg_status s = first_oob(ctx, dxy, n, &f);
        if (s != RG_OK) return s;
        if (f < n) {
            double pt[2];
            CK(cudaMemcpy(pt, dxy + 2 * f, sizeof pt, cudaMemcpyDeviceToHost));
            *hit_oob = true;
            *ox = pt[0];
            *oy = pt[1];
            return ingest_counted(ctx, dxy, f);
        }
    }
    return ingest_counted(ctx, dxy, n, defer);
}

// defer: a device span's K1 stop check may be left to the caller (k1_finish
// or the deferred check in prune_agglomerate_fused); strict policy never defers.
rg_status ingest_any(rg_ctx* ctx, const double* xy, u64 n, rg_memkind kind, bool defer = false) {
    rg_status s = reopen_accumulator(ctx);
    if (s != RG_OK) return s;
    if (n == 0) return RG_OK;
    bool oob = false;
    double ox = 0, oy = 0;
    if (kind == RG_MEM_DEVICE) {
        s = ingest_span(ctx, xy, n, &oob, &ox, &oy, defer && ctx->p.oob_policy != RG_OOB_STRICT);
        if (s != RG_OK) return s;
        return oob ? oob_error(ctx, ox, oy) : RG_OK;
    }
    // Host span: double-buffered H2D staging overlapped with K1.
    s = ensure_stage(ctx, n, false);
    if (s != RG_OK) return s;
    const u64 ch = ctx->stage_pts;
    const u64 chunks = (n + ch - 1) / ch;
    auto enqueue_copy = [&](u64 i) -> rg_status {
        const int b = (int)(i & 1);
        const u64 off = i * ch;
        const u64 len = std::min(ch, n - off);
        CK(cudaStreamWaitEvent(ctx->copy_st, ctx->done[b], 0));
        CK(cudaMemcpyAsync(ctx->stage[b], xy + 2 * off, len * 2 * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->copy_st));
        CK(cudaEventRecord(ctx->copied[b], ctx->copy_st));
        return RG_OK;
    };
    for (u64 i = 0; i < std::min<u64>(2, chunks); ++i) {
        s = enqueue_copy(i);
        if (s != RG_OK) return s;
    }
    // the order probe runs on the first chunk only; later chunks reuse its
    // verdict (the staging buffers alternate, so the per-buffer memo would
    // probe every chunk)
    struct VerdictScope {
        rg_ctx* c;
        ~VerdictScope() { c->chunk_verdict = -1; }
    } verdict_scope{ctx};
    ctx->chunk_verdict = -1;
    for (u64 i = 0; i < chunks; ++i) {
        const int b = (int)(i & 1);
        const u64 off = i * ch;
        const u64 len = std::min(ch, n - off);
        CK(cudaStreamWaitEvent(ctx->st, ctx->copied[b], 0));
        s = ingest_span(ctx, ctx->stage[b], len, &oob, &ox, &oy);
        if (s != RG_OK) return s;
        if (i == 0 && ctx->probe_ptr == ctx->stage[b]) ctx->chunk_verdict = ctx->probe_unordered;
        CK(cudaEventRecord(ctx->done[b], ctx->st));
        if (oob) {
            CK(cudaStreamSynchronize(ctx->copy_st));
            return oob_error(ctx, ox, oy);
        }
        if (i + 2 < chunks) {
            s = enqueue_copy(i + 2);
            if (s != RG_OK) return s;
        }
    }
    CK(cudaStreamSynchronize(ctx->copy_st));
    return RG_OK;
}

rg_status ensure_sig_capacity(rg_ctx* ctx, u64 n) {
    if (ctx->sig_cap >= n && ctx->sig_key) return RG_OK;
    dfree(ctx->sig_key);
    dfree(ctx->sig_cnt);
    dfree(ctx->npts);
    dfree(ctx->min_key);
    dfree(ctx->parent);
    dfree(ctx->size);
    dfree(ctx->tile_cid);
    dfree(ctx->slot_of);
    dfree(ctx->root_cid);
    dfree(ctx->root_key);
    dfree(ctx->root_key_sorted);
    dfree(ctx->root_idx);
    dfree(ctx->root_idx_sorted);
    dfree(ctx->edges);
    dfree(ctx->edge_n);
    ctx->sig_cap = 0;
    const u64 c = std::max<u64>(n, 1024);
    CK(dalloc(&ctx->sig_key, c));
    CK(dalloc(&ctx->sig_cnt, c));
    CK(dalloc(&ctx->npts, c));
    CK(dalloc(&ctx->min_key, c));
    CK(dalloc(&ctx->parent, c));
    CK(dalloc(&ctx->size, c));
    CK(dalloc(&ctx->tile_cid, c));
    CK(dalloc(&ctx->slot_of, c));
    CK(dalloc(&ctx->root_cid, c));
    CK(dalloc(&ctx->root_key, c));
    CK(dalloc(&ctx->root_key_sorted, c));
    CK(dalloc(&ctx->root_idx, c));
    CK(dalloc(&ctx->root_idx_sorted, c));
    CK(dalloc(&ctx->edges, (c + 31) / 32 * 128));
    CK(dalloc(&ctx->edge_n, (c + 31) / 32));
    ctx->sig_cap = c;
    return RG_OK;
}

rg_status ensure_sort_temp(rg_ctx* ctx, u64 n, int bits) {
    const size_t need = sort_pairs_temp_bytes(std::max<u64>(n, 1), bits);
    if (ctx->sort_temp_bytes >= need && ctx->sort_temp) return RG_OK;
    dfree(ctx->sort_temp);
    ctx->sort_temp_bytes = 0;
    CK(cudaMalloc(&ctx->sort_temp, need));
    ctx->sort_temp_bytes = need;
    return RG_OK;
}

bool use_sorted_k3(const rg_ctx* ctx) {
    static const char* force = std::getenv("RG_K3");  // "hash" forces the hash-probe path
    if (force && std::strcmp(force, "hash") == 0) return false;
    return ctx->p.distance <= 2 && ctx->used < 0x7fffffffull;  // S <= D = used
}

rg_status ensure_col_arrays(rg_ctx* ctx, u64 cols) {
    if (ctx->s_cols >= cols) return RG_OK;
    dfree(ctx->s_col_cnt);
    dfree(ctx->s_col_off);
    ctx->s_cols = 0;
    CK(dalloc(&ctx->s_col_cnt, cols + 1));
    CK(dalloc(&ctx->s_col_off, cols + 1));
    ctx->s_cols = cols;
    return RG_OK;
}

// The table's SIG marks after a sorted-path K2 (which records slot_of
// instead of rewriting the table): SIG | (cluster id + 1) once clusters
// exist (K4 then resolves a tile with one table load), else SIG | dense
// index (the hash-probe K3's form).
// Cluster id per K2 index (tile_cid), scattered from the sorted ids when the
// device view, the labelling pass or the SIG marks need it.
rg_status ensure_tile_cid(rg_ctx* ctx) {
    if (!ctx->tile_cid_pending) return RG_OK;
    if (ctx->n_sig) {
        k_scatter_cid<<<grid_for(ctx->n_sig, ctx->n_sm), 256, 0, ctx->st>>>(
            ctx->root_idx_sorted, ctx->s_cid, ctx->n_sig, ctx->tile_cid);
        ++ctx->launches;
        CK(cudaGetLastError());
    }
    ctx->tile_cid_pending = false;
    return RG_OK;
}

rg_status mark_table(rg_ctx* ctx, bool with_cids) {
    if (!ctx->sig_deferred) return RG_OK;
    if (with_cids) {
        rg_status s = ensure_tile_cid(ctx);
        if (s != RG_OK) return s;
    }
    if (!ctx->slot_of_valid) {  // K2 ran on the pairs: look the slots up
        rg_status si = settle_insert(ctx);
        if (si != RG_OK) return si;
        CK(launch_find_slots(table_of(ctx), ctx->sig_key, ctx->n_sig, ctx->slot_of, ctx->n_sm,
                             ctx->st));
        ++ctx->launches;
        ctx->slot_of_valid = true;
    }
    CK(launch_mark_sig(table_of(ctx), ctx->slot_of, with_cids ? ctx->tile_cid : nullptr,
                       ctx->n_sig, ctx->n_sm, ctx->st));
    ++ctx->launches;
    ctx->sig_deferred = false;
    ctx->table_cids = with_cids;
    return RG_OK;
}

// K2 (+ window_fix / dedupe pre-passes) enqueued on the stream; the
// significant count stays on the device (ctr->n_sig).
rg_status prune_enqueue(rg_ctx* ctx, bool window_fix) {
    ctx->lk_valid = false;
    if (ctx->state != rg_ctx::kAccum) {
        // prune() on a consumed accumulator returns nothing (empty table).
        rg_status s = reopen_accumulator(ctx);
        if (s != RG_OK) return s;
    }
    // a deferred K1 round has not reported its key count yet: size for its bound
    const u64 used = ctx->k1.active ? k1_used_bound(ctx) : ctx->used;
    rg_status s = ensure_sig_capacity(ctx, used);
    if (s != RG_OK) return s;
    zero_field(ctx, &ctx->ctr->n_sig);
    ctx->tile_cid_pending = false;
    // the pairs of a partitioned contraction stand in for the table scan
    // (consumed here: any later change of the table invalidates them)
    const bool from_pairs = ctx->pairs_k2 && ctx->slots && used && use_sorted_k3(ctx) &&
                            !window_fix && !(dedupe_active(ctx) && ctx->ut);
    ctx->pairs_k2 = false;
    if (!from_pairs) {  // everything below reads the table: a KP3 in flight must land first
        rg_status si = settle_insert(ctx);
        if (si != RG_OK) return si;
    }
    if (ctx->slots && used) {
        const bool hash_k3 = !use_sorted_k3(ctx);
        if (window_fix) {
            if (ctx->wf_cap < ctx->cap) {
                dfree(ctx->wf_keep);
                ctx->wf_cap = 0;
                CK(dalloc(&ctx->wf_keep, ctx->cap));
                ctx->wf_cap = ctx->cap;
            }
            CK(launch_window_mark(table_of(ctx), ctx->cap, ctx->p.threshold, ctx->grid.bits_x,
                                  ctx->wf_keep, ctx->n_sm, ctx->st));
            ++ctx->launches;
        }
        if (dedupe_active(ctx) && ctx->ut) {
            // threshold and reported counts follow the deduplicated counts
            // (accumulator.hpp:165-169; window_fix decided on raw counts)
            CK(launch_dedupe_counts(table_of(ctx), ctx->cap, ut_table(ctx), ctx->n_sm, ctx->st));
            ++ctx->launches;
        }
        // the sorted K3's column histogram is built by K2 itself
        const u64 cols = hash_k3 ? 0 : sorted_columns(ctx->grid.bits_x);
        if (cols) {
            s = ensure_col_arrays(ctx, cols);
            if (s != RG_OK) return s;
            CK(cudaMemsetAsync(ctx->s_col_cnt, 0, (cols + 1) * sizeof(u32), ctx->st));
        }
        if (ctx->k2_lb_words < compact_lb_words(ctx->cap)) {
            dfree(ctx->k2_lb);
            ctx->k2_lb_words = 0;
            CK(dalloc(&ctx->k2_lb, compact_lb_words(ctx->cap)));
            ctx->k2_lb_words = compact_lb_words(ctx->cap);
        }
        if (from_pairs) {
            CK(launch_compact_pairs(ctx->pk_units, ctx->pk_dcnt, ctx->pk_n_units, ctx->pair_key,
                                    ctx->pair_cnt, ctx->p.threshold, ctx->sig_key, ctx->sig_cnt,
                                    cols ? ctx->s_col_cnt : nullptr, ctx->grid.bits_y, ctx->ctr,
                                    ctx->n_sm, ctx->st));
            ctx->slot_of_valid = false;  // looked up if SIG marks are ever needed (mark_table)
        } else {
            CK(launch_compact(table_of(ctx), ctx->cap, ctx->p.threshold,
                              window_fix ? ctx->wf_keep : nullptr, ctx->sig_key, ctx->sig_cnt,
                              ctx->parent, hash_k3 ? ctx->size : nullptr, ctx->npts,
                              ctx->min_key, ctx->root_cid, cols ? ctx->s_col_cnt : nullptr,
                              hash_k3 ? nullptr : ctx->slot_of, ctx->ctr, ctx->n_sm, ctx->st,
                              ctx->k2_lb));
            ctx->slot_of_valid = true;
        }
        ++ctx->launches;
        ctx->col_hist_ready = cols != 0;
        if (ctx->alt_dirty && ctx->slots_alt && ctx->cap_alt == ctx->cap) {
            // clear the idle table on aux_st while K3 runs (K3 is not
            // bandwidth-bound); the next ingest waits on ev_alt
            CK(cudaEventRecord(ctx->ev_alt, ctx->st));
            CK(cudaStreamWaitEvent(ctx->aux_st, ctx->ev_alt, 0));
            CK(launch_table_clear(ctx->slots_alt, ctx->cap_alt, ctx->n_sm, ctx->aux_st));
            ++ctx->launches;
            CK(cudaEventRecord(ctx->ev_alt, ctx->aux_st));
            ctx->alt_dirty = false;
            ctx->alt_ready = true;
        }
        ctx->sig_deferred = !hash_k3;
        ctx->table_cids = false;
    ctx->tile_cid_pending = false;
    }
    return RG_OK;
}

rg_status prune_impl(rg_ctx* ctx, bool window_fix = false) {
    PhaseTimer timer(ctx, &ctx->ms_prune);
    rg_status s = prune_enqueue(ctx, window_fix);
    if (s != RG_OK) return s;
    CK(cudaMemcpyAsync(&ctx->hctr->n_sig, &ctx->ctr->n_sig, sizeof(u64), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    timer.stop();
    ctx->n_sig = ctx->hctr->n_sig;
    ctx->state = rg_ctx::kSig;
    ctx->sorted = false;
    ctx->table_dirty = true;
    ctx->res = ctx->grid;
    ctx->res_is_canvas = true;
    ctx->n_roots = ctx->n_kept = 0;
    return RG_OK;
}


// Sorted K3. n = an upper bound of the significant count when `fused` (the
// kernels read the exact count from ctr->n_sig; CUB calls cover the bound,
// and entries past the count are never read back); results are read back by
// the caller then.
constexpr rg_status kK1Stopped = (rg_status)1000;  // internal: a deferred K1 round stopped

rg_status agglomerate_sorted_impl(rg_ctx* ctx, u64 n_bound = ~0ull, bool fused = false,
                                  bool check_k1 = false, bool speculate = false) {
    const u64 n = fused ? n_bound : ctx->n_sig;
    const int kb = (int)(ctx->res.bits_x + ctx->res.bits_y);
    if (ctx->s_cap < n || !ctx->s_flag) {
        dfree(ctx->s_flag);
        dfree(ctx->s_scan);
        dfree(ctx->s_clu_root);
        dfree(ctx->s_cid);
        ctx->s_cap = 0;
        const u64 c = std::max<u64>(n, 1024);
        CK(dalloc(&ctx->s_flag, c));
        CK(dalloc(&ctx->s_scan, c));
        CK(dalloc(&ctx->s_clu_root, c));
        CK(dalloc(&ctx->s_cid, c));
        ctx->s_cap = c;
    }
    const u64 ecap = std::max<u64>(n, 1024) * (u64)std::min(ctx->n_offsets, 12);
    if (ctx->s_edge_cap < ecap) {
        dfree(ctx->s_edges);
        ctx->s_edge_cap = 0;
        CK(dalloc(&ctx->s_edges, ecap));
        ctx->s_edge_cap = ecap;
    }
    const u64 cols = sorted_columns(ctx->res.bits_x);
    if (cols) {
        rg_status s = ensure_col_arrays(ctx, cols);
        if (s != RG_OK) return s;
    }
    const size_t tb = sorted_temp_bytes(n, kb, ctx->res.bits_x);
    if (ctx->sort_temp_bytes < tb || !ctx->sort_temp) {
        dfree(ctx->sort_temp);
        ctx->sort_temp_bytes = 0;
        CK(cudaMalloc(&ctx->sort_temp, tb));
        ctx->sort_temp_bytes = tb;
    }
    SortedLaunch L;
    L.sig_key = ctx->sig_key;
    L.sig_cnt = ctx->sig_cnt;
    L.n_sig_dev = &ctx->ctr->n_sig;
    L.n_sig = n;
    L.bits_y = ctx->res.bits_y;
    L.key_bits = (u32)kb;
    L.delta = ctx->p.distance;
    L.manhattan = ctx->p.metric == RG_METRIC_MANHATTAN;
    L.mu = ctx->p.min_cluster_size;
    L.iota = ctx->root_idx;
    L.ktmp = ctx->root_key;
    L.col_cnt = cols ? ctx->s_col_cnt : nullptr;
    L.col_off = cols ? ctx->s_col_off : nullptr;
    L.skey = ctx->root_key_sorted;
    L.perm = ctx->root_idx_sorted;
    L.parent = ctx->parent;
    L.size = ctx->size;
    L.npts = ctx->npts;
    L.flag = ctx->s_flag;
    L.scan = ctx->s_scan;
    L.tile_cid_b = nullptr;  // K2-order ids are scattered on demand (ensure_tile_cid)
    ctx->tile_cid_pending = true;
    L.cid_s = ctx->s_cid;
    L.clu_root = ctx->s_clu_root;
    L.edges = ctx->s_edges;
    L.edge_cap = ctx->s_edge_cap;
    L.temp = ctx->sort_temp;
    L.temp_bytes = ctx->sort_temp_bytes;
    L.ctr = ctx->ctr;
    L.host_ctr = ctx->hctr;
    L.n_sm = ctx->n_sm;
    // K2's histogram is valid for the set it compacted (canvas packing)
    L.col_hist_ready = ctx->col_hist_ready;
    ctx->npts_pending = false;
    L.npts_deferred = &ctx->npts_pending;
    ctx->col_hist_ready = false;  // one use: the segmented-sort path consumes col_cnt
    zero_field(ctx, &ctx->ctr->n_roots);
    zero_field(ctx, &ctx->ctr->n_kept);
    int launched = 0;
    L.launches = &launched;
    L.check_k1_stop = check_k1;
    L.speculate = speculate && fused;
    ctx->k3_speculated = false;
    L.speculated = &ctx->k3_speculated;
    const cudaError_t e3 = launch_agglomerate_sorted(L, ctx->st);
    ctx->launches += launched;
    if (e3 == cudaErrorNotReady && check_k1) return kK1Stopped;
    CK(e3);
    if (fused) return RG_OK;
    CK(cudaMemcpyAsync(&ctx->hctr->n_roots, &ctx->ctr->n_roots, 2 * sizeof(u64),
                       cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->n_roots = ctx->hctr->n_roots;
    ctx->n_kept = ctx->hctr->n_kept;
    ctx->sorted = true;
    return RG_OK;
}

rg_status agglomerate_impl(rg_ctx* ctx) {
    if (ctx->state == rg_ctx::kAccum)
        return set_err(ctx, RG_ERR_STATE, "agglomerate requires a pruned or loaded tile set");
    PhaseTimer timer(ctx, &ctx->ms_agg);
    ctx->n_roots = ctx->n_kept = 0;
    ctx->sorted = false;
    if (ctx->n_sig == 0) {
        ctx->state = rg_ctx::kAgg;
        return RG_OK;
    }
    if (use_sorted_k3(ctx)) {
        rg_status s = agglomerate_sorted_impl(ctx);
        if (s != RG_OK) return s;
        timer.stop();
        ctx->state = rg_ctx::kAgg;
        return RG_OK;
    }
    if (ctx->state == rg_ctx::kAgg) {
        // agglomerating the same set again: K2 / the load path initialised
        // the per-root accumulators only once
        CK(cudaMemsetAsync(ctx->size, 0, ctx->n_sig * sizeof(u32), ctx->st));
        CK(cudaMemsetAsync(ctx->npts, 0, ctx->n_sig * sizeof(u64), ctx->st));
        CK(cudaMemsetAsync(ctx->min_key, 0xff, ctx->n_sig * sizeof(u64), ctx->st));
        CK(cudaMemsetAsync(ctx->root_cid, 0xff, ctx->n_sig * sizeof(int), ctx->st));
    }
    {
        rg_status ms = mark_table(ctx, false);  // the hash-probe K3 resolves tiles via SIG marks
        if (ms != RG_OK) return ms;
    }
    ctx->tile_cid_pending = false;  // the hash-probe K3 writes tile_cid itself
    AggLaunch A;
    A.sig_key = ctx->sig_key;
    A.sig_cnt = ctx->sig_cnt;
    A.n_sig_dev = &ctx->ctr->n_sig;
    A.n_sig = ctx->n_sig;
    A.t = table_of(ctx);
    A.bits_y = ctx->res.bits_y;
    A.bits_x = ctx->res.bits_x;
    A.offsets = ctx->offsets;
    A.n_offsets = ctx->n_offsets;
    A.cheb1 = ctx->p.metric == RG_METRIC_CHEBYSHEV && ctx->p.distance == 1;
    A.mu = ctx->p.min_cluster_size;
    A.parent = ctx->parent;
    A.size = ctx->size;
    A.npts = ctx->npts;
    A.min_key = ctx->min_key;
    A.root_cid = ctx->root_cid;
    A.tile_cid = ctx->tile_cid;
    A.root_key = ctx->root_key;
    A.root_idx = ctx->root_idx;
    A.root_key_sorted = ctx->root_key_sorted;
    A.root_idx_sorted = ctx->root_idx_sorted;
    A.edges = ctx->edges;
    A.edge_n = ctx->edge_n;
    A.ctr = ctx->ctr;
    A.n_sm = ctx->n_sm;
    zero_field(ctx, &ctx->ctr->n_roots);
    zero_field(ctx, &ctx->ctr->n_kept);
    CK(launch_agglomerate(A, ctx->st));
    ctx->launches += 4;
    CK(cudaMemcpyAsync(&ctx->hctr->n_roots, &ctx->ctr->n_roots, 2 * sizeof(u64),
                       cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->n_roots = ctx->hctr->n_roots;
    ctx->n_kept = ctx->hctr->n_kept;
    rg_status s = ensure_sort_temp(ctx, ctx->n_kept, (int)(ctx->res.bits_x + ctx->res.bits_y));
    if (s != RG_OK) return s;
    A.sort_temp = ctx->sort_temp;
    A.sort_temp_bytes = ctx->sort_temp_bytes;
    CK(launch_order_and_label(A, ctx->n_kept, ctx->st));
    ctx->launches += ctx->n_kept ? 5 : 1;  // cub onesweep passes + ids + labels (approx.)
    CK(cudaStreamSynchronize(ctx->st));
    timer.stop();
    ctx->state = rg_ctx::kAgg;
    return RG_OK;
}

bool same_params(const rg_params& a, const rg_params& b) {
    return a.precision == b.precision && a.x_min == b.x_min && a.x_max == b.x_max &&
           a.y_min == b.y_min && a.y_max == b.y_max;
}

}  // namespace

// ============================================================== C-ABI

extern "C" {

int rg_abi_version(void) { return RG_ABI_VERSION; }

const char* rg_status_string(rg_status s) {
    switch (s) {
        case RG_OK: return "ok";
        case RG_ERR_CONFIG: return "config error";
        case RG_ERR_OOB: return "out of bounds";
        case RG_ERR_CUDA: return "cuda error";
        case RG_ERR_OOM: return "out of device memory";
        case RG_ERR_STATE: return "invalid state";
        case RG_ERR_ARG: return "invalid argument";
        case RG_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown";
}

int rg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int usable = 0;
    for (int d = 0; d < n; ++d) {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10 &&
            prop.minor == 0)
            ++usable;
    }
    return usable;
}

void rg_params_default(rg_params* out) {
    if (!out) return;
    std::memset(out, 0, sizeof *out);
    out->precision = 3.5;
    out->x_min = -180.0;
    out->x_max = 180.0;
    out->y_min = -90.0;
    out->y_max = 90.0;
    out->threshold = 5;
    out->distance = 1;
    out->metric = RG_METRIC_CHEBYSHEV;
    out->min_cluster_size = 4;
    out->mode = RG_MODE_COUNT_ONLY;
    out->oob_policy = RG_OOB_SKIP;
}

rg_status rg_params_validate(const rg_params* p, char* err, size_t err_len) {
    if (!p) return RG_ERR_ARG;
    std::string msg;
    rg_status s = validate(p, msg);
    if (err && err_len) {
        std::snprintf(err, err_len, "%s", msg.c_str());
    }
    return s;
}

double rg_params_scale(const rg_params* p) { return std::pow(10.0, p->precision); }

int64_t rg_params_min_column(const rg_params* p) {
    return (int64_t)std::floor(p->x_min * rg_params_scale(p));
}

int64_t rg_params_max_column(const rg_params* p) {
    return (int64_t)std::floor(p->x_max * rg_params_scale(p));
}

double rg_params_tile_bound(const rg_params* p) {
    // GridParams::tile_bound core.hpp:126-131
    const double s = rg_params_scale(p);
    const double cols = std::floor(p->x_max * s) - std::floor(p->x_min * s) + 1.0;
    const double rows = std::floor(p->y_max * s) - std::floor(p->y_min * s) + 1.0;
    return cols * rows;
}

const char* rg_last_error(const rg_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

rg_status rg_create(const rg_params* p, int device, rg_ctx** out) {
    if (!p || !out) return set_err(nullptr, RG_ERR_ARG, "null argument");
    *out = nullptr;
    std::string msg;
    rg_status vs = validate(p, msg);
    if (vs != RG_OK) return set_err(nullptr, vs, "%s", msg.c_str());
    int n_dev = 0;
    cudaError_t e = cudaGetDeviceCount(&n_dev);
    if (e != cudaSuccess || n_dev == 0) {
        cudaGetLastError();
        return set_err(nullptr, RG_ERR_CUDA, "no CUDA device available (%s)",
                       e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    }
    if (device < 0) cudaGetDevice(&device);
    if (device >= n_dev) return set_err(nullptr, RG_ERR_ARG, "device %d out of range", device);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return set_err(nullptr, RG_ERR_CUDA, "%s", cudaGetErrorString(e));
    if (prop.major != 10 || prop.minor != 0)
        return set_err(nullptr, RG_ERR_CUDA,
                       "device %d is sm_%d%d; this library is built for sm_100a only", device,
                       prop.major, prop.minor);
    DevGuard guard(device);
    {
        // keep freed stream-ordered scratch in the pool (see salloc)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            u64 keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    rg_ctx* ctx = new rg_ctx();
    ctx->p = *p;
    ctx->device = device;
    ctx->n_sm = prop.multiProcessorCount;
    ctx->grid = make_grid(*p);
    ctx->res = ctx->grid;
    {
        const double sc = ctx->grid.scale, lim = 2147483647.0;
        const double c[4] = {std::floor(p->x_min * sc), std::floor(p->x_max * sc),
                             std::floor(p->y_min * sc), std::floor(p->y_max * sc)};
        ctx->narrow = true;
        for (double v : c) ctx->narrow = ctx->narrow && v > -lim && v < lim;
    }
    ctx->max_warps = contract_max_warps(ctx->n_sm);
    auto fail = [&](cudaError_t err, const char* what) {
        set_err(nullptr, err == cudaErrorMemoryAllocation ? RG_ERR_OOM : RG_ERR_CUDA,
                "CUDA error in %s: %s", what, cudaGetErrorString(err));
        rg_destroy(ctx);
        return err == cudaErrorMemoryAllocation ? RG_ERR_OOM : RG_ERR_CUDA;
    };
    if ((e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(e, "stream");
    ctx->st = ctx->own;
    if ((e = cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking)) != cudaSuccess)
        return fail(e, "stream");
    {
        // side work (the idle table's clear, a deferred KP3) yields to the main stream
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&ctx->aux_st, cudaStreamNonBlocking, lo)) != cudaSuccess)
            return fail(e, "stream");
    }
    if ((e = cudaEventCreateWithFlags(&ctx->ev_kp3, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "event");
    if ((e = cudaEventCreateWithFlags(&ctx->ev_alt, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->t0)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->ev_k2)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->ev_k3)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->ev_end)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->ev_c0)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->ev_c1)) != cudaSuccess) return fail(e, "event");
    if ((e = cudaEventCreate(&ctx->t1)) != cudaSuccess) return fail(e, "event");
    for (int b = 0; b < 2; ++b) {
        if ((e = cudaEventCreateWithFlags(&ctx->copied[b], cudaEventDisableTiming)) !=
            cudaSuccess)
            return fail(e, "event");
        if ((e = cudaEventCreateWithFlags(&ctx->done[b], cudaEventDisableTiming)) != cudaSuccess)
            return fail(e, "event");
    }
    if ((e = dalloc(&ctx->ctr, 1)) != cudaSuccess) return fail(e, "cudaMalloc counters");
    if ((e = cudaMallocHost((void**)&ctx->hctr, sizeof(Counters))) != cudaSuccess)
        return fail(e, "cudaMallocHost");
    std::memset(ctx->hctr, 0, sizeof(Counters));
    if ((e = cudaMemset(ctx->ctr, 0, sizeof(Counters))) != cudaSuccess)
        return fail(e, "cudaMemset");
    for (int b = 0; b < 2; ++b)
        if ((e = dalloc(&ctx->part[b], 2 * (u64)ctx->max_warps + 64)) != cudaSuccess)  // <= 2 per warp
            return fail(e, "cudaMalloc partials");
    if ((e = dalloc(&ctx->scratch, 8)) != cudaSuccess) return fail(e, "cudaMalloc scratch");
    const std::vector<int2> off = forward_offsets(*p);
    ctx->n_offsets = (int)off.size();
    if ((e = dalloc(&ctx->offsets, off.size())) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMemcpy(ctx->offsets, off.data(), off.size() * sizeof(int2),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(e, "cudaMemcpy offsets");
    *out = ctx;
    return RG_OK;
}

void rg_destroy(rg_ctx* ctx) {
    if (!ctx) return;
    DevGuard guard(ctx->device);
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->copy_st) cudaStreamSynchronize(ctx->copy_st);
    if (ctx->aux_st) cudaStreamSynchronize(ctx->aux_st);
    dfree(ctx->slots);
    dfree(ctx->slots_alt);
    dfree(ctx->ctr);
    if (ctx->hctr) cudaFreeHost(ctx->hctr);
    dfree(ctx->part[0]);
    dfree(ctx->part[1]);
    dfree(ctx->scratch);
    dfree(ctx->wf_keep);
    dfree(ctx->ps);
    dfree(ctx->ut);
    dfree(ctx->cp_xy);
    dfree(ctx->cp_off);
    dfree(ctx->sig_key);
    dfree(ctx->sig_cnt);
    dfree(ctx->npts);
    dfree(ctx->min_key);
    dfree(ctx->parent);
    dfree(ctx->size);
    dfree(ctx->tile_cid);
    dfree(ctx->slot_of);
    dfree(ctx->root_cid);
    dfree(ctx->root_key);
    dfree(ctx->root_key_sorted);
    dfree(ctx->root_idx);
    dfree(ctx->root_idx_sorted);
    dfree(ctx->edges);
    dfree(ctx->edge_n);
    dfree(ctx->s_flag);
    dfree(ctx->s_scan);
    dfree(ctx->s_clu_root);
    dfree(ctx->s_cid);
    dfree(ctx->s_edges);
    dfree(ctx->s_col_cnt);
    dfree(ctx->s_col_off);
    if (ctx->part_scratch) cudaFree(ctx->part_scratch);
    ctx->part_scratch = nullptr;
    dfree(ctx->pair_key);
    dfree(ctx->pair_cnt);
    dfree(ctx->lk_tab);
    dfree(ctx->lk_ids);
    dfree(ctx->k2_lb);
    for (int b = 0; b < 2; ++b) {
        if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
        if (ctx->pin_free[b]) cudaEventDestroy(ctx->pin_free[b]);
    }
    dfree(ctx->sort_temp);
    dfree(ctx->offsets);
    for (int b = 0; b < 2; ++b) {
        dfree(ctx->stage[b]);
        dfree(ctx->lstage[b]);
        if (ctx->copied[b]) cudaEventDestroy(ctx->copied[b]);
        if (ctx->done[b]) cudaEventDestroy(ctx->done[b]);
    }
    if (ctx->t0) cudaEventDestroy(ctx->t0);
    if (ctx->ev_k2) cudaEventDestroy(ctx->ev_k2);
    if (ctx->ev_k3) cudaEventDestroy(ctx->ev_k3);
    if (ctx->ev_end) cudaEventDestroy(ctx->ev_end);
    if (ctx->t1) cudaEventDestroy(ctx->t1);
    if (ctx->ev_alt) cudaEventDestroy(ctx->ev_alt);
    if (ctx->ev_kp3) cudaEventDestroy(ctx->ev_kp3);
    if (ctx->aux_st) cudaStreamDestroy(ctx->aux_st);
    if (ctx->copy_st) cudaStreamDestroy(ctx->copy_st);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

rg_status rg_set_stream(rg_ctx* ctx, void* stream) {
    if (!ctx) return RG_ERR_ARG;
    DevGuard guard(ctx->device);
    CK(cudaStreamSynchronize(ctx->st));
    ctx->st = stream ? (cudaStream_t)stream : ctx->own;
    return RG_OK;
}

rg_status rg_synchronize(rg_ctx* ctx) {
    if (!ctx) return RG_ERR_ARG;
    DevGuard guard(ctx->device);
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

static rg_status settle_stream(rg_ctx* ctx);

rg_status rg_ingest(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (n && !xy) return set_err(ctx, RG_ERR_ARG, "null point buffer");
    DevGuard guard(ctx->device);
    return ingest_any(ctx, xy, n, kind);
}

// ------------------------------------------------------ streaming ingest
// PointSource reads (io.hpp:21-36) drained chunk by chunk (ingest_all
// io.hpp:226-241) with the source's next read overlapped with the current
// chunk's H2D copy and K1: the context hands out one of two pinned host
// buffers, the caller fills it, rg_stream_submit enqueues the copy (copy
// stream) and K1 (compute stream) and returns; K1's stop check of a chunk
// runs when the next chunk is submitted (or at rg_stream_end).
rg_status rg_stream_begin(rg_ctx* ctx, uint64_t chunk_points) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx->streaming) return set_err(ctx, RG_ERR_STATE, "a stream is already open");
    DevGuard guard(ctx->device);
    rg_status s = reopen_accumulator(ctx);
    if (s != RG_OK) return s;
    const u64 want = std::max<u64>(1024, std::min<u64>(chunk_points ? chunk_points : (1ull << 22),
                                                       kStagePoints));
    if (ctx->pin_pts < want) {
        for (int b = 0; b < 2; ++b) {
            if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
            ctx->pin[b] = nullptr;
        }
        ctx->pin_pts = 0;
        for (int b = 0; b < 2; ++b) {
            CK(cudaMallocHost((void**)&ctx->pin[b], want * 2 * sizeof(double)));
            if (!ctx->pin_free[b]) CK(cudaEventCreateWithFlags(&ctx->pin_free[b],
                                                               cudaEventDisableTiming));
        }
        ctx->pin_pts = want;
    }
    s = ensure_stage(ctx, ctx->pin_pts, false);
    if (s != RG_OK) return s;
    ctx->pin_next = 0;
    ctx->pin_held = -1;
    ctx->stream_chunks = 0;
    ctx->chunk_verdict = -1;
    ctx->streaming = true;
    return RG_OK;
}

rg_status rg_stream_buffer(rg_ctx* ctx, double** buf, uint64_t* capacity) {
    if (!ctx || !buf || !capacity) return RG_ERR_ARG;
    if (!ctx->streaming) return set_err(ctx, RG_ERR_STATE, "rg_stream_begin first");
    DevGuard guard(ctx->device);
    const int b = ctx->pin_next;
    CK(cudaEventSynchronize(ctx->pin_free[b]));  // (never recorded: complete)
    ctx->pin_held = b;
    *buf = ctx->pin[b];
    *capacity = ctx->pin_pts;
    return RG_OK;
}

rg_status rg_stream_submit(rg_ctx* ctx, uint64_t n) {
    if (!ctx) return RG_ERR_ARG;
    if (!ctx->streaming || ctx->pin_held < 0)
        return set_err(ctx, RG_ERR_STATE, "rg_stream_buffer first");
    if (n > ctx->pin_pts) return set_err(ctx, RG_ERR_ARG, "more points than the buffer holds");
    DevGuard guard(ctx->device);
    const int b = ctx->pin_held;
    ctx->pin_held = -1;
    ctx->pin_next = 1 - b;
    if (n == 0) return RG_OK;
    if (ctx->k1.active) {  // the previous chunk's stop check (it has usually finished)
        rg_status s = k1_finish(ctx);
        if (s != RG_OK) return s;
    }
    CK(cudaStreamWaitEvent(ctx->copy_st, ctx->done[b], 0));  // device staging b is free
    CK(cudaMemcpyAsync(ctx->stage[b], ctx->pin[b], n * 2 * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->copy_st));
    CK(cudaEventRecord(ctx->pin_free[b], ctx->copy_st));
    CK(cudaEventRecord(ctx->copied[b], ctx->copy_st));
    CK(cudaStreamWaitEvent(ctx->st, ctx->copied[b], 0));
    bool oob = false;
    double ox = 0, oy = 0;
    rg_status s = ingest_span(ctx, ctx->stage[b], n, &oob, &ox, &oy,
                              ctx->p.oob_policy != RG_OOB_STRICT);
    if (s != RG_OK) return s;
    CK(cudaEventRecord(ctx->done[b], ctx->st));
    // the first chunk's order verdict holds for the rest of the stream
    if (ctx->stream_chunks++ == 0 && ctx->probe_ptr == ctx->stage[b])
        ctx->chunk_verdict = ctx->probe_unordered;
    if (oob) {
        ctx->streaming = false;
        ctx->chunk_verdict = -1;
        CK(cudaStreamSynchronize(ctx->copy_st));
        return oob_error(ctx, ox, oy);
    }
    return RG_OK;
}

rg_status rg_stream_end(rg_ctx* ctx) {
    if (!ctx) return RG_ERR_ARG;
    if (!ctx->streaming) return RG_OK;
    DevGuard guard(ctx->device);
    ctx->streaming = false;
    ctx->chunk_verdict = -1;
    if (ctx->k1.active) {
        rg_status s = k1_finish(ctx);
        if (s != RG_OK) return s;
    }
    CK(cudaStreamSynchronize(ctx->copy_st));
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

// Any other call on a context with an open stream closes it first (its
// counters and table must be final).
static rg_status settle_stream(rg_ctx* ctx) {
    if (ctx->insert_pending) {  // (only after an error between ingest and prune)
        DevGuard guard(ctx->device);
        const rg_status si = settle_insert(ctx);
        if (si != RG_OK) return si;
    }
    return ctx->streaming ? rg_stream_end(ctx) : RG_OK;
}

static rg_status clone_into(rg_ctx* ctx, rg_ctx* src) {
    if (src->state == rg_ctx::kAccum && src->slots && src->used) {
        CK(dalloc(&ctx->slots, src->cap));
        ctx->cap = src->cap;
        CK(cudaStreamSynchronize(src->st));
        CK(cudaMemcpyAsync(ctx->slots, src->slots, src->cap * sizeof(Slot),
                           cudaMemcpyDeviceToDevice, ctx->st));
        ctx->used = src->used;
    }
    if (src->state == rg_ctx::kAccum && src->ps && src->ps_used) {
        CK(dalloc(&ctx->ps, src->ps_cap));
        CK(dalloc(&ctx->ut, src->ut_cap));
        CK(cudaMemcpyAsync(ctx->ps, src->ps, src->ps_cap * sizeof(PtKey),
                           cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaMemcpyAsync(ctx->ut, src->ut, src->ut_cap * sizeof(Slot),
                           cudaMemcpyDeviceToDevice, ctx->st));
        ctx->ps_cap = src->ps_cap;
        ctx->ut_cap = src->ut_cap;
        ctx->ps_used = src->ps_used;
    }
    ctx->ingested = src->ingested;
    ctx->skipped = src->skipped;
    rg_status s = push_counters(ctx);
    if (s != RG_OK) return s;
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

rg_status rg_clone(rg_ctx* src, rg_ctx** out) {
    if (!src || !out) return set_err(nullptr, RG_ERR_ARG, "null argument");
    if (src) {
        const rg_status ss = settle_stream(src);
        if (ss != RG_OK) return ss;
    }
    *out = nullptr;
    rg_ctx* dst = nullptr;
    rg_status s = rg_create(&src->p, src->device, &dst);
    if (s != RG_OK) return s;
    DevGuard guard(src->device);
    s = clone_into(dst, src);
    if (s != RG_OK) {
        set_err(nullptr, s, "%s", rg_last_error(dst));
        rg_destroy(dst);
        return s;
    }
    *out = dst;
    return RG_OK;
}

rg_status rg_merge(rg_ctx* dst, rg_ctx* src) {
    if (dst) {
        const rg_status ss = settle_stream(dst);
        if (ss != RG_OK) return ss;
    }
    rg_ctx* ctx = dst;
    if (!dst || !src) return RG_ERR_ARG;
    if (dst == src) return set_err(dst, RG_ERR_ARG, "cannot merge an accumulator into itself");
    if (!same_params(dst->p, src->p))
        return set_err(dst, RG_ERR_CONFIG, "merge requires equal grid parameters");
    if (dst->device != src->device)
        return set_err(dst, RG_ERR_UNSUPPORTED, "merge across devices is not supported");
    DevGuard guard(dst->device);
    rg_status s = reopen_accumulator(dst);
    if (s != RG_OK) return s;
    {
        rg_ctx* c2 = src;
        if (c2->state != rg_ctx::kAccum) {
            s = reopen_accumulator(c2);
            if (s != RG_OK) return set_err(dst, s, "%s", c2->err.c_str());
        }
        cudaStreamSynchronize(c2->st);
    }
    if (src->slots && src->used) {
        const u64 need = (u64)((double)(dst->used + src->used) / kMaxLoad) + 1;
        if (!dst->slots || dst->cap < need) {
            s = grow_table(dst, table_cap(need));
            if (s != RG_OK) return s;
        }
        CK(cudaMemsetAsync(dst->scratch, 0, sizeof(u64), dst->st));
        CK(launch_table_fold(src->slots, src->cap, table_of(dst), dst->scratch, dst->n_sm,
                             dst->st));
        ++dst->launches;
        u64 claimed = 0;
        CK(cudaMemcpyAsync(&dst->hctr->pad0[0], dst->scratch, sizeof(u64),
                           cudaMemcpyDeviceToHost, dst->st));
        CK(cudaStreamSynchronize(dst->st));
        claimed = dst->hctr->pad0[0];
        dst->used += claimed;
    }
    if (dedupe_active(dst) && src->ps && src->ps_used) {
        // the merged point multiset is deduplicated as a whole at prune
        s = ensure_ut(dst);
        if (s != RG_OK) return s;
        s = ensure_ps(dst, src->ps_used);
        if (s != RG_OK) return s;
        CK(cudaMemsetAsync(dst->scratch, 0, sizeof(u64), dst->st));
        CK(launch_ps_fold(src->ps, src->ps_cap, dst->grid, point_set(dst), ut_table(dst),
                          dst->scratch, dst->n_sm, dst->st));
        ++dst->launches;
        CK(cudaMemcpyAsync(&dst->hctr->pad0[0], dst->scratch, sizeof(u64),
                           cudaMemcpyDeviceToHost, dst->st));
        CK(cudaStreamSynchronize(dst->st));
        dst->ps_used += dst->hctr->pad0[0];
    }
    dst->ingested += src->ingested;
    dst->skipped += src->skipped;
    s = push_counters(dst);
    if (s != RG_OK) return s;
    CK(cudaStreamSynchronize(dst->st));  // the folds above read src's buffers
    // Leave src empty (accumulator.hpp:150-153).
    {
        DevGuard g2(src->device);
        rg_ctx* c2 = src;
        if (c2->slots) {
            cudaError_t e = launch_table_clear(c2->slots, c2->cap, c2->n_sm, c2->st);
            ++c2->launches;
            if (e != cudaSuccess) return cuda_err(dst, e, "clear merged source");
        }
        if (c2->ps && c2->ps_used) {
            CK(cudaMemsetAsync(c2->ps, 0xff, c2->ps_cap * sizeof(PtKey), c2->st));
            CK(launch_table_clear(c2->ut, c2->ut_cap, c2->n_sm, c2->st));
            ++c2->launches;
        }
        c2->ps_used = 0;
        c2->used = c2->ingested = c2->skipped = 0;
        s = push_counters(c2);
        if (s != RG_OK) return set_err(dst, s, "%s", c2->err.c_str());
    }
    return RG_OK;
}

rg_status rg_key_packing(rg_ctx* ctx, int64_t* origin_x, int64_t* origin_y, uint32_t* bits_y) {
    if (!ctx) return RG_ERR_ARG;
    if (origin_x) *origin_x = ctx->grid.origin_x;
    if (origin_y) *origin_y = ctx->grid.origin_y;
    if (bits_y) *bits_y = ctx->grid.bits_y;
    return RG_OK;
}

rg_status rg_export_entries(rg_ctx* ctx, uint64_t* keys, uint64_t* counts, uint64_t cap,
                            uint64_t* n_out, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    const u64 d = (ctx->state == rg_ctx::kAccum && ctx->slots) ? ctx->used : 0;
    if (n_out) *n_out = d;
    if (d == 0 || cap == 0) return RG_OK;
    if (cap < d) return set_err(ctx, RG_ERR_ARG, "export buffer holds %llu of %llu entries",
                                (unsigned long long)cap, (unsigned long long)d);
    if (!keys || !counts) return set_err(ctx, RG_ERR_ARG, "null buffer");
    DevGuard guard(ctx->device);
    u64 *dk = (u64*)keys, *dc = (u64*)counts;
    if (kind == RG_MEM_HOST) {
        CK(dalloc(&dk, d));
        CK(dalloc(&dc, d));
    }
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(u64), ctx->st));
    CK(launch_export(ctx->slots, ctx->cap, dk, dc, ctx->scratch, ctx->n_sm, ctx->st));
    ++ctx->launches;
    if (kind == RG_MEM_HOST) {
        CK(cudaMemcpyAsync(keys, dk, d * 8, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaMemcpyAsync(counts, dc, d * 8, cudaMemcpyDeviceToHost, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    if (kind == RG_MEM_HOST) {
        dfree(dk);
        dfree(dc);
    }
    return RG_OK;
}

rg_status rg_route_pairs(rg_ctx* ctx, const uint64_t* keys, const uint64_t* counts, uint64_t n,
                         int64_t col_min, uint64_t col_width, const uint32_t* bin_splits,
                         uint32_t n_parts, uint64_t* out_keys, uint64_t* out_counts,
                         uint64_t* part_counts) {
    if (!ctx) return RG_ERR_ARG;
    if (n_parts == 0 || n_parts > 1024 || col_width == 0)
        return set_err(ctx, RG_ERR_ARG, "rg_route_pairs: 1..1024 parts and a positive width");
    if (!part_counts || (n && (!keys || !counts || !out_keys || !out_counts)) ||
        (n_parts > 1 && !bin_splits))
        return set_err(ctx, RG_ERR_ARG, "null buffer");
    DevGuard guard(ctx->device);
    CK(cudaMemsetAsync(part_counts, 0, n_parts * sizeof(u64), ctx->st));
    if (n) {
        u64* cursor = nullptr;
        CK(salloc(&cursor, n_parts, ctx->st));
        const u32 by = ctx->grid.bits_y;
        const int g = grid_for(n, ctx->n_sm, 8);
        const u64* k = (const u64*)keys;
        const u64* c = (const u64*)counts;
        u64* pc = (u64*)part_counts;
        k_route_count<<<g, 256, 0, ctx->st>>>(k, n, by, (long long)col_min, col_width, bin_splits,
                                              n_parts, pc);
        k_route_offsets<<<1, 32, 0, ctx->st>>>(pc, n_parts, cursor);
        k_route_scatter<<<g, 256, 0, ctx->st>>>(k, c, n, by, (long long)col_min, col_width,
                                                bin_splits, n_parts, cursor, (u64*)out_keys,
                                                (u64*)out_counts);
        ctx->launches += 3;
        CK(cudaGetLastError());
        sfree(cursor, ctx->st);
    }
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

rg_status rg_ingest_counts(rg_ctx* ctx, const uint64_t* keys, const uint64_t* counts,
                           uint64_t n, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (dedupe_active(ctx))
        return set_err(ctx, RG_ERR_UNSUPPORTED,
                       "count pairs cannot be deduplicated (dedupe_points needs the points)");
    if (n && (!keys || !counts)) return set_err(ctx, RG_ERR_ARG, "null buffer");
    DevGuard guard(ctx->device);
    rg_status s = reopen_accumulator(ctx);
    if (s != RG_OK) return s;
    if (n == 0) return RG_OK;
    const u64 need = (u64)((double)(ctx->used + n) / kMaxLoad) + 1;
    if (!ctx->slots || ctx->cap < need) {
        s = grow_table(ctx, table_cap(need));
        if (s != RG_OK) return s;
    }
    const u64 *dk = (const u64*)keys, *dc = (const u64*)counts;
    u64 *tk = nullptr, *tc = nullptr;
    if (kind == RG_MEM_HOST) {
        CK(dalloc(&tk, n));
        CK(dalloc(&tc, n));
        CK(cudaMemcpyAsync(tk, keys, n * 8, cudaMemcpyHostToDevice, ctx->st));
        CK(cudaMemcpyAsync(tc, counts, n * 8, cudaMemcpyHostToDevice, ctx->st));
        dk = tk;
        dc = tc;
    }
    // keys must come from rg_export_entries / rg_route_pairs of a context with
    // the same parameters: anything else would alias the table's EMPTY word
    CK(cudaMemsetAsync(ctx->scratch, 0, 3 * sizeof(u64), ctx->st));
    {
        const u64 want = (n + 255) / 256;
        k_check_keys<<<(int)std::max<u64>(1, std::min<u64>(want, (u64)ctx->n_sm * 8)), 256, 0,
                       ctx->st>>>(dk, n, ctx->res.bits_x + ctx->res.bits_y, ctx->scratch + 2);
        ++ctx->launches;
        u64 bad = 0;
        CK(cudaMemcpyAsync(&bad, ctx->scratch + 2, sizeof bad, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (bad) {
            dfree(tk);
            dfree(tc);
            return set_err(ctx, RG_ERR_ARG,
                           "%llu of %llu keys are not packed keys of this context (use "
                           "rg_export_entries of a context with the same parameters)",
                           (unsigned long long)bad, (unsigned long long)n);
        }
    }
    CK(launch_pairs_fold(dk, dc, n, table_of(ctx), ctx->scratch, ctx->scratch + 1, ctx->n_sm,
                         ctx->st));
    ++ctx->launches;
    CK(cudaMemcpyAsync(&ctx->hctr->pad0[0], ctx->scratch, 2 * sizeof(u64), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    dfree(tk);
    dfree(tc);
    ctx->used += ctx->hctr->pad0[0];
    ctx->ingested += ctx->hctr->pad0[1];
    return push_counters(ctx);
}

rg_status rg_entry_count(rg_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    *out = ctx->state == rg_ctx::kAccum ? ctx->used : 0;
    return RG_OK;
}

rg_status rg_total_ingested(rg_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    *out = ctx->ingested;
    return RG_OK;
}

rg_status rg_skipped(rg_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    *out = ctx->skipped;
    return RG_OK;
}

rg_status rg_count_of(rg_ctx* ctx, int64_t tx, int64_t ty, uint64_t* out) {
    if (!ctx || !out) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    *out = 0;
    if (ctx->state != rg_ctx::kAccum || !ctx->slots || ctx->used == 0) return RG_OK;
    const Grid& g = ctx->grid;
    const long long kx = tx - g.origin_x, ky = ty - g.origin_y;
    if (kx < 0 || ky < 0 || kx >= (1ll << g.bits_x) || ky >= (1ll << g.bits_y)) return RG_OK;
    DevGuard guard(ctx->device);
    const u64 key = ((u64)kx << g.bits_y) | (u64)ky;
    k_count_of<<<1, 1, 0, ctx->st>>>(table_of(ctx), key, ctx->scratch);
    ++ctx->launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&ctx->hctr->pad0[1], ctx->scratch, sizeof(u64), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    *out = ctx->hctr->pad0[1];
    return RG_OK;
}

rg_status rg_export_counts(rg_ctx* ctx, int64_t* tx, int64_t* ty, uint64_t* count, uint64_t cap,
                           uint64_t* n_out) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (ctx->state != rg_ctx::kAccum || !ctx->slots || ctx->used == 0) {
        if (n_out) *n_out = 0;
        return RG_OK;
    }
    DevGuard guard(ctx->device);
    std::vector<Slot> host(ctx->cap);
    CK(cudaMemcpyAsync(host.data(), ctx->slots, ctx->cap * sizeof(Slot), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    std::vector<std::pair<u64, u64>> rows;
    rows.reserve(ctx->used);
    for (const Slot& s : host)
        if (s.key != kEmpty) rows.emplace_back(s.key, s.count);
    std::sort(rows.begin(), rows.end());
    const Grid& g = ctx->grid;
    const u64 ymask = (1ull << g.bits_y) - 1;
    const u64 w = std::min<u64>(cap, rows.size());
    for (u64 i = 0; i < w; ++i) {
        if (tx) tx[i] = g.origin_x + (long long)(rows[i].first >> g.bits_y);
        if (ty) ty[i] = g.origin_y + (long long)(rows[i].first & ymask);
        if (count) count[i] = rows[i].second;
    }
    if (n_out) *n_out = rows.size();
    return RG_OK;
}

rg_status rg_prune(rg_ctx* ctx, uint64_t* n_significant) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    DevGuard guard(ctx->device);
    rg_status s = prune_impl(ctx);
    if (s == RG_OK && n_significant) *n_significant = ctx->n_sig;
    return s;
}

rg_status rg_window_fix(rg_ctx* ctx, uint64_t* n_significant) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    DevGuard guard(ctx->device);
    rg_status s = prune_impl(ctx, true);
    if (s == RG_OK && n_significant) *n_significant = ctx->n_sig;
    return s;
}

rg_status rg_load_significant(rg_ctx* ctx, const int64_t* tx, const int64_t* ty,
                              const uint64_t* count, uint64_t n, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (n && (!tx || !ty)) return set_err(ctx, RG_ERR_ARG, "null tile buffer");
    if (n >= 0x7fffffffull) return set_err(ctx, RG_ERR_UNSUPPORTED, "too many tiles");
    DevGuard guard(ctx->device);
    // Tile extents decide the key packing: the canvas packing when every tile
    // lies on the canvas (then labelling points works), else a packing that
    // covers the tiles' bounding box.
    long long mnx = 0, mxx = 0, mny = 0, mxy = 0;
    if (kind == RG_MEM_DEVICE && n) {
        long long* ext = (long long*)&ctx->hctr->pad0[0];  // pinned
        ext[0] = LLONG_MAX;
        ext[1] = LLONG_MIN;
        ext[2] = LLONG_MAX;
        ext[3] = LLONG_MIN;
        CK(cudaMemcpyAsync(ctx->scratch, ext, 4 * 8, cudaMemcpyHostToDevice, ctx->st));
        CK(launch_tile_extents((const long long*)tx, (const long long*)ty, n,
                               (long long*)ctx->scratch, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaMemcpyAsync(ext, ctx->scratch, 4 * 8, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        mnx = ext[0], mxx = ext[1], mny = ext[2], mxy = ext[3];
    }
    for (u64 i = 0; kind != RG_MEM_DEVICE && i < n; ++i) {
        if (i == 0 || tx[i] < mnx) mnx = tx[i];
        if (i == 0 || tx[i] > mxx) mxx = tx[i];
        if (i == 0 || ty[i] < mny) mny = ty[i];
        if (i == 0 || ty[i] > mxy) mxy = ty[i];
    }
    const Grid& g = ctx->grid;
    Grid res = g;
    bool on_canvas = n == 0 || (mnx >= g.origin_x && mny >= g.origin_y &&
                                (u64)(mxx - g.origin_x) < (1ull << g.bits_x) &&
                                (u64)(mxy - g.origin_y) < (1ull << g.bits_y));
    if (!on_canvas) {
        const double w = (double)mxx - (double)mnx + 1.0;
        const double h = (double)mxy - (double)mny + 1.0;
        const u32 bx = bits_for(w), by = std::max<u32>(kBlockBits, bits_for(h));
        if (bx + by > 63)
            return set_err(ctx, RG_ERR_UNSUPPORTED,
                           "tile set spans too large a range for a 63-bit packed key");
        res.origin_x = mnx;
        res.origin_y = mny;
        res.ox32 = (int)mnx;
        res.oy32 = (int)mny;
        res.bits_x = bx;
        res.bits_y = by;
    }
    // Fresh table sized for n keys.
    ctx->state = rg_ctx::kAccum;
    ctx->table_dirty = true;
    rg_status s = reopen_accumulator(ctx);
    if (s != RG_OK) return s;
    const u64 need = next_pow2(std::max<u64>((u64)((double)n / 0.5) + 1, 1024));
    if (!ctx->slots || ctx->cap < need) {
        if (ctx->slots) dfree(ctx->slots);
        ctx->cap = 0;
        s = alloc_table(ctx, need, &ctx->slots);
        if (s != RG_OK) return s;
        ctx->cap = need;
    }
    ctx->res = res;  // the table is keyed with this packing
    s = ensure_sig_capacity(ctx, n);
    if (s != RG_OK) return s;
    if (n) {
        const long long* dtx = (const long long*)tx;
        const long long* dty = (const long long*)ty;
        const u64* dcnt = (const u64*)count;
        long long *htx = nullptr, *hty = nullptr;
        u64* hcnt = nullptr;
        if (kind == RG_MEM_HOST) {
            CK(dalloc(&htx, n));
            CK(dalloc(&hty, n));
            CK(cudaMemcpyAsync(htx, tx, n * 8, cudaMemcpyHostToDevice, ctx->st));
            CK(cudaMemcpyAsync(hty, ty, n * 8, cudaMemcpyHostToDevice, ctx->st));
            if (count) {
                CK(dalloc(&hcnt, n));
                CK(cudaMemcpyAsync(hcnt, count, n * 8, cudaMemcpyHostToDevice, ctx->st));
            }
            dtx = htx, dty = hty, dcnt = hcnt;
        }
        CK(launch_load_tiles(dtx, dty, dcnt, n, res.origin_x, res.origin_y, res.bits_y,
                             table_of(ctx), ctx->sig_key, ctx->sig_cnt, ctx->parent, ctx->size,
                             ctx->npts, ctx->min_key, ctx->root_cid, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaStreamSynchronize(ctx->st));
        dfree(htx);
        dfree(hty);
        dfree(hcnt);
    }
    ctx->hctr->n_sig = n;
    CK(cudaMemcpyAsync(&ctx->ctr->n_sig, &ctx->hctr->n_sig, sizeof(u64), cudaMemcpyHostToDevice,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->used = n;
    ctx->n_sig = n;
    ctx->res = res;
    ctx->res_is_canvas = on_canvas;
    ctx->col_hist_ready = false;
    ctx->sig_deferred = false;
    ctx->table_cids = false;
    ctx->tile_cid_pending = false;
    ctx->state = rg_ctx::kSig;
    ctx->sorted = false;
    ctx->table_dirty = true;
    return RG_OK;
}

rg_status rg_agglomerate(rg_ctx* ctx, uint64_t* n_clusters) {
    if (!ctx) return RG_ERR_ARG;
    DevGuard guard(ctx->device);
    rg_status s = agglomerate_impl(ctx);
    if (s == RG_OK && n_clusters) *n_clusters = ctx->n_kept;
    return s;
}

rg_status rg_get_stats(rg_ctx* ctx, rg_stats* out) {
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (ctx) resolve_contract_timer(ctx);
    if (!ctx || !out) return RG_ERR_ARG;
    std::memset(out, 0, sizeof *out);
    out->n_points = ctx->ingested + ctx->skipped;
    out->n_ingested = ctx->ingested;
    out->n_skipped = ctx->skipped;
    out->peak_accumulator_entries = ctx->used;
    out->n_significant = ctx->state == rg_ctx::kAccum ? 0 : ctx->n_sig;
    out->n_components = ctx->n_roots;
    out->n_clusters = ctx->n_kept;
    out->table_capacity = ctx->cap;
    out->table_grows = ctx->grows;
    out->ms_contract = ctx->ms_contract;
    out->ms_prune = ctx->ms_prune;
    out->ms_agglomerate = ctx->ms_agg;
    out->ms_label = ctx->ms_label;
    return RG_OK;
}

// cluster_sequential's prune + agglomerate on the sorted K3 path with one
// host synchronisation at the end: K2 leaves the significant count on the
// device and K3 is sized by the entry count (its upper bound). Phase times
// come from events read after the final synchronisation.
// K2 + K3 enqueued back to back with one host read in between (K3 sizes its
// launches from the significant count and the longest column). When K1's
// stop check was deferred (rg_cluster on a device span), that read also
// carries K1's counters; if a warp ran out of budget the speculative K2/K3
// are dropped, K1 is finished (growth, resumed segments) and K2/K3 rerun.
rg_status prune_agglomerate_fused(rg_ctx* ctx, bool window_fix) {
    const bool deferred = ctx->k1.active;
    CK(cudaEventRecord(ctx->ev_k2, ctx->st));
    rg_status s = prune_enqueue(ctx, window_fix);
    if (s != RG_OK) return s;
    CK(cudaEventRecord(ctx->ev_k3, ctx->st));
    const u64 bound = deferred ? k1_used_bound(ctx) : ctx->used;
    ctx->n_roots = ctx->n_kept = 0;
    // K3 without its sizing read: launches sized for the bound, the exact
    // count read on the device, the bucketed path assumed; max_col and K1's
    // stop flag are checked in the counters read at the end of the call
    // (RG_K3_SPEC=0: always wait for the sizing read).
    static const bool spec_off = [] {
        const char* v = std::getenv("RG_K3_SPEC");
        return v && std::strcmp(v, "0") == 0;
    }();
    ctx->k3_speculated = false;
    if (bound) {
        // Only for small tables: with a large one the host read's bubble is
        // where the idle table's clear (0.5 GB of writes for config 4) runs
        // alone; without the bubble it competes with K3 (config 4: 2.46 ->
        // 2.56 ms), while config 1 gains 5 % (0.211 -> 0.201 ms).
        const bool small_table = ctx->cap * sizeof(Slot) <= (64ull << 20);
        s = agglomerate_sorted_impl(ctx, bound, true, deferred,
                                    !spec_off && !ctx->k3_no_spec && small_table);
        if (s == kK1Stopped) {
            s = k1_finish(ctx);
            if (s != RG_OK) return s;
            return prune_agglomerate_fused(ctx, window_fix);
        }
        if (s != RG_OK) return s;
    } else {
        zero_field(ctx, &ctx->ctr->n_roots);
        zero_field(ctx, &ctx->ctr->n_kept);
    }
    CK(cudaEventRecord(ctx->ev_end, ctx->st));
    {  // the table is complete when the call returns
        rg_status si = settle_insert(ctx);
        if (si != RG_OK) return si;
    }
    CK(cudaMemcpyAsync(ctx->hctr, ctx->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    check_fingerprint(ctx);
    if (ctx->k3_speculated) {
        ctx->k3_speculated = false;
        if (deferred && ctx->hctr->stopped) {
            // a warp ran out of budget (the table must grow): K2/K3 ran on an
            // incomplete table; finish K1 and run them again
            s = k1_finish(ctx);
            if (s != RG_OK) return s;
            return prune_agglomerate_fused(ctx, window_fix);
        }
        if (ctx->hctr->max_col > sorted_bucket_max_column()) {
            // a column too long for the bucketed sort (its blocks skipped the
            // oversized buckets): again, with the sizing read choosing the path
            if (deferred) {
                ctx->used = ctx->hctr->used;
                ctx->ingested = ctx->hctr->ingested;
                ctx->skipped = ctx->hctr->skipped;
                ctx->k1.active = false;
            }
            ctx->k3_no_spec = true;
            s = prune_agglomerate_fused(ctx, window_fix);
            ctx->k3_no_spec = false;
            return s;
        }
    }
    if (deferred) {  // K1's counters arrive with K3's
        ctx->used = ctx->hctr->used;
        ctx->ingested = ctx->hctr->ingested;
        ctx->skipped = ctx->hctr->skipped;
        ctx->k1.active = false;
    }
    resolve_contract_timer(ctx);
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ctx->ev_k2, ctx->ev_k3);
    cudaEventElapsedTime(&b, ctx->ev_k3, ctx->ev_end);
    ctx->ms_prune += a;
    ctx->ms_agg += b;
    ctx->n_sig = ctx->hctr->n_sig;
    ctx->n_roots = ctx->hctr->n_roots;
    ctx->n_kept = ctx->hctr->n_kept;
    ctx->table_dirty = true;
    ctx->res = ctx->grid;
    ctx->res_is_canvas = true;
    ctx->sorted = bound != 0;
    ctx->state = rg_ctx::kAgg;
    return RG_OK;
}

static rg_status reset_impl(rg_ctx* ctx) {
    ctx->state = rg_ctx::kAccum;
    ctx->table_dirty = true;
    rg_status s = reopen_accumulator(ctx);
    if (s != RG_OK) return s;
    ctx->ingested = ctx->skipped = 0;
    ctx->ms_contract = ctx->ms_prune = ctx->ms_agg = ctx->ms_label = 0;
    return push_counters(ctx);
}

rg_status rg_reset(rg_ctx* ctx) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    DevGuard guard(ctx->device);
    return reset_impl(ctx);
}

rg_status rg_cluster(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                     rg_stats* stats) {
    return rg_cluster_ex(ctx, xy, n, kind, 0u, stats);
}

rg_status rg_cluster_ex(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                        uint32_t flags, rg_stats* stats) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (flags & ~(uint32_t)RG_CLUSTER_WINDOW_FIX)
        return set_err(ctx, RG_ERR_ARG, "unknown rg_cluster_ex flags 0x%x", flags);
    if (n && !xy) return set_err(ctx, RG_ERR_ARG, "null point buffer");
    DevGuard guard(ctx->device);
    // cluster_sequential builds a fresh accumulator (pipeline.hpp:98).
    rg_status s = reset_impl(ctx);
    if (s != RG_OK) return s;
    const bool sorted_k3 = use_sorted_k3(ctx);
    // with the sorted K3 the K1 stop check rides on K3's host read
    const bool wf_req = (flags & RG_CLUSTER_WINDOW_FIX) != 0;
    ctx->allow_pairs_k2 = sorted_k3 && !wf_req && kind == RG_MEM_DEVICE;
    s = ingest_any(ctx, xy, n, kind, sorted_k3 && n < 0x7fffffffull);
    ctx->allow_pairs_k2 = false;
    if (s != RG_OK) return s;
    u64 peak = ctx->used;
    const bool wf = (flags & RG_CLUSTER_WINDOW_FIX) != 0;
    if (sorted_k3) {
        const bool deferred = ctx->k1.active;
        s = prune_agglomerate_fused(ctx, wf);
        if (s != RG_OK) return s;
        if (deferred) peak = ctx->used;
    } else {
        s = prune_impl(ctx, wf);
        if (s != RG_OK) return s;
        s = agglomerate_impl(ctx);
        if (s != RG_OK) return s;
    }
    ctx->used = peak;  // peak_accumulator_entries pipeline.hpp:100
    if (stats) return rg_get_stats(ctx, stats);
    return RG_OK;
}

rg_status rg_prune_agglomerate(rg_ctx* ctx, uint32_t flags, rg_stats* stats) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx) {
        const rg_status ss = settle_stream(ctx);
        if (ss != RG_OK) return ss;
    }
    if (flags & ~(uint32_t)RG_CLUSTER_WINDOW_FIX)
        return set_err(ctx, RG_ERR_ARG, "unknown rg_prune_agglomerate flags 0x%x", flags);
    DevGuard guard(ctx->device);
    rg_status s = RG_OK;
    const u64 peak = ctx->used;
    const bool wf = (flags & RG_CLUSTER_WINDOW_FIX) != 0;
    if (ctx->state == rg_ctx::kAccum && use_sorted_k3(ctx)) {
        s = prune_agglomerate_fused(ctx, wf);
    } else {
        s = prune_impl(ctx, wf);
        if (s == RG_OK) s = agglomerate_impl(ctx);
    }
    if (s != RG_OK) return s;
    ctx->used = peak;
    if (stats) return rg_get_stats(ctx, stats);
    return RG_OK;
}

rg_status rg_get_significant(rg_ctx* ctx, int64_t* tx, int64_t* ty, uint64_t* count,
                             int64_t* cluster_id, uint64_t cap, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx->state == rg_ctx::kAccum)
        return set_err(ctx, RG_ERR_STATE, "no significant tiles: call rg_prune first");
    DevGuard guard(ctx->device);
    const u64 n = ctx->n_sig;
    const u64 w = std::min<u64>(cap, n);
    if (w == 0) return RG_OK;
    const int bits = (int)(ctx->res.bits_x + ctx->res.bits_y);
    u64* ks = nullptr;
    u32 *iota = nullptr, *order = nullptr;
    void* temp = nullptr;
    if (ctx->state == rg_ctx::kAgg && ctx->sorted) {
        order = ctx->root_idx_sorted;  // K3 already sorted the keys
    } else {
        CK(dalloc(&ks, n));
        CK(dalloc(&iota, n));
        CK(dalloc(&order, n));
        const size_t tb = sort_pairs_temp_bytes(n, bits);
        CK(cudaMalloc(&temp, tb));
        CK(launch_iota(iota, n, ctx->n_sm, ctx->st));
        CK(sort_pairs(temp, tb, ctx->sig_key, ks, iota, order, n, bits, ctx->st));
        ctx->launches += 6;
    }
    long long *dtx = (long long*)tx, *dty = (long long*)ty, *dcid = (long long*)cluster_id;
    u64* dcnt = (u64*)count;
    if (kind == RG_MEM_HOST) {
        dtx = dty = dcid = nullptr;
        dcnt = nullptr;
        if (tx) CK(salloc(&dtx, w, ctx->st));
        if (ty) CK(salloc(&dty, w, ctx->st));
        if (count) CK(salloc(&dcnt, w, ctx->st));
        if (cluster_id) CK(salloc(&dcid, w, ctx->st));
    }
    if (ctx->state == rg_ctx::kAgg && ctx->sorted) {
        k_gather_sorted_keys<<<grid_for(w, ctx->n_sm), 256, 0, ctx->st>>>(
            ctx->root_key_sorted, ctx->root_idx_sorted, ctx->sig_cnt, ctx->s_cid, w, ctx->res, dtx,
            dty, dcnt, dcid);
        CK(cudaGetLastError());
    } else {
        CK(launch_gather_sorted(order, ctx->sig_key, ctx->sig_cnt,
                                ctx->state == rg_ctx::kAgg ? ctx->tile_cid : nullptr, w, ctx->res,
                                dtx, dty, dcnt, dcid, ctx->n_sm, ctx->st));
    }
    ++ctx->launches;
    if (kind == RG_MEM_HOST) {
        if (tx) CK(cudaMemcpyAsync(tx, dtx, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (ty) CK(cudaMemcpyAsync(ty, dty, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (count) CK(cudaMemcpyAsync(count, dcnt, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (cluster_id) CK(cudaMemcpyAsync(cluster_id, dcid, w * 8, cudaMemcpyDeviceToHost, ctx->st));
    }
    if (kind == RG_MEM_HOST) {
        sfree(dtx, ctx->st);
        sfree(dty, ctx->st);
        sfree(dcnt, ctx->st);
        sfree(dcid, ctx->st);
    }
    CK(cudaStreamSynchronize(ctx->st));
    if (temp) cudaFree(temp);
    dfree(ks);
    dfree(iota);
    if (!(ctx->state == rg_ctx::kAgg && ctx->sorted)) dfree(order);
    return RG_OK;
}

rg_status rg_get_clusters(rg_ctx* ctx, uint64_t* n_tiles, uint64_t* n_points, int64_t* first_tx,
                          int64_t* first_ty, uint64_t cap, rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (ctx->state != rg_ctx::kAgg)
        return set_err(ctx, RG_ERR_STATE, "no clusters: call rg_agglomerate first");
    DevGuard guard(ctx->device);
    const u64 w = std::min<u64>(cap, ctx->n_kept);
    if (w == 0) return RG_OK;
    u64 *dnt = (u64*)n_tiles, *dnp = (u64*)n_points;
    long long *dfx = (long long*)first_tx, *dfy = (long long*)first_ty;
    if (kind == RG_MEM_HOST) {
        dnt = dnp = nullptr;
        dfx = dfy = nullptr;
        if (n_tiles) CK(dalloc(&dnt, w));
        if (n_points) CK(dalloc(&dnp, w));
        if (first_tx) CK(dalloc(&dfx, w));
        if (first_ty) CK(dalloc(&dfy, w));
    }
    if (n_points && ctx->sorted && ctx->npts_pending) {
        CK(launch_cluster_npts(ctx->s_cid, ctx->root_idx_sorted, ctx->sig_cnt, ctx->n_sig,
                               ctx->s_clu_root, ctx->n_kept, ctx->npts, ctx->n_sm, ctx->st));
        ++ctx->launches;
        ctx->npts_pending = false;
    }
    k_cluster_facts<<<grid_for(w, ctx->n_sm), 256, 0, ctx->st>>>(
        ctx->root_key_sorted, ctx->root_idx_sorted, ctx->sorted ? ctx->s_clu_root : nullptr, w,
        ctx->size, ctx->npts, ctx->res, dnt, dnp, dfx, dfy);
    ++ctx->launches;
    CK(cudaGetLastError());
    if (kind == RG_MEM_HOST) {
        if (n_tiles) CK(cudaMemcpyAsync(n_tiles, dnt, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (n_points) CK(cudaMemcpyAsync(n_points, dnp, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (first_tx) CK(cudaMemcpyAsync(first_tx, dfx, w * 8, cudaMemcpyDeviceToHost, ctx->st));
        if (first_ty) CK(cudaMemcpyAsync(first_ty, dfy, w * 8, cudaMemcpyDeviceToHost, ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    if (kind == RG_MEM_HOST) {
        dfree(dnt);
        dfree(dnp);
        dfree(dfx);
        dfree(dfy);
    }
    return RG_OK;
}

rg_status rg_device_result(rg_ctx* ctx, rg_device_view* out) {
    if (!ctx || !out) return RG_ERR_ARG;
    if (ctx->state == rg_ctx::kAccum)
        return set_err(ctx, RG_ERR_STATE, "no significant tiles: call rg_prune first");
    out->key = (const uint64_t*)ctx->sig_key;
    out->count = (const uint64_t*)ctx->sig_cnt;
    if (ctx->state == rg_ctx::kAgg) {
        DevGuard guard(ctx->device);
        rg_status s = ensure_tile_cid(ctx);
        if (s != RG_OK) return s;
        CK(cudaStreamSynchronize(ctx->st));
    }
    out->cluster_id = ctx->state == rg_ctx::kAgg ? ctx->tile_cid : nullptr;
    out->n_significant = ctx->n_sig;
    out->n_clusters = ctx->n_kept;
    out->origin_x = ctx->res.origin_x;
    out->origin_y = ctx->res.origin_y;
    out->key_bits_y = ctx->res.bits_y;
    out->reserved = 0;
    return RG_OK;
}

void rg_decode_key(const rg_device_view* v, uint64_t key, int64_t* tx, int64_t* ty) {
    if (tx) *tx = v->origin_x + (int64_t)(key >> v->key_bits_y);
    if (ty) *ty = v->origin_y + (int64_t)(key & ((1ull << v->key_bits_y) - 1));
}

rg_status rg_label_points(rg_ctx* ctx, const double* xy, uint64_t n, int32_t* labels,
                          rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (n && (!xy || !labels)) return set_err(ctx, RG_ERR_ARG, "null buffer");
    if (ctx->state != rg_ctx::kAgg)
        return set_err(ctx, RG_ERR_STATE, "labelling requires rg_agglomerate first");
    if (!ctx->res_is_canvas)
        return set_err(ctx, RG_ERR_UNSUPPORTED,
                       "labelling points needs significant tiles on the canvas");
    if (n == 0) return RG_OK;
    DevGuard guard(ctx->device);
    PhaseTimer timer(ctx, &ctx->ms_label);
    if (!ctx->slots) {
        // no table (empty significant set): every label is -1
        if (kind == RG_MEM_DEVICE) {
            CK(cudaMemsetAsync(labels, 0xff, n * sizeof(int32_t), ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
        } else {
            std::memset(labels, 0xff, n * sizeof(int32_t));
        }
        return RG_OK;
    }
    static const bool k4_table = [] {  // RG_K4=table: always the count-table lookups (A/B)
        const char* v = std::getenv("RG_K4");
        return v && std::strcmp(v, "table") == 0;
    }();
    if (kind == RG_MEM_DEVICE && ctx->sorted && ((uintptr_t)xy & 15) == 0 && ctx->narrow &&
        !k4_table && n >= (1ull << 22) && buffer_unordered(ctx, xy, n)) {
        // K4': no spatial order, so labels come from a cell table of the
        // kept tiles (L2-sized) instead of the count table
        const u32 kb = ctx->res.bits_x + ctx->res.bits_y;
        if (kb <= 37 && ctx->res.bits_y >= 3 && ctx->n_kept < 0x7ffffff0ull) {
            if (!ctx->lk_valid) {
                if (ctx->lk_ids_cap < ctx->n_sig) {
                    dfree(ctx->lk_ids);
                    ctx->lk_ids_cap = 0;
                    CK(dalloc(&ctx->lk_ids, std::max<u64>(ctx->n_sig, 1024)));
                    ctx->lk_ids_cap = std::max<u64>(ctx->n_sig, 1024);
                }
                u64 cells = std::max<u64>(1024, ctx->n_sig / 4);  // grown below if more
                u64* dctr = ctx->scratch + 4;
                for (int attempt = 0;; ++attempt) {
                    const u64 nb = cell_buckets(cells);
                    if (ctx->lk_cap < nb) {
                        dfree(ctx->lk_tab);
                        ctx->lk_cap = 0;
                        CK(dalloc(&ctx->lk_tab, 2 * nb));
                        ctx->lk_cap = nb;
                    }
                    ctx->lk_nb = nb;
                    CK(launch_cells_build(ctx->root_key_sorted, ctx->s_cid, &ctx->ctr->n_sig,
                                          ctx->n_sig, ctx->lk_tab, nb, ctx->res.bits_y, dctr,
                                          ctx->n_sm, ctx->st));
                    ++ctx->launches;
                    u64 h[2];
                    CK(cudaMemcpyAsync(h, dctr, sizeof h, cudaMemcpyDeviceToHost, ctx->st));
                    CK(cudaStreamSynchronize(ctx->st));
                    if (!(u32)h[1]) break;
                    if (attempt > 8) return set_err(ctx, RG_ERR_CUDA, "cell table did not fit");
                    cells = std::max<u64>(cells * 2, h[0] * 2);  // every cell counted fits now
                }
                CK(launch_cells_mixed(ctx->root_key_sorted, ctx->s_cid, &ctx->ctr->n_sig,
                                      ctx->n_sig, ctx->lk_tab, ctx->lk_nb, ctx->res.bits_y,
                                      ctx->scratch + 4, ctx->lk_ids, ctx->n_sm, ctx->st));
                ctx->launches += 2;
                ctx->lk_valid = true;
            }
            CK(launch_label_cells(xy, n, ctx->grid, ctx->lk_tab, ctx->lk_nb, ctx->lk_ids, labels,
                                  ctx->n_sm, ctx->st));
            ++ctx->launches;
            CK(cudaStreamSynchronize(ctx->st));
            return RG_OK;
        }
    }
    {
        rg_status ms = mark_table(ctx, true);
        if (ms == RG_OK && !ctx->table_cids) ms = ensure_tile_cid(ctx);
        if (ms != RG_OK) return ms;
    }
    if (kind == RG_MEM_DEVICE) {
        CK(launch_label_points(xy, n, ctx->grid, table_of(ctx), ctx->tile_cid, ctx->table_cids,
                               labels, ctx->narrow, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaStreamSynchronize(ctx->st));
        return RG_OK;
    }
    rg_status s = ensure_stage(ctx, n, true);
    if (s != RG_OK) return s;
    const u64 ch = ctx->stage_pts;
    for (u64 off = 0; off < n; off += ch) {
        const int b = (int)((off / ch) & 1);
        const u64 len = std::min(ch, n - off);
        CK(cudaMemcpyAsync(ctx->stage[b], xy + 2 * off, len * 16, cudaMemcpyHostToDevice,
                           ctx->st));
        CK(launch_label_points(ctx->stage[b], len, ctx->grid, table_of(ctx), ctx->tile_cid,
                               ctx->table_cids, ctx->lstage[b], ctx->narrow, ctx->n_sm, ctx->st));
        ++ctx->launches;
        CK(cudaMemcpyAsync(labels + off, ctx->lstage[b], len * 4, cudaMemcpyDeviceToHost,
                           ctx->st));
    }
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

rg_status rg_cluster_points(rg_ctx* ctx, const double* xy, uint64_t n, rg_memkind kind,
                            uint64_t* n_points, uint64_t* n_clusters) {
    if (!ctx) return RG_ERR_ARG;
    if (n && !xy) return set_err(ctx, RG_ERR_ARG, "null point buffer");
    if (ctx->state != rg_ctx::kAgg)
        return set_err(ctx, RG_ERR_STATE, "cluster points require rg_agglomerate first");
    if (!ctx->res_is_canvas)
        return set_err(ctx, RG_ERR_UNSUPPORTED,
                       "cluster points need significant tiles on the canvas");
    if (n >= 0xffffffffull)
        return set_err(ctx, RG_ERR_UNSUPPORTED, "cluster points: at most 2^32-2 points per call");
    DevGuard guard(ctx->device);
    PhaseTimer timer(ctx, &ctx->ms_label);
    ctx->cp_valid = false;
    const u64 C = ctx->n_kept;
    dfree(ctx->cp_xy);
    dfree(ctx->cp_off);
    ctx->cp_xy = nullptr;
    ctx->cp_n = 0;
    CK(dalloc(&ctx->cp_off, C + 1));
    CK(cudaMemsetAsync(ctx->cp_off, 0, (C + 1) * sizeof(u64), ctx->st));
    ctx->cp_c = C;
    if (n == 0 || C == 0) {
        CK(cudaStreamSynchronize(ctx->st));
        ctx->cp_valid = true;
        if (n_points) *n_points = 0;
        if (n_clusters) *n_clusters = C;
        return RG_OK;
    }
    // every buffer below is released on every path out of this block
    struct Tmp {
        double* xy = nullptr;
        int* lab = nullptr;
        u32 *ia = nullptr, *ib = nullptr;
        u64 *ka = nullptr, *kb = nullptr;
        void* temp = nullptr;
        ~Tmp() {
            dfree(xy);
            dfree(lab);
            dfree(ia);
            dfree(ib);
            dfree(ka);
            dfree(kb);
            if (temp) cudaFree(temp);
        }
    } T;
    const double* dxy = xy;
    if (kind == RG_MEM_HOST) {
        CK(dalloc(&T.xy, 2 * n));
        CK(cudaMemcpyAsync(T.xy, xy, n * 16, cudaMemcpyHostToDevice, ctx->st));
        dxy = T.xy;
    }
    CK(dalloc(&T.lab, n));
    {
        rg_status ms = mark_table(ctx, true);
        if (ms == RG_OK && !ctx->table_cids) ms = ensure_tile_cid(ctx);
        if (ms != RG_OK) return ms;
    }
    CK(launch_label_points(dxy, n, ctx->grid, table_of(ctx), ctx->tile_cid, ctx->table_cids, T.lab,
                           ctx->narrow, ctx->n_sm, ctx->st));
    ++ctx->launches;
    if (((uintptr_t)dxy & 15) == 0) {
        // v2: counting sort by cluster, then a shared-memory sort per cluster
        struct Tmp2 {
            u64 *cnt = nullptr, *off = nullptr;
            double* grp = nullptr;
            u32 *flag = nullptr, *pos = nullptr;
            void* temp = nullptr;
            ~Tmp2() {
                dfree(cnt);
                dfree(off);
                dfree(grp);
                dfree(flag);
                dfree(pos);
                if (temp) cudaFree(temp);
            }
        } V;
        PointsV2 P2;
        CK(dalloc(&V.cnt, C + 1));
        CK(dalloc(&V.off, C + 1));
        P2.temp_bytes = cluster_points_v2_temp_bytes(n, C);
        CK(cudaMalloc(&V.temp, P2.temp_bytes));
        P2.xy = dxy;
        P2.labels = T.lab;
        P2.n = n;
        P2.n_clusters = C;
        P2.dedupe = ctx->p.dedupe_points ? 1 : 0;
        P2.cnt = V.cnt;
        P2.off = V.off;
        P2.scratch = ctx->scratch;
        P2.temp = V.temp;
        P2.n_sm = ctx->n_sm;
        u64 m = 0, mx = 0;
        CK(launch_cluster_points_v2_count(P2, ctx->st, &m, &mx));
        ctx->launches += 4;
        if (mx <= cluster_points_v2_cap()) {
            CK(dalloc(&ctx->cp_xy, 2 * std::max<u64>(m, 1)));
            if (P2.dedupe) {
                CK(dalloc(&V.grp, 2 * std::max<u64>(m, 1)));
                CK(dalloc(&V.flag, std::max<u64>(m, 1)));
                CK(dalloc(&V.pos, std::max<u64>(m, 1)));
                P2.grp = (double2*)V.grp;
                P2.out = (double2*)ctx->cp_xy;
            } else {
                P2.grp = (double2*)ctx->cp_xy;  // grouped and sorted in place: the output
                P2.out = nullptr;
            }
            P2.flag = V.flag;
            P2.pos = V.pos;
            P2.out_off = ctx->cp_off;
            CK(launch_cluster_points_v2(P2, m, ctx->st));
            ctx->launches += P2.dedupe ? 5 : 2;
            if (!P2.dedupe)
                CK(cudaMemcpyAsync(ctx->cp_off, V.off, (C + 1) * sizeof(u64),
                                   cudaMemcpyDeviceToDevice, ctx->st));
            CK(cudaMemcpyAsync(&ctx->hctr->pad0[1], ctx->cp_off + C, sizeof(u64),
                               cudaMemcpyDeviceToHost, ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            ctx->cp_n = ctx->hctr->pad0[1];
            ctx->cp_valid = true;
            if (n_points) *n_points = ctx->cp_n;
            if (n_clusters) *n_clusters = C;
            return RG_OK;
        }
        // a cluster larger than one block's shared memory: the radix path below
    }
    CK(dalloc(&T.ia, n));
    CK(dalloc(&T.ib, n));
    CK(dalloc(&T.ka, n + 1));
    CK(dalloc(&T.kb, n + 1));
    CK(dalloc(&ctx->cp_xy, 2 * n));
    PointsLaunch L;
    L.xy = dxy;
    L.labels = T.lab;
    L.n = n;
    L.n_clusters = C;
    L.dedupe = ctx->p.dedupe_points ? 1 : 0;
    L.idx_a = T.ia;
    L.idx_b = T.ib;
    L.key_a = T.ka;
    L.key_b = T.kb;
    L.m_dev = ctx->scratch;
    L.m_host = &ctx->hctr->pad0[0];
    L.temp_bytes = cluster_points_temp_bytes(n);
    CK(cudaMalloc(&T.temp, L.temp_bytes));
    L.temp = T.temp;
    L.out_xy = ctx->cp_xy;
    L.offsets = ctx->cp_off;
    L.n_sm = ctx->n_sm;
    CK(launch_cluster_points(L, ctx->st));
    ctx->launches += 9;
    CK(cudaMemcpyAsync(&ctx->hctr->pad0[1], ctx->cp_off + C, sizeof(u64), cudaMemcpyDeviceToHost,
                       ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    ctx->cp_n = ctx->hctr->pad0[1];
    ctx->cp_valid = true;
    if (n_points) *n_points = ctx->cp_n;
    if (n_clusters) *n_clusters = C;
    return RG_OK;
}

rg_status rg_get_cluster_points(rg_ctx* ctx, double* xy, uint64_t cap, uint64_t* offsets,
                                rg_memkind kind) {
    if (!ctx) return RG_ERR_ARG;
    if (!ctx->cp_valid) return set_err(ctx, RG_ERR_STATE, "call rg_cluster_points first");
    DevGuard guard(ctx->device);
    const cudaMemcpyKind mk =
        kind == RG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const u64 w = std::min<u64>(cap, ctx->cp_n);
    if (xy && w) CK(cudaMemcpyAsync(xy, ctx->cp_xy, w * 16, mk, ctx->st));
    if (offsets) CK(cudaMemcpyAsync(offsets, ctx->cp_off, (ctx->cp_c + 1) * 8, mk, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return RG_OK;
}

uint64_t rg_kernel_launches(const rg_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
