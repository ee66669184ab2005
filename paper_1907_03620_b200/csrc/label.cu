// label.cu — K4: per-point cluster labels (point-retaining variant), sm_100a.
//
// RASTER' keeps every in-bounds point with its tile (accumulator.hpp:131) and
// hands a kept tile's points to its cluster (agglomerate.hpp:70-76, 183);
// labeled_points (metrics.hpp:78-83) flattens that into (point, cluster id).
// The device form is the same information in input order: one int32 per
// point = cluster id of its tile, -1 for out-of-bounds points and for points
// of tiles that are not significant or whose component was dropped.
//
// One streaming pass with the same structure as K1: each warp walks
// contiguous segments (so consecutive rows come from the same clusters),
// coalesced 16-byte point loads double-buffered across batches, one
// projection per point, __match_any_sync so one lane per distinct tile does
// the lookup, and a per-warp direct-mapped shared-memory cache of
// tile -> cluster id so only the first occurrence of a tile probes the HBM
// table (whose value word holds SIG_BIT|index after K2). Labels are stored
// coalesced.
#include "common.cuh"
#include "internal.h"

namespace rg {

constexpr int kLWarps = 4;
constexpr int kLBatch = 2;
constexpr int kLRing = 4;     // rows in flight per warp (cp.async ring)
constexpr int kLCache = 128;
constexpr u32 kLRowsPerSeg = 256;

struct LSmem {
    u64 ckey[kLCache];  // cache keys (KeyOps) -> cluster id
    int ccid[kLCache];
    unsigned char owner[kLCache];
};

// One row: every lane looks its tile up in the per-warp cache (direct-mapped
// by position in an 8 x 16-tile window, as in K1); lanes that miss probe the
// table themselves (equal keys in a row probe the same lines) and one lane
// per slot installs the result.
template <bool kNarrow, bool kCid>
__device__ __forceinline__ int l_row(const Grid& g, const Table& t, const int* tile_cid, double x,
                                     double y, LSmem& w, int lane) {
    using K = KeyOps<kNarrow>;
    const u64 key = K::cache_key(g, x, y);
    const bool valid = key != kEmpty;
    const u32 cs = K::slot(key, g.bits_y);
    const bool hit = valid && w.ckey[cs] == key;
    int cid = hit ? w.ccid[cs] : -1;
    const bool miss = valid && !hit;
    if (ballot(miss)) {
        if (miss) {
            const u64 v = table_find(t, K::table_key(key, g.bits_y));
            if (kCid)
                cid = (v != kEmpty && (v & kSigBit)) ? (int)(u32)v - 1 : -1;
            else
                cid = (v != kEmpty && (v & kSigBit)) ? tile_cid[v & ~kSigBit] : -1;
            w.owner[cs] = (unsigned char)lane;
        }
        __syncwarp();
        if (miss && w.owner[cs] == lane) {
            w.ckey[cs] = key;
            w.ccid[cs] = cid;
        }
        __syncwarp();
    }
    return cid;
}

// Segments of kLRowsPerSeg rows are dealt to warps round-robin; each warp
// streams its rows through a per-lane cp.async ring like K1.
template <bool kAligned, bool kNarrow, bool kCid>
__global__ void __launch_bounds__(kLWarps * 32, 8) k_label_points(const double* xy, u64 n, Grid g,
                                                                  Table t, const int* tile_cid,
                                                                  int* labels) {
    __shared__ LSmem s_warp[kLWarps];
    __shared__ __align__(16) double2 s_ring[kLWarps][kLRing][32];
    const int lane = threadIdx.x & 31;
    LSmem& w = s_warp[threadIdx.x >> 5];
    double2 (*ring)[32] = s_ring[threadIdx.x >> 5];
    for (int i = lane; i < kLCache; i += 32) w.ckey[i] = kEmpty;
    __syncwarp();
    const u64 pol = evict_first_policy();
    const u64 n_rows = (n + 31) / 32;
    const u64 n_seg = (n_rows + kLRowsPerSeg - 1) / kLRowsPerSeg;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 seg = warp; seg < n_seg; seg += n_warps) {
        const u64 p0 = seg * kLRowsPerSeg * 32;
        const u32 valid = (u32)min(n - p0, (u64)kLRowsPerSeg * 32);
        const u32 nr = (valid + 31) / 32;
        const double2* base = reinterpret_cast<const double2*>(xy) + p0 + lane;
        const double* xb = xy + 2 * p0;
        int* lab = labels + p0 + lane;
        auto issue = [&](u32 row) {
            if (row < nr) {
                const u32 idx = row * 32 + lane;
                if (idx < valid) {
                    double2* dst = &ring[row % kLRing][lane];
                    if (kAligned) {
                        cp_async16(dst, base + row * 32, pol);
                    } else {
                        dst->x = xb[2 * (u64)idx];
                        dst->y = xb[2 * (u64)idx + 1];
                    }
                }
            }
            cp_async_commit();
        };
#pragma unroll
        for (int k = 0; k < kLRing; ++k) issue(k);
        for (u32 j = 0; j < nr; j += kLBatch) {
            cp_async_wait<kLRing - kLBatch>();
            double x[kLBatch], y[kLBatch];
#pragma unroll
            for (int b = 0; b < kLBatch; ++b) {
                const u32 row = j + b;
                if (row * 32 + lane < valid) {
                    const double2 v = ring[row % kLRing][lane];
                    x[b] = v.x;
                    y[b] = v.y;
                } else {
                    x[b] = y[b] = __longlong_as_double(0x7ff8000000000000ll);
                }
            }
#pragma unroll
            for (int b = 0; b < kLBatch; ++b) issue(j + kLRing + b);
#pragma unroll
            for (int b = 0; b < kLBatch; ++b) {
                const int cid = l_row<kNarrow, kCid>(g, t, tile_cid, x[b], y[b], w, lane);
                if ((j + b) * 32 + lane < valid) lab[(j + b) * 32] = cid;
            }
        }
        cp_async_wait<0>();
    }
}

static int g_label_blocks_per_sm = 0;

template <bool kCid>
static void label_dispatch(const double* xy, u64 n, Grid g, Table t, const int* tile_cid,
                           int* labels, bool narrow, int blocks, cudaStream_t st) {
    const bool aligned = ((uintptr_t)xy & 15) == 0;
    if (aligned && narrow)
        k_label_points<true, true, kCid><<<blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else if (aligned)
        k_label_points<true, false, kCid><<<blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else if (narrow)
        k_label_points<false, true, kCid><<<blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else
        k_label_points<false, false, kCid><<<blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
}

cudaError_t launch_label_points(const double* xy, u64 n, Grid g, Table t, const int* tile_cid,
                                bool table_cids, int* labels, bool narrow, int n_sm,
                                cudaStream_t st) {
    if (!g_label_blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_label_blocks_per_sm,
                                                      k_label_points<true, false, false>,
                                                      kLWarps * 32, 0);
        if (g_label_blocks_per_sm < 1) g_label_blocks_per_sm = 1;
    }
    const u64 rows = (n + 31) / 32;
    const u64 segs = (rows + kLRowsPerSeg - 1) / kLRowsPerSeg;
    u64 blocks = (segs + kLWarps - 1) / kLWarps;
    const u64 cap = (u64)n_sm * g_label_blocks_per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    if (table_cids)
        label_dispatch<true>(xy, n, g, t, tile_cid, labels, narrow, (int)blocks, st);
    else
        label_dispatch<false>(xy, n, g, t, tile_cid, labels, narrow, (int)blocks, st);
    return cudaGetLastError();
}

}  // namespace rg
