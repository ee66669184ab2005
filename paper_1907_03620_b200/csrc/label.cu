// label.cu — K4: per-point cluster labels (point-retaining variant), sm_100a.
//
// RASTER' keeps every in-bounds point with its tile (accumulator.hpp:131) and
// hands a kept tile's points to its cluster (agglomerate.hpp:70-76, 183);
// labeled_points (metrics.hpp:78-83) flattens that into (point, cluster id).
// The device form is the same information in input order: one int32 per
// point = cluster id of its tile, -1 for out-of-bounds points and for points
// of tiles that are not significant or whose component was dropped.
//
// One streaming pass: coalesced 16-byte point loads (evict-first), one
// projection, one hash probe (the table's value word holds SIG_BIT|index
// after K2) and one gather of the tile's id; the int32 store is coalesced.
// Within a row the warp deduplicates keys with __match_any_sync so only one
// lane per distinct tile probes the table.
#include "common.cuh"
#include "internal.h"

namespace rg {

constexpr int kLBatch = 4;

template <bool kAligned>
__global__ void __launch_bounds__(256) k_label_points(const double* xy, u64 n, Grid g, Table t,
                                                       const int* tile_cid, int* labels) {
    const int lane = threadIdx.x & 31;
    const u64 n_rows = (n + 31) / 32;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    const u64 pol = evict_first_policy();
    for (u64 r = warp * kLBatch; r < n_rows; r += n_warps * kLBatch) {
        double xs[kLBatch], ys[kLBatch];
#pragma unroll
        for (int b = 0; b < kLBatch; ++b) {
            const u64 idx = (r + b) * 32 + lane;
            if (idx < n) {
                if (kAligned) {
                    const double2 v = ld_point_stream(reinterpret_cast<const double2*>(xy) + idx, pol);
                    xs[b] = v.x;
                    ys[b] = v.y;
                } else {
                    xs[b] = xy[2 * idx];
                    ys[b] = xy[2 * idx + 1];
                }
            } else {
                xs[b] = ys[b] = __longlong_as_double(0x7ff8000000000000ll);
            }
        }
#pragma unroll
        for (int b = 0; b < kLBatch; ++b) {
            const u64 idx = (r + b) * 32 + lane;
            const bool inb = in_bounds(g, xs[b], ys[b]);
            const u64 key = inb ? pack_key(g, xs[b], ys[b]) : kEmpty;
            const u32 peers = __match_any_sync(kFull, key);
            const int leader = __ffs(peers) - 1;
            int cid = -1;
            if (inb && lane == leader) {
                const u64 v = table_find(t, key);
                if (v != kEmpty && (v & kSigBit)) cid = tile_cid[v & ~kSigBit];
            }
            cid = __shfl_sync(kFull, cid, leader);
            if (idx < n) labels[idx] = inb ? cid : -1;
        }
    }
}

cudaError_t launch_label_points(const double* xy, u64 n, Grid g, Table t, const int* tile_cid,
                                int* labels, int n_sm, cudaStream_t st) {
    const u64 rows = (n + 31) / 32;
    const u64 warps_needed = (rows + kLBatch - 1) / kLBatch;
    u64 blocks = (warps_needed + 7) / 8;
    const u64 cap = (u64)n_sm * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    if (((uintptr_t)xy & 15) == 0)
        k_label_points<true><<<(int)blocks, 256, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else
        k_label_points<false><<<(int)blocks, 256, 0, st>>>(xy, n, g, t, tile_cid, labels);
    return cudaGetLastError();
}

}  // namespace rg
