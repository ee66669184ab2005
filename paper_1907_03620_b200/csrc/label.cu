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

constexpr int kLWarps = 8;
constexpr int kLBatch = 2;
constexpr int kLCache = 128;
constexpr u64 kLRowsPerSeg = 64;

struct LRows {
    double x[kLBatch], y[kLBatch];
};

template <bool kAligned>
__device__ __forceinline__ void l_load(const double* xy, u64 p0, u32 left, int lane, u64 pol,
                                       LRows& o) {
    if (kAligned && left == 32 * kLBatch) {
        const double2* base = reinterpret_cast<const double2*>(xy) + p0 + lane;
#pragma unroll
        for (int b = 0; b < kLBatch; ++b) {
            const double2 v = ld_point_stream(base + b * 32, pol);
            o.x[b] = v.x;
            o.y[b] = v.y;
        }
        return;
    }
#pragma unroll
    for (int b = 0; b < kLBatch; ++b) {
        if ((u32)(b * 32 + lane) < left) {
            if (kAligned) {
                const double2 v =
                    ld_point_stream(reinterpret_cast<const double2*>(xy) + p0 + b * 32 + lane, pol);
                o.x[b] = v.x;
                o.y[b] = v.y;
            } else {
                const double* q = xy + 2 * (p0 + b * 32 + lane);
                o.x[b] = q[0];
                o.y[b] = q[1];
            }
        } else {
            o.x[b] = o.y[b] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
}

struct LSmem {
    u64 ckey[kLCache];
    int ccid[kLCache];
    unsigned char owner[kLCache];
};

__device__ __forceinline__ u32 l_slot(u64 key, u32 bits_y) {
    return (((u32)(key >> bits_y) & 7u) << 4) | ((u32)key & 15u);
}

template <bool kNarrow>
__device__ __forceinline__ u64 l_key(const Grid& g, double x, double y) {
    if (kNarrow) {
        const int tx = __double2int_rd(__dmul_rn(x, g.scale));
        const int ty = __double2int_rd(__dmul_rn(y, g.scale));
        return ((u64)(u32)(tx - (int)g.origin_x) << g.bits_y) | (u32)(ty - (int)g.origin_y);
    }
    return pack_key(g, x, y);
}

template <bool kNarrow>
__device__ __forceinline__ void l_batch(const Grid& g, const Table& t, const int* tile_cid,
                                        const LRows& cur, u64 p0, u32 left, LSmem& w, int lane,
                                        u32 lane_bit, int* labels) {
#pragma unroll
    for (int b = 0; b < kLBatch; ++b) {
        const bool inb = in_bounds(g, cur.x[b], cur.y[b]);
        const u64 kk = l_key<kNarrow>(g, cur.x[b], cur.y[b]);
        const u64 key = inb ? kk : kEmpty;
        const u32 peers = __match_any_sync(kFull, key);
        const int leader_lane = __ffs(peers) - 1;
        const bool leader = inb && ((peers & (0u - peers)) == lane_bit);
        const u32 cs = l_slot(key, g.bits_y);
        int cid = -1;
        bool miss = false;
        if (leader) {
            if (w.ckey[cs] == key)
                cid = w.ccid[cs];
            else
                miss = true;
        }
        if (__any_sync(kFull, miss)) {
            if (miss) {
                const u64 v = table_find(t, key);
                cid = (v != kEmpty && (v & kSigBit)) ? tile_cid[v & ~kSigBit] : -1;
                w.owner[cs] = (unsigned char)lane;
            }
            __syncwarp();
            if (miss && w.owner[cs] == lane) {
                w.ckey[cs] = key;
                w.ccid[cs] = cid;
            }
        }
        __syncwarp();
        cid = __shfl_sync(kFull, cid, leader_lane);
        if ((u32)(b * 32 + lane) < left) labels[p0 + b * 32 + lane] = inb ? cid : -1;
    }
}

template <bool kAligned, bool kNarrow>
__global__ void __launch_bounds__(kLWarps * 32) k_label_points(const double* xy, u64 n, Grid g,
                                                               Table t, const int* tile_cid,
                                                               int* labels) {
    __shared__ LSmem s_warp[kLWarps];
    const int lane = threadIdx.x & 31;
    const u32 lane_bit = 1u << lane;
    LSmem& w = s_warp[threadIdx.x >> 5];
    for (int i = lane; i < kLCache; i += 32) w.ckey[i] = kEmpty;
    __syncwarp();
    const u64 pol = evict_first_policy();
    const u64 n_rows = (n + 31) / 32;
    const u64 n_seg = (n_rows + kLRowsPerSeg - 1) / kLRowsPerSeg;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 seg = warp; seg < n_seg; seg += n_warps) {
        const u64 p_end = min((seg + 1) * kLRowsPerSeg * 32, n);
        u64 p0 = seg * kLRowsPerSeg * 32;
        u32 left = (u32)min(p_end - p0, (u64)(32 * kLBatch));
        LRows ra, rb;
        l_load<kAligned>(xy, p0, left, lane, pol, ra);
        while (true) {
            u64 pn = p0 + 32 * kLBatch;
            u32 left_n = pn < p_end ? (u32)min(p_end - pn, (u64)(32 * kLBatch)) : 0u;
            if (left_n) l_load<kAligned>(xy, pn, left_n, lane, pol, rb);
            l_batch<kNarrow>(g, t, tile_cid, ra, p0, left, w, lane, lane_bit, labels);
            if (!left_n) break;
            p0 = pn;
            left = left_n;
            pn = p0 + 32 * kLBatch;
            left_n = pn < p_end ? (u32)min(p_end - pn, (u64)(32 * kLBatch)) : 0u;
            if (left_n) l_load<kAligned>(xy, pn, left_n, lane, pol, ra);
            l_batch<kNarrow>(g, t, tile_cid, rb, p0, left, w, lane, lane_bit, labels);
            if (!left_n) break;
            p0 = pn;
            left = left_n;
        }
    }
}

static int g_label_blocks_per_sm = 0;

cudaError_t launch_label_points(const double* xy, u64 n, Grid g, Table t, const int* tile_cid,
                                int* labels, bool narrow, int n_sm, cudaStream_t st) {
    if (!g_label_blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_label_blocks_per_sm,
                                                      k_label_points<true, false>, kLWarps * 32, 0);
        if (g_label_blocks_per_sm < 1) g_label_blocks_per_sm = 1;
    }
    const u64 rows = (n + 31) / 32;
    const u64 segs = (rows + kLRowsPerSeg - 1) / kLRowsPerSeg;
    u64 blocks = (segs + kLWarps - 1) / kLWarps;
    const u64 cap = (u64)n_sm * g_label_blocks_per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    const bool aligned = ((uintptr_t)xy & 15) == 0;
    if (aligned && narrow)
        k_label_points<true, true><<<(int)blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else if (aligned)
        k_label_points<true, false><<<(int)blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else if (narrow)
        k_label_points<false, true><<<(int)blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    else
        k_label_points<false, false><<<(int)blocks, kLWarps * 32, 0, st>>>(xy, n, g, t, tile_cid, labels);
    return cudaGetLastError();
}

}  // namespace rg
