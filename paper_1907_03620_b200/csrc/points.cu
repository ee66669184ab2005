// points.cu — RASTER' output on the device: the in-bounds points of every
// kept cluster, grouped by cluster id and ordered by point_less inside a
// cluster (Mode::retain_points: take_points agglomerate.hpp:70-76, the point
// sort of finalize_clusters :183, point_less core.hpp:22-24), optionally
// deduplicated (TileAccumulator::dedupe accumulator.hpp:199-204).
//
// Pipeline over the M labelled points (label >= 0 from K4):
//   1. select  — indices of labelled points (warp-aggregated append; the
//                order is irrelevant, the sort below is total);
//   2. three stable LSD radix passes (CUB onesweep) over (label, x, y):
//      y bits, then x bits, then the label's ceil(log2 C) bits — the
//      composite order is label, then x, then y, i.e. point_less per cluster;
//   3. gather  — the sorted points (16 B each) and, with dedupe, a flag per
//                point that differs from its predecessor, compacted in order;
//   4. offsets — cluster k occupies [off[k], off[k+1]).
// Doubles are sorted through an order-preserving u64 image; x + 0.0 maps
// -0.0 to +0.0 first so that points equal under operator== (core.hpp:17)
// get equal keys.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.h"

namespace rg {

__device__ __forceinline__ u64 ord_key(double d) {
    const u64 b = (u64)__double_as_longlong(d + 0.0);
    return (b >> 63) ? ~b : (b | (1ull << 63));
}

__global__ void k_select_labelled(const int* labels, u64 n, u32* idx, u64* m) {
    const int lane = threadIdx.x & 31;
    for (u64 base = (blockIdx.x * (u64)blockDim.x + threadIdx.x) - lane; base < n;
         base += (u64)gridDim.x * blockDim.x) {
        const u64 i = base + lane;
        const bool keep = i < n && labels[i] >= 0;
        const u32 bal = __ballot_sync(kFull, keep);
        if (!bal) continue;
        u64 at = 0;
        if (lane == 0) at = atomicAdd(m, (u64)__popc(bal));
        at = __shfl_sync(kFull, at, 0);
        if (keep) idx[at + __popc(bal & ((1u << lane) - 1))] = (u32)i;
    }
}

// which: 0 = y, 1 = x
__global__ void k_coord_keys(const double* xy, const u32* idx, u64 m, int which, u64* key) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m;
         i += (u64)gridDim.x * blockDim.x)
        key[i] = ord_key(xy[2 * (u64)idx[i] + (which ? 0 : 1)]);
}

__global__ void k_label_keys(const int* labels, const u32* idx, u64 m, u32* key) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m;
         i += (u64)gridDim.x * blockDim.x)
        key[i] = (u32)labels[idx[i]];
}

// flag[i] = 1 unless point i equals point i-1 of the same cluster (dedupe).
__global__ void k_dup_flags(const double* xy, const u32* idx, const u32* lab, u64 m, int dedupe,
                            u32* flag) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m;
         i += (u64)gridDim.x * blockDim.x) {
        u32 f = 1;
        if (dedupe && i > 0 && lab[i] == lab[i - 1]) {
            const u64 a = idx[i], b = idx[i - 1];
            f = !(xy[2 * a] == xy[2 * b] && xy[2 * a + 1] == xy[2 * b + 1]);
        }
        flag[i] = f;
    }
}

// pos = exclusive scan of flag; writes kept points and, at every cluster
// boundary, the offsets of the clusters between the previous label and this
// one (clusters with no points get empty ranges).
__global__ void k_emit_points(const double* xy, const u32* idx, const u32* lab, const u32* flag,
                              const u32* pos, u64 m, u64 n_clusters, double* out, u64* off) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i <= m;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 p = i < m ? pos[i] : (m ? pos[m - 1] + flag[m - 1] : 0);
        if (i < m && flag[i]) {
            const u64 a = idx[i];
            out[2 * p] = xy[2 * a];  // 8-byte aligned inputs are allowed
            out[2 * p + 1] = xy[2 * a + 1];
        }
        const u64 lo = i == 0 ? 0 : (u64)lab[i - 1] + 1;
        const u64 hi = i == m ? n_clusters : (u64)lab[i];
        for (u64 c = lo; c <= hi && c <= n_clusters; ++c) off[c] = p;
    }
}

static int grid_of(u64 n, int n_sm) {
    const u64 want = (n + 255) / 256;
    const u64 cap = (u64)n_sm * 8;
    return (int)(want == 0 ? 1 : (want < cap ? want : cap));
}

static int bits_for_count(u64 c) {
    int b = 1;
    while (b < 32 && (1ull << b) < c) ++b;
    return b;
}

size_t cluster_points_temp_bytes(u64 m) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs((void*)nullptr, a, (const u64*)nullptr, (u64*)nullptr,
                                    (const u32*)nullptr, (u32*)nullptr, (int)m);
    cub::DeviceRadixSort::SortPairs((void*)nullptr, b, (const u32*)nullptr, (u32*)nullptr,
                                    (const u32*)nullptr, (u32*)nullptr, (int)m);
    cub::DeviceScan::ExclusiveSum((void*)nullptr, c, (const u32*)nullptr, (u32*)nullptr, (int)m);
    return std::max(a, std::max(b, c));
}

cudaError_t launch_cluster_points(const PointsLaunch& L, cudaStream_t st) {
    cudaError_t e;
    const int gs = grid_of(L.n, L.n_sm);
    if ((e = cudaMemsetAsync(L.m_dev, 0, sizeof(u64), st)) != cudaSuccess) return e;
    k_select_labelled<<<gs, 256, 0, st>>>(L.labels, L.n, L.idx_a, L.m_dev);
    if ((e = cudaMemcpyAsync(L.m_host, L.m_dev, sizeof(u64), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const u64 m = *L.m_host;
    const int gm = grid_of(m + 1, L.n_sm);
    if (m > 1) {
        size_t tb = L.temp_bytes;
        // y, then x (stable), then label (stable): point_less within clusters
        k_coord_keys<<<gm, 256, 0, st>>>(L.xy, L.idx_a, m, 0, L.key_a);
        if ((e = cub::DeviceRadixSort::SortPairs(L.temp, tb, L.key_a, L.key_b, L.idx_a, L.idx_b,
                                                 (int)m, 0, 64, st)) != cudaSuccess)
            return e;
        k_coord_keys<<<gm, 256, 0, st>>>(L.xy, L.idx_b, m, 1, L.key_a);
        tb = L.temp_bytes;
        if ((e = cub::DeviceRadixSort::SortPairs(L.temp, tb, L.key_a, L.key_b, L.idx_b, L.idx_a,
                                                 (int)m, 0, 64, st)) != cudaSuccess)
            return e;
    }
    u32* lab_a = reinterpret_cast<u32*>(L.key_a);
    u32* lab_b = reinterpret_cast<u32*>(L.key_b);
    k_label_keys<<<gm, 256, 0, st>>>(L.labels, L.idx_a, m, lab_a);
    const u32* idx = L.idx_a;
    const u32* lab = lab_a;
    if (m > 1) {
        size_t tb = L.temp_bytes;
        if ((e = cub::DeviceRadixSort::SortPairs(L.temp, tb, lab_a, lab_b, L.idx_a, L.idx_b,
                                                 (int)m, 0, bits_for_count(L.n_clusters),
                                                 st)) != cudaSuccess)
            return e;
        idx = L.idx_b;
        lab = lab_b;
    }
    // key_a/key_b hold n + 1 u64 words: their upper halves are free now
    u32* flag = reinterpret_cast<u32*>(L.key_a) + (m + 1);
    u32* pos = reinterpret_cast<u32*>(L.key_b) + (m + 1);
    k_dup_flags<<<gm, 256, 0, st>>>(L.xy, idx, lab, m, L.dedupe, flag);
    if (m) {
        size_t tb = L.temp_bytes;
        if ((e = cub::DeviceScan::ExclusiveSum(L.temp, tb, flag, pos, (int)m, st)) != cudaSuccess)
            return e;
    }
    k_emit_points<<<gm, 256, 0, st>>>(L.xy, idx, lab, flag, pos, m, L.n_clusters, L.out_xy,
                                      L.offsets);
    return cudaGetLastError();
}

}  // namespace rg
