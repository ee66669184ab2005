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

// ---------------------------------------------------------------------------
// v2 (default): group by cluster with a counting sort, then sort each
// cluster's points in shared memory. The labelled points of a cluster are
// few (config 4: about 500), so the per-cluster sort replaces the three
// 64-bit radix passes over all M points; clusters larger than kCpCap take
// the v1 path above.
//   hist     — points per cluster (runs of equal labels pre-summed per warp);
//   scan     — cluster starts off[c];
//   scatter  — points into their cluster's range (order inside arbitrary);
//   sort     — one block per cluster: bitonic sort of (x, y) order keys in
//              shared memory, written back in place (the signs of zeros
//              travel with the point); with dedupe, a flag per point that
//              differs from its predecessor;
//   (dedupe) — scan of the flags, emit, per-cluster offsets.
// ---------------------------------------------------------------------------
constexpr u32 kCpCap = 4096;
constexpr int kCpThreads = 256;
constexpr size_t kCpSmem = kCpCap * (8 + 8 + 1);

// Per-warp runs of equal labels: returns, for the run head, the run length
// (0 for other lanes) and every lane's rank inside its run.
__device__ __forceinline__ u32 label_runs(int lab, int lane, u32* rank) {
    const int prev = __shfl_up_sync(kFull, lab, 1);
    const bool head = lane == 0 || prev != lab;
    const u32 heads = __ballot_sync(kFull, head);
    const u32 le = heads & (0xffffffffu >> (31 - lane));
    const int hl = 31 - __clz(le);  // this lane's run head
    *rank = (u32)(lane - hl);
    const u32 after = heads & ~(0xffffffffu >> (31 - lane));  // heads above this lane
    const int next = after ? __ffs(after) - 1 : 32;
    return head ? (u32)(next - lane) : 0u;
}

__global__ void k_cp_hist(const int* labels, u64 n, u64* cnt) {
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const int lab = i < n ? labels[i] : -1;
        u32 rank;
        const u32 len = label_runs(lab, lane, &rank);
        if (len && lab >= 0) atomicAdd(cnt + lab, (u64)len);
    }
}

__global__ void k_cp_max(const u64* off, u64 C, u64* mx) {
    u64 m = 0;
    for (u64 c = blockIdx.x * (u64)blockDim.x + threadIdx.x; c < C;
         c += (u64)gridDim.x * blockDim.x)
        m = max(m, off[c + 1] - off[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

__global__ void k_cp_scatter(const double2* xy, const int* labels, u64 n, u64* cursor,
                             double2* grp) {
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const int lab = i < n ? labels[i] : -1;
        u32 rank;
        const u32 len = label_runs(lab, lane, &rank);
        u64 base = 0;
        if (len && lab >= 0) base = atomicAdd(cursor + lab, (u64)len);
        const int hl = lane - (int)rank;
        base = __shfl_sync(kFull, base, hl);
        if (lab >= 0) grp[base + rank] = xy[i];
    }
}

__device__ __forceinline__ double from_ord(u64 k, bool neg_zero) {
    const u64 b = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
    const double d = __longlong_as_double((long long)b);
    return neg_zero ? -0.0 : d;
}

// one block per cluster (persistent); flag (dedupe) may be null
__global__ void __launch_bounds__(kCpThreads) k_cp_sort(double2* grp, const u64* off, u64 C,
                                                        u32* flag) {
    extern __shared__ u64 sh_cp[];  // kCpSmem bytes
    u64* kx = sh_cp;
    u64* ky = sh_cp + kCpCap;
    unsigned char* zs = (unsigned char*)(ky + kCpCap);  // bit 0: x was -0.0, bit 1: y -0.0
    for (u64 c = blockIdx.x; c < C; c += gridDim.x) {
        const u64 lo = off[c];
        const u32 len = (u32)(off[c + 1] - lo);
        if (len > kCpCap) continue;  // the host sends such inputs down the v1 path
        u32 P = 2;
        while (P < len) P <<= 1;
        for (u32 i = threadIdx.x; i < P; i += kCpThreads) {
            if (i < len) {
                const double2 v = grp[lo + i];
                kx[i] = ord_key(v.x);
                ky[i] = ord_key(v.y);
                zs[i] = (unsigned char)((v.x == 0.0 && signbit(v.x) ? 1 : 0) |
                                        (v.y == 0.0 && signbit(v.y) ? 2 : 0));
            } else {
                kx[i] = ky[i] = ~0ull;
                zs[i] = 0;
            }
        }
        __syncthreads();
        // bitonic network; compare-exchange c of a stage pairs
        // i = c + (c & ~(j - 1)) with i + j, so every thread works
        for (u32 k = 2; k <= P; k <<= 1) {
            for (u32 j = k >> 1; j > 0; j >>= 1) {
                for (u32 c = threadIdx.x; c < P / 2; c += kCpThreads) {
                    const u32 i = c + (c & ~(j - 1)), l = i + j;
                    const bool asc = (i & k) == 0;
                    const u64 ax = kx[i], ay = ky[i], bx = kx[l], by = ky[l];
                    const bool a_gt = ax > bx || (ax == bx && ay > by);
                    if (a_gt == asc && (ax != bx || ay != by)) {
                        kx[i] = bx;
                        ky[i] = by;
                        kx[l] = ax;
                        ky[l] = ay;
                        const unsigned char t = zs[i];
                        zs[i] = zs[l];
                        zs[l] = t;
                    }
                }
                __syncthreads();
            }
        }
        for (u32 i = threadIdx.x; i < len; i += kCpThreads) {
            grp[lo + i] = make_double2(from_ord(kx[i], zs[i] & 1), from_ord(ky[i], zs[i] & 2));
            if (flag) flag[lo + i] = i == 0 || kx[i] != kx[i - 1] || ky[i] != ky[i - 1];
        }
        __syncthreads();
    }
}

// dedupe: kept points compacted; cluster c starts at pos[off[c]]
__global__ void k_cp_emit(const double2* grp, const u32* flag, const u32* pos, u64 m,
                          const u64* off, u64 C, double2* out, u64* out_off) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m;
         i += (u64)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = grp[i];
    for (u64 c = blockIdx.x * (u64)blockDim.x + threadIdx.x; c <= C;
         c += (u64)gridDim.x * blockDim.x)
        out_off[c] = off[c] < m ? pos[off[c]] : (m ? pos[m - 1] + flag[m - 1] : 0);
}

size_t cluster_points_v2_temp_bytes(u64 n, u64 C) {
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum((void*)nullptr, a, (const u64*)nullptr, (u64*)nullptr,
                                  (int)(C + 1));
    cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const u32*)nullptr, (u32*)nullptr, (int)n);
    return std::max(a, b);
}

// Phase 1 (host synchronises): counts, offsets, M and the largest cluster.
cudaError_t launch_cluster_points_v2_count(const PointsV2& L, cudaStream_t st, u64* m_host,
                                           u64* max_host) {
    cudaError_t e;
    const int gs = grid_of(L.n, L.n_sm);
    if ((e = cudaMemsetAsync(L.cnt, 0, (L.n_clusters + 1) * sizeof(u64), st)) != cudaSuccess)
        return e;
    k_cp_hist<<<gs, 256, 0, st>>>(L.labels, L.n, L.cnt);
    size_t tb = L.temp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(L.temp, tb, L.cnt, L.off, (int)(L.n_clusters + 1),
                                           st)) != cudaSuccess)
        return e;
    if ((e = cudaMemsetAsync(L.scratch, 0, sizeof(u64), st)) != cudaSuccess) return e;
    k_cp_max<<<grid_of(L.n_clusters, L.n_sm), 256, 0, st>>>(L.off, L.n_clusters, L.scratch);
    if ((e = cudaMemcpyAsync(m_host, L.off + L.n_clusters, sizeof(u64), cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
        return e;
    if ((e = cudaMemcpyAsync(max_host, L.scratch, sizeof(u64), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    return cudaStreamSynchronize(st);
}

u32 cluster_points_v2_cap() { return kCpCap; }

// Phase 2: scatter, per-cluster sort, (dedupe) compaction. Without dedupe
// the grouped array is the output (grp == out) and off the offsets.
cudaError_t launch_cluster_points_v2(const PointsV2& L, u64 m, cudaStream_t st) {
    cudaError_t e;
    if ((e = cudaMemcpyAsync(L.cnt, L.off, (L.n_clusters + 1) * sizeof(u64),
                             cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return e;
    const int gs = grid_of(L.n, L.n_sm);
    k_cp_scatter<<<gs, 256, 0, st>>>(reinterpret_cast<const double2*>(L.xy), L.labels, L.n, L.cnt,
                                     L.grp);
    const int gc = (int)std::min<u64>(L.n_clusters, (u64)L.n_sm * 4);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cp_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCpSmem);
        attr = true;
    }
    if (gc)
        k_cp_sort<<<gc, kCpThreads, kCpSmem, st>>>(L.grp, L.off, L.n_clusters,
                                                   L.dedupe ? L.flag : nullptr);
    if (L.dedupe && m) {
        size_t tb = L.temp_bytes;
        if ((e = cub::DeviceScan::ExclusiveSum(L.temp, tb, L.flag, L.pos, (int)m, st)) !=
            cudaSuccess)
            return e;
        k_cp_emit<<<grid_of(std::max<u64>(m, L.n_clusters + 1), L.n_sm), 256, 0, st>>>(
            L.grp, L.flag, L.pos, m, L.off, L.n_clusters, L.out, L.out_off);
    }
    return cudaGetLastError();
}

}  // namespace rg
