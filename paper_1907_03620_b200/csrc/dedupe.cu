// dedupe.cu — dedupe_points for the point-retaining mode on the device.
//
// The reference keeps every point per tile and, at prune, reduces each
// tile's points to unique coordinates; the threshold then applies to the
// deduplicated count (TileAccumulator::prune accumulator.hpp:160-174,
// dedupe :199-204; window_fix agglomerate.hpp:238-241 reports the same
// deduplicated count). count_of / for_each_count keep reporting raw counts
// (:179, :188-191), and window_fix decides on raw counts (:225).
//
// Device form, without storing per-tile point lists:
//   * a point set (16-B slots {x bits, y bits}, open addressing) holds every
//     distinct in-bounds point seen so far; -0.0 is stored as +0.0 so that
//     points equal under operator== (core.hpp:17) share a slot;
//   * a second tile table ("unique counts") gets +1 for the tile of every
//     point that was new to the set.
// At prune the raw count word of every occupied tile is replaced by its
// unique count before K2, so the threshold, the reported counts and the
// clusters follow the deduplicated counts. The set insert is a single
// 128-bit CAS per probe (no torn reads: the CAS returns the slot atomically).
#include "common.cuh"
#include "internal.h"

namespace rg {

__device__ __forceinline__ u64 mix64(u64 v) {
    v ^= v >> 30;
    v *= 0xbf58476d1ce4e5b9ull;
    v ^= v >> 27;
    v *= 0x94d049bb133111ebull;
    return v ^ (v >> 31);
}

// true when (xb, yb) was not in the set before this call
__device__ __forceinline__ bool ps_insert(const PointSet& ps, u64 xb, u64 yb) {
    PtKey want;
    want.x = xb;
    want.y = yb;
    PtKey empty;
    empty.x = kEmpty;
    empty.y = kEmpty;
    u64 i = mix64(xb ^ mix64(yb)) & ps.mask;
    while (true) {
        const PtKey old = atomicCAS(ps.slots + i, empty, want);
        if (old.x == kEmpty && old.y == kEmpty) return true;
        if (old.x == xb && old.y == yb) return false;
        i = (i + 1) & ps.mask;
    }
}

__device__ __forceinline__ u64 canon_bits(double v) {
    return (u64)__double_as_longlong(v + 0.0);  // -0.0 + 0.0 = +0.0
}

__global__ void k_dedupe_ingest(const double* xy, u64 n, Grid g, PointSet ps, Table ut,
                                u64* n_new) {
    u64 mine = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (!in_bounds(g, x, y)) continue;
        if (ps_insert(ps, canon_bits(x), canon_bits(y))) {
            table_add(ut, pack_key(g, x, y), 1);
            ++mine;
        }
    }
    if (mine) atomicAdd(n_new, mine);
}

// Merge: every point of src new to dst adds to dst's unique counts.
__global__ void k_ps_fold(const PtKey* src, u64 src_cap, Grid g, PointSet dst, Table ut,
                          u64* n_new) {
    u64 mine = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < src_cap;
         i += (u64)gridDim.x * blockDim.x) {
        const PtKey k = src[i];
        if (k.x == kEmpty && k.y == kEmpty) continue;
        if (ps_insert(dst, k.x, k.y)) {
            table_add(ut, pack_key(g, __longlong_as_double((long long)k.x),
                                   __longlong_as_double((long long)k.y)), 1);
            ++mine;
        }
    }
    if (mine) atomicAdd(n_new, mine);
}

__global__ void k_ps_rehash(const PtKey* src, u64 src_cap, PointSet dst) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < src_cap;
         i += (u64)gridDim.x * blockDim.x) {
        const PtKey k = src[i];
        if (k.x == kEmpty && k.y == kEmpty) continue;
        ps_insert(dst, k.x, k.y);
    }
}

// Raw count word -> unique count, for every occupied tile (before K2).
__global__ void k_dedupe_counts(Table t, u64 cap, Table ut) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < cap;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 k = t.slots[i].key;
        if (k == kEmpty) continue;
        const u64 u = table_find(ut, k);
        t.slots[i].count = u == kEmpty ? 0 : u;
    }
}

static int grid_of(u64 n, int n_sm) {
    const u64 want = (n + 255) / 256;
    const u64 cap = (u64)n_sm * 16;
    return (int)(want == 0 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_dedupe_ingest(const double* xy, u64 n, Grid g, PointSet ps, Table ut,
                                 u64* n_new, int n_sm, cudaStream_t st) {
    k_dedupe_ingest<<<grid_of(n, n_sm), 256, 0, st>>>(xy, n, g, ps, ut, n_new);
    return cudaGetLastError();
}

cudaError_t launch_ps_fold(const PtKey* src, u64 src_cap, Grid g, PointSet dst, Table ut,
                           u64* n_new, int n_sm, cudaStream_t st) {
    k_ps_fold<<<grid_of(src_cap, n_sm), 256, 0, st>>>(src, src_cap, g, dst, ut, n_new);
    return cudaGetLastError();
}

cudaError_t launch_ps_rehash(const PtKey* src, u64 src_cap, PointSet dst, int n_sm,
                             cudaStream_t st) {
    k_ps_rehash<<<grid_of(src_cap, n_sm), 256, 0, st>>>(src, src_cap, dst);
    return cudaGetLastError();
}

cudaError_t launch_dedupe_counts(Table t, u64 cap, Table ut, int n_sm, cudaStream_t st) {
    k_dedupe_counts<<<grid_of(cap, n_sm), 256, 0, st>>>(t, cap, ut);
    return cudaGetLastError();
}

}  // namespace rg
