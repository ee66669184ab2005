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
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace rg {

constexpr int kLWarps = 4;
constexpr int kLBatch = 2;
#ifndef RG_K4_RING
#define RG_K4_RING 4
#endif
#ifndef RG_K4_MINBLOCKS
#define RG_K4_MINBLOCKS 12  // (config 4 labels: 8 blocks/SM 2.00 ms, 10: 2.00, 12: 1.96, 14 and 16: 2.10)
#endif
constexpr int kLRing = RG_K4_RING;     // rows in flight per warp (cp.async ring)
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
__global__ void __launch_bounds__(kLWarps * 32, RG_K4_MINBLOCKS) k_label_points(const double* xy, u64 n, Grid g,
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

// ------------------------------------------- K4' (inputs without order)
// With no spatial order every point misses the per-warp cache and probes
// the HBM count table: a random sector of a table far larger than L2. Here
// the labels come from a CELL table of the kept tiles, dense enough to stay
// in L2 while the points stream past evict-first. A cell is 8 x 8 tiles;
// its 16-byte entry holds the cell id, the cluster id of its kept tiles and
// a 64-bit mask of which of its tiles are kept. A cell whose kept tiles
// belong to several clusters (rare) points into a per-tile id array instead
// (ids in mask order). Entries sit two to a 32-byte bucket; a point reads
// its cell's home bucket (rarely the next), tests one mask bit, done.
//   w0 = (cell id + 1) | info << 32, info = cluster id + 1, or kMixed | base
//   w1 = kept-tile mask (bit = (kx & 7) * 8 + (ky & 7))
constexpr u32 kMixed = 0x80000000u;
constexpr int kCellBits = 3;

__device__ __forceinline__ u64 cell_bucket(u32 cell, u64 nb) {
    u64 h = (u64)cell * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
    return __umul64hi(h, nb);
}
__device__ __forceinline__ u32 cell_of(u64 key, u32 bits_y) {
    const u64 kx = key >> bits_y, ky = key & ((1ull << bits_y) - 1);
    return (u32)(((kx >> kCellBits) << (bits_y - kCellBits)) | (ky >> kCellBits));
}
__device__ __forceinline__ u32 cell_bit(u64 key, u32 bits_y) {
    return (u32)(((key >> bits_y) & 7) * 8 + (key & 7));
}

// Pass 1: insert every kept tile's cell and mask bit (cell ids are unique per
// table, inserted with one CAS); a cell meeting a second cluster id is
// flagged mixed. *n_cells counts cells; *over flags a table that filled up.
__global__ void k_cells_build(const u64* skey, const int* cid, const u64* n_p, ulonglong2* tab,
                              u64 nb, u32 bits_y, u64 cap_cells, u64* n_cells, u32* over) {
    __shared__ u32 s_new;
    if (threadIdx.x == 0) s_new = 0;
    __syncthreads();
    const u64 n = *n_p;
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;  // whole warps: the aggregation below is warp-wide
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const int c = i < n ? cid[i] : -1;
        const u64 key = c >= 0 ? skey[i] : 0;
        const u32 cell = cell_of(key, bits_y);
        // tiles of one column and cell are consecutive in sorted order: one
        // lane per (cell, cluster) group inserts the group's mask bits
        const u64 tag = c >= 0 ? ((u64)cell << 32) | (u32)c : ~0ull;
        const u32 peers = __match_any_sync(kFull, tag);
        const u64 mine = c >= 0 ? 1ull << cell_bit(key, bits_y) : 0;
        const u64 bits = (u64)__reduce_or_sync(peers, (u32)mine) |
                         ((u64)__reduce_or_sync(peers, (u32)(mine >> 32)) << 32);
        bool fresh = false;
        if (c >= 0 && lane == __ffs(peers) - 1) {
        const u64 want = (u64)(cell + 1) | ((u64)(u32)(c + 1) << 32);
        u64 b = cell_bucket(cell, nb);
        ulonglong2* e = nullptr;
        for (u64 probes = 0; probes < nb && !e; ++probes) {
#pragma unroll 1
            for (int j = 0; j < 2; ++j) {
                ulonglong2* q = tab + 2 * b + j;
                u64 w0 = atomicCAS(&q->x, 0ull, want);
                if (w0 == 0) {  // new cell
                    fresh = true;
                    e = q;
                    break;
                }
                if ((u32)w0 == cell + 1) {
                    if ((u32)(w0 >> 32) != (u32)(c + 1) && !((w0 >> 32) & kMixed))
                        atomicOr(&q->x, (u64)kMixed << 32);
                    e = q;
                    break;
                }
            }
            b = b + 1 == nb ? 0 : b + 1;
        }
        if (e)
            atomicOr(&e->y, bits);
        else
            *over = 1;
        }
        // new cells counted per block (one global counter would serialise)
        const u32 nf = __popc(__ballot_sync(kFull, fresh));
        if (lane == 0 && nf) atomicAdd(&s_new, nf);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_new && atomicAdd(n_cells, (u64)s_new) + s_new > cap_cells) *over = 1;
}

// Pass 2: mixed cells get a base in the per-tile id array.
__global__ void k_cells_mixed_base(ulonglong2* tab, u64 n_entries, u64* next) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_entries;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 w0 = tab[i].x;
        if (!w0 || !((w0 >> 32) & kMixed)) continue;
        const u64 base = atomicAdd(next, (u64)__popcll(tab[i].y));
        tab[i].x = (w0 & 0xffffffffull) | ((u64)(kMixed | (u32)base) << 32);
    }
}

__device__ __forceinline__ const ulonglong2* cell_find(const ulonglong2* tab, u64 nb, u32 cell,
                                                       u64 pol);

// Pass 3: kept tiles of mixed cells write their id at base + rank in mask.
__global__ void k_cells_mixed_ids(const u64* skey, const int* cid, const u64* n_p,
                                  const ulonglong2* tab, u64 nb, u32 bits_y, int* ids) {
    const u64 n = *n_p;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const int c = cid[i];
        if (c < 0) continue;
        const u64 key = skey[i];
        const ulonglong2* e = cell_find(tab, nb, cell_of(key, bits_y), 0);
        const u32 info = (u32)(e->x >> 32);
        if (!(info & kMixed)) continue;
        const u32 bit = cell_bit(key, bits_y);
        ids[(info & ~kMixed) + __popcll(e->y & ((1ull << bit) - 1))] = c;
    }
}

__device__ __forceinline__ void ld_entry(const ulonglong2* p, u64 pol, u64& a, u64& b) {
    asm volatile("ld.global.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
                 : "=l"(a), "=l"(b)
                 : "l"(p), "l"(pol));
}

// Both entries of a 32-byte bucket with ONE 256-bit load (sm_100): a warp's
// 32 lookups go to 32 different sectors, and the load/store unit handles one
// sector per cycle, so two 16-byte loads per bucket cost twice the cycles
// (k_label_cells was bound by the LSU data pipe, 71 % of its peak).
__device__ __forceinline__ void ld_bucket(const ulonglong2* p, u64 pol, u64& a0, u64& m0, u64& a1,
                                          u64& m1) {
    asm volatile("ld.global.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(a0), "=l"(m0), "=l"(a1), "=l"(m1)
                 : "l"(p), "l"(pol));
}

// Cell entry or nullptr (build-time lookups use pol = 0: no hint needed).
__device__ __forceinline__ const ulonglong2* cell_find(const ulonglong2* tab, u64 nb, u32 cell,
                                                       u64) {
    u64 b = cell_bucket(cell, nb);
    while (true) {
        bool open = false;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const u64 w0 = tab[2 * b + j].x;
            if ((u32)w0 == cell + 1) return tab + 2 * b + j;
            open |= w0 == 0;
        }
        if (open) return nullptr;
        b = b + 1 == nb ? 0 : b + 1;
    }
}

__device__ __forceinline__ void st_label_stream(int* p, int v) {
    asm volatile("st.global.cs.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Resolves a cell entry pair for one point: 1 = found (label in c), 0 = the
// search must go on, -1 = an empty entry ends it (no kept tile).
__device__ __forceinline__ int cell_try(u64 a0, u64 m0, u64 a1, u64 m1, u32 cell, u32 bit,
                                        const int* ids, int& c) {
    u64 w = 0, m = 0;
    if ((u32)a0 == cell + 1) {
        w = a0;
        m = m0;
    } else if ((u32)a1 == cell + 1) {
        w = a1;
        m = m1;
    }
    if (w) {
        if ((m >> bit) & 1) {
            const u32 info = (u32)(w >> 32);
            c = (info & kMixed) ? __ldg(ids + (info & ~kMixed) + __popcll(m & ((1ull << bit) - 1)))
                                : (int)info - 1;
        }
        return 1;
    }
    return (!a0 || !a1) ? -1 : 0;
}

// Lookups of kLkIlp points per thread and trip: the point loads are in
// flight together; each lookup reads one 32-byte bucket (2 entries) and walks
// on only when a full bucket does not hold the cell. (One point per trip is
// fastest: the kernel is bound by random L2 sectors, and more points per
// thread only delay the lookups behind the point loads.)
#ifndef RG_K4P_ILP
#define RG_K4P_ILP 1  // (config 4 random-order labels: 1 point per thread and trip 4.44 ms, 2: 4.62, 4: 4.71, 8: 6.01)
#endif
constexpr int kLkIlp = RG_K4P_ILP;
__global__ void __launch_bounds__(256) k_label_cells(const double2* xy, u64 n, Grid g,
                                                     const ulonglong2* tab, u64 nb,
                                                     const int* ids, int* labels) {
    const u64 pol_pts = evict_first_policy();
    u64 pol_tab;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_tab));
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 base = blockIdx.x * (u64)blockDim.x + threadIdx.x; base < n;
         base += stride * kLkIlp) {
        u64 key[kLkIlp];
        bool ok[kLkIlp];
#pragma unroll
        for (int j = 0; j < kLkIlp; ++j) {
            const u64 i = base + (u64)j * stride;
            ok[j] = false;
            key[j] = 0;
            if (i < n) {
                const double2 v = ld_point_stream(xy + i, pol_pts);
                key[j] = pack_key(g, v.x, v.y);
                ok[j] = in_bounds(g, v.x, v.y);
            }
        }
#pragma unroll
        for (int j = 0; j < kLkIlp; ++j) {
            const u64 i = base + (u64)j * stride;
            if (i >= n) continue;
            int c = -1;
            if (ok[j]) {
                const u32 cell = cell_of(key[j], g.bits_y), bit = cell_bit(key[j], g.bits_y);
                u64 b = cell_bucket(cell, nb);
                while (true) {
                    u64 a0, m0, a1, m1;
#ifdef RG_K4P_LD128
                    ld_entry(tab + 2 * b, pol_tab, a0, m0);
                    ld_entry(tab + 2 * b + 1, pol_tab, a1, m1);
#else
                    ld_bucket(tab + 2 * b, pol_tab, a0, m0, a1, m1);
#endif
                    if (cell_try(a0, m0, a1, m1, cell, bit, ids, c)) break;
                    b = b + 1 == nb ? 0 : b + 1;
                }
            }
            st_label_stream(labels + i, c);
        }
    }
}

u64 cell_buckets(u64 cells) { return std::max<u64>(16, (u64)((double)cells / (2 * 0.6)) + 1); }

cudaError_t launch_cells_build(const u64* skey, const int* cid, const u64* n_dev, u64 n_bound,
                               ulonglong2* tab, u64 nb, u32 bits_y, u64* counters, int n_sm,
                               cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(tab, 0, nb * 32, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(counters, 0, 3 * sizeof(u64), st);
    if (e != cudaSuccess) return e;
    const u64 want = (n_bound + 255) / 256;
    const int blocks = (int)std::max<u64>(1, std::min<u64>(want, (u64)n_sm * 8));
    // counters: [0] cells, [1] overflow flag, [2] mixed-id cursor
    k_cells_build<<<blocks, 256, 0, st>>>(skey, cid, n_dev, tab, nb, bits_y,
                                          (u64)((double)nb * 2 * 0.85), counters,
                                          (u32*)(counters + 1));
    return cudaGetLastError();
}

cudaError_t launch_cells_mixed(const u64* skey, const int* cid, const u64* n_dev, u64 n_bound,
                               ulonglong2* tab, u64 nb, u32 bits_y, u64* counters, int* ids,
                               int n_sm, cudaStream_t st) {
    const u64 we = (nb * 2 + 255) / 256;
    k_cells_mixed_base<<<(int)std::max<u64>(1, std::min<u64>(we, (u64)n_sm * 8)), 256, 0, st>>>(
        tab, nb * 2, counters + 2);
    const u64 want = (n_bound + 255) / 256;
    k_cells_mixed_ids<<<(int)std::max<u64>(1, std::min<u64>(want, (u64)n_sm * 8)), 256, 0, st>>>(
        skey, cid, n_dev, tab, nb, bits_y, ids);
    return cudaGetLastError();
}

cudaError_t launch_label_cells(const double* xy, u64 n, Grid g, const ulonglong2* tab, u64 nb,
                               const int* ids, int* labels, int n_sm, cudaStream_t st) {
    const u64 want = (n + 256 * kLkIlp - 1) / (256 * kLkIlp);
    const int blocks = (int)std::max<u64>(1, std::min<u64>(want, (u64)n_sm * 8));
    k_label_cells<<<blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(xy), n, g, tab, nb, ids,
                                          labels);
    return cudaGetLastError();
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
