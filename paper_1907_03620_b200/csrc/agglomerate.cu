// agglomerate.cu — K3: connected components over the significant tiles, the
// mu size filter and canonical relabelling, for sm_100a.
//
// Replaces connected_components (agglomerate.hpp:124-170: flat index +
// explicit-stack DFS with one hash probe per neighbour offset), the size
// filter in agglomerate (:196-201) and finalize_clusters (:175-191).
//
// Algorithm (all O(S), no full sort):
//   1. union   — one thread per significant tile probes the forward half of
//                the delta-ball (the ball is symmetric, so every adjacent
//                pair is seen exactly once) in the HBM hash table, whose
//                value word already holds SIG_BIT|index after K2, and unites
//                the two components. Union-find hooks the larger root under
//                the smaller (ECL-CC style CAS loop, path halving in find),
//                which keeps parent[x] <= x and converges in O(S α) work even
//                for config 5's 10^4-tile chains, where label propagation
//                would need diameter-many rounds.
//   2. compress — parent[i] = root(i).
//   3. reduce  — per root: tile count, point count and the smallest packed
//                key (= the cluster's lexicographically smallest tile, the
//                sort key of finalize_clusters :186-189).
//   4. select  — roots with size >= mu are appended as (min_key, root).
//   5. order   — the C kept roots (C <= S) are radix-sorted by min_key; the
//                rank is the canonical cluster id (:189-190).
//   6. label   — every tile gets the id of its root (or -1).
#include <climits>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "internal.h"

namespace rg {

__device__ __forceinline__ u32 ld_parent(const u32* p) {
    u32 v;
    asm volatile("ld.global.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ u32 uf_find(u32* parent, u32 v) {
    u32 par = ld_parent(parent + v);
    if (par != v) {
        u32 prev = v, next;
        while (par > (next = ld_parent(parent + par))) {
            parent[prev] = next;  // path halving; monotone, benign race
            prev = par;
            par = next;
        }
    }
    return par;
}

__device__ __forceinline__ void uf_unite(u32* parent, u32 a, u32 b) {
    u32 ra = uf_find(parent, a);
    u32 rb = uf_find(parent, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 t = ra;
            ra = rb;
            rb = t;
        }
        // hook ra (larger) under rb (smaller)
        const u32 old = atomicCAS(parent + ra, ra, rb);
        if (old == ra) return;
        ra = old;  // ra was hooked meanwhile: continue from its new parent
    }
}

struct Offsets {
    const int2* d;  // forward half of the delta-ball
    int n;
    int cheb1;      // d == {(0,1), (1,-1), (1,0), (1,1)}: Chebyshev, delta 1
};

// Significant-tile index of (kx+dx, ky+dy), or 0xffffffff.
__device__ __forceinline__ u32 sig_index(const Table& t, long long kx, long long ky, int dx, int dy,
                                         u32 bits_y, long long xlim, long long ylim) {
    const long long nx = kx + dx, ny = ky + dy;
    if (nx < 0 || nx >= xlim || ny < 0 || ny >= ylim) return 0xffffffffu;
    const u64 v = table_find(t, ((u64)nx << bits_y) | (u64)ny);
    return (v != kEmpty && (v & kSigBit)) ? (u32)(v & ~kSigBit) : 0xffffffffu;
}

__device__ __forceinline__ u32 lfind(volatile u32* lp, u32 x) {
    u32 p;
    while ((p = lp[x]) != x) x = p;
    return x;
}

__device__ __forceinline__ void lunite(u32* lp, u32 a, u32 b) {
    volatile u32* v = lp;
    u32 ra = lfind(v, a), rb = lfind(v, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 tmp = ra;
            ra = rb;
            rb = tmp;
        }
        const u32 old = atomicCAS(lp + ra, ra, rb);
        if (old == ra) return;
        ra = lfind(v, old);
        rb = lfind(v, rb);
    }
}

constexpr int kStoredNb = 4;  // neighbour indices kept per tile for the warp-local pass

// Union step. Tiles come in compaction (bucket) order, so a warp's 32
// consecutive tiles are mostly spatial neighbours. Each warp:
//   1. probes the forward neighbours of its 32 tiles in the counting table
//      (for Chebyshev delta 1 the two orthogonal probes are issued together
//      and the diagonals only when needed — they are otherwise reached
//      through the orthogonal neighbours);
//   2. resolves edges between its own tiles with a shared-memory union-find
//      over lanes and points every tile at its local component's smallest
//      member (a plain store: no other thread writes these entries in this
//      kernel, so nothing can be overwritten);
//   3. writes the edges that leave the warp into the warp's fixed slots of
//      the edge list (no atomics), for k_union_edges.
// Global union-find work therefore runs once every tile is linked to its
// local root (short finds) and as one uniform thread per edge, instead of as
// divergent per-lane loops here.
struct EdgeList {
    uint2* e;    // kEdgeSlots per warp window
    u32* n;      // edges per window
};
constexpr int kEdgeSlots = 32 * kStoredNb;

// Two lookups with their first loads in flight together (latency-bound:
// random buckets, short chains), each finished by its own probe loop only
// when the first slot holds a different key.
__device__ __forceinline__ void sig_index2(const Table& t, long long kx, long long ky, int2 d0,
                                           int2 d1, u32 bits_y, long long xlim, long long ylim,
                                           u32& o0, u32& o1) {
    const long long x0 = kx + d0.x, y0 = ky + d0.y, x1 = kx + d1.x, y1 = ky + d1.y;
    const bool ok0 = !(x0 < 0 || x0 >= xlim || y0 < 0 || y0 >= ylim);
    const bool ok1 = !(x1 < 0 || x1 >= xlim || y1 < 0 || y1 >= ylim);
    const u64 q0 = ((u64)x0 << bits_y) | (u64)y0, q1 = ((u64)x1 << bits_y) | (u64)y1;
    Probe p0(q0, t), p1(q1, t);
    u64 k0 = kEmpty, v0 = 0, k1 = kEmpty, v1 = 0;
    if (ok0) ld_slot(t.slots + p0.slot(), k0, v0);
    if (ok1) ld_slot(t.slots + p1.slot(), k1, v1);
    while (ok0 && k0 != q0 && k0 != kEmpty) {
        p0.next(t);
        ld_slot(t.slots + p0.slot(), k0, v0);
    }
    while (ok1 && k1 != q1 && k1 != kEmpty) {
        p1.next(t);
        ld_slot(t.slots + p1.slot(), k1, v1);
    }
    o0 = (ok0 && k0 == q0 && (v0 & kSigBit)) ? (u32)(v0 & ~kSigBit) : 0xffffffffu;
    o1 = (ok1 && k1 == q1 && (v1 & kSigBit)) ? (u32)(v1 & ~kSigBit) : 0xffffffffu;
}

__global__ void __launch_bounds__(256) k_union(const u64* sig_key, const u64* n_sig_p, Table t,
                                               u32 bits_y, u32 bits_x, Offsets off, u32* parent,
                                               EdgeList el) {
    __shared__ u32 s_par[8][32];
    const u64 n_sig = *n_sig_p;
    const int lane = threadIdx.x & 31;
    u32* lp = s_par[threadIdx.x >> 5];
    const long long ymask = (1ll << bits_y) - 1;
    const long long xlim = 1ll << bits_x, ylim = 1ll << bits_y;
    const bool wide = off.n > kStoredNb;  // some edges are united here (delta > 1)
    const u64 span = (n_sig + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 base = i - lane;
        const u64 win = base / 32;
        const bool valid = i < n_sig;
        lp[lane] = lane;
        u32 nb[kStoredNb];
#pragma unroll
        for (int o = 0; o < kStoredNb; ++o) nb[o] = 0xffffffffu;
        if (valid) {
            const u64 key = sig_key[i];
            const long long kx = (long long)(key >> bits_y);
            const long long ky = (long long)key & ymask;
            if (off.cheb1) {
                sig_index2(t, kx, ky, make_int2(0, 1), make_int2(1, 0), bits_y, xlim, ylim, nb[0],
                           nb[2]);
                if (nb[2] == 0xffffffffu) {
                    if (nb[0] == 0xffffffffu)
                        sig_index2(t, kx, ky, make_int2(1, -1), make_int2(1, 1), bits_y, xlim,
                                   ylim, nb[1], nb[3]);
                    else
                        nb[1] = sig_index(t, kx, ky, 1, -1, bits_y, xlim, ylim);
                }
            } else {
                for (int o = 0; o < off.n; ++o) {
                    const int2 d = off.d[o];
                    const u32 j = sig_index(t, kx, ky, d.x, d.y, bits_y, xlim, ylim);
                    if (j == 0xffffffffu) continue;
                    if (o < kStoredNb)
                        nb[o] = j;
                    else
                        uf_unite(parent, (u32)i, j);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int o = 0; o < kStoredNb; ++o)
            if (nb[o] != 0xffffffffu && nb[o] >= base && nb[o] < base + 32)
                lunite(lp, (u32)lane, nb[o] - (u32)base);
        __syncwarp();
        const u32 r = lfind(lp, (u32)lane);
        if (valid && r != (u32)lane) {
            const u32 target = (u32)base + r;  // < i: keeps parent[x] <= x
            if (!wide)
                parent[i] = target;
            else if (atomicCAS(parent + i, (u32)i, target) != (u32)i)
                uf_unite(parent, (u32)i, target);
        }
        // edges leaving the warp -> this window's fixed slots
        u32 ext = 0;
#pragma unroll
        for (int o = 0; o < kStoredNb; ++o)
            if (nb[o] != 0xffffffffu && (nb[o] < base || nb[o] >= base + 32)) {
                bool dup = false;
#pragma unroll
                for (int q = 0; q < o; ++q) dup |= nb[q] == nb[o];
                if (!dup) ext |= 1u << o;
            }
        const u32 cnt = __popc(ext);
        u32 incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        uint2* slots = el.e + win * kEdgeSlots;
        u32 at = incl - cnt;
#pragma unroll
        for (int o = 0; o < kStoredNb; ++o)
            if (ext >> o & 1) slots[at++] = make_uint2((u32)base + r, nb[o]);
        if (lane == 31) el.n[win] = incl;
        __syncwarp();
    }
}

// Window-external edges: one warp per window, one lane per edge.
__global__ void k_union_edges(EdgeList el, const u64* n_sig_p, u32* parent) {
    const u64 n_win = (*n_sig_p + 31) / 32;
    const int lane = threadIdx.x & 31;
    for (u64 w = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; w < n_win;
         w += ((u64)gridDim.x * blockDim.x) >> 5) {
        const u32 n = el.n[w];
        for (u32 j = lane; j < n; j += 32) {
            const uint2 v = el.e[w * kEdgeSlots + j];
            uf_unite(parent, v.x, v.y);
        }
    }
}

// Flatten + per-root reductions. Flatten: every thread writes only its own
// entry, and only with a root, so concurrent walks never see (or leave
// behind) a non-root written late (a path-halving find here would race:
// another thread could overwrite parent[i] with a non-root ancestor after i
// stored its root). Reductions: tile count, point count and smallest packed
// key per root (accumulators were initialised by K2 / the load path). Tiles
// of one component sit in runs of consecutive indices (compaction order is
// bucket order), so each warp reduces its contiguous runs with a segmented
// shuffle reduction and only run heads touch global memory.
__global__ void k_compress_reduce(u32* parent, const u64* sig_key, const u64* sig_cnt,
                                  const u64* n_sig_p, u32* size, u64* npts, u64* min_key) {
    const u64 n_sig = *n_sig_p;
    const int lane = threadIdx.x & 31;
    const u64 span = ((n_sig + 31) / 32) * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const bool valid = i < n_sig;
        u32 r = 0xffffffffu;
        if (valid) {
            const u32 old = ld_parent(parent + i);
            u32 next;
            r = old;
            while (r > (next = ld_parent(parent + r))) r = next;
            if (r != old) parent[i] = r;
        }
        u32 cnt = valid ? 1u : 0u;
        u64 pts = valid && sig_cnt ? sig_cnt[i] : 0ull;
        u64 mk = valid ? sig_key[i] : kEmpty;
        const u32 prev = __shfl_up_sync(kFull, r, 1);
        const bool head = lane == 0 || prev != r;
        const u32 heads = __ballot_sync(kFull, head);
        const u32 run = __popc(heads & (0xffffffffu >> (31 - lane)));  // 1-based run id
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 orun = __shfl_down_sync(kFull, run, o);
            const u32 oc = __shfl_down_sync(kFull, cnt, o);
            const u64 op = __shfl_down_sync(kFull, pts, o);
            const u64 om = __shfl_down_sync(kFull, mk, o);
            if (lane + o < 32 && orun == run) {
                cnt += oc;
                pts += op;
                mk = om < mk ? om : mk;
            }
        }
        if (head && valid) {
            atomicAdd(size + r, cnt);
            atomicAdd(npts + r, pts);
            atomicMin(min_key + r, mk);
        }
    }
}

// Roots with size >= mu -> (min_key, root) pairs; counts components.
__global__ void k_select_roots(const u32* parent, const u32* size, const u64* min_key,
                               const u64* n_sig_p, u64 mu, u64* out_key, u32* out_root,
                               Counters* ctr) {
    // Each warp takes 256 consecutive tiles (8 per lane) and issues one
    // append atomic for all of them: a per-32-tile atomic on a single
    // counter serialises in L2 (measured 150 us at S = 8.75M).
    constexpr int kItems = 8;
    const u64 n_sig = *n_sig_p;
    const int lane = threadIdx.x & 31;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    u64 roots = 0;
    for (u64 base = warp * 32 * kItems; base < n_sig; base += n_warps * 32 * kItems) {
        u32 keep_bits = 0, nkeep = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const u64 i = base + j * 32 + lane;
            const bool root = i < n_sig && parent[i] == (u32)i;
            const bool keep = root && size[i] >= mu;
            roots += root;
            keep_bits |= (u32)keep << j;
            nkeep += keep;
        }
        u32 incl = nkeep;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const u32 total = __shfl_sync(kFull, incl, 31);
        u64 at = 0;
        if (lane == 31 && total) at = atomicAdd(&ctr->n_kept, (u64)total);
        at = __shfl_sync(kFull, at, 31);
        u64 pos = at + incl - nkeep;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if (keep_bits >> j & 1) {
                const u64 i = base + j * 32 + lane;
                out_key[pos] = min_key[i];
                out_root[pos] = (u32)i;
                ++pos;
            }
        }
    }
    const u32 r = __reduce_add_sync(kFull, (u32)roots);
    if (lane == 0 && r) atomicAdd(&ctr->n_roots, (u64)r);
}

__global__ void k_assign_ids(const u32* root_sorted, const u64* n_kept_p, int* root_cid) {
    const u64 n = *n_kept_p;
    for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < n;
         k += (u64)gridDim.x * blockDim.x)
        root_cid[root_sorted[k]] = (int)k;
}

__global__ void k_label_tiles(const u32* parent, const int* root_cid, const u64* n_sig_p,
                              int* tile_cid) {
    const u64 n_sig = *n_sig_p;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_sig;
         i += (u64)gridDim.x * blockDim.x)
        tile_cid[i] = root_cid[parent[i]];
}

// Load path (agglomerate(SignificantTiles) with caller tiles): pack and insert
// every tile as significant with its dense index.
__global__ void k_load_tiles(const long long* tx, const long long* ty, const u64* cnt, u64 n,
                             long long ox, long long oy, u32 bits_y, Table t, u64* sig_key,
                             u64* sig_cnt, u32* parent, u32* size, u64* npts, u64* min_key,
                             int* root_cid) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u64 key = ((u64)(tx[i] - ox) << bits_y) | (u64)(ty[i] - oy);
        sig_key[i] = key;
        sig_cnt[i] = cnt ? cnt[i] : 0;
        parent[i] = (u32)i;
        size[i] = 0;
        npts[i] = 0;
        min_key[i] = kEmpty;
        root_cid[i] = -1;
        const u64 slot = table_claim(t, key);
        t.slots[slot].count = kSigBit | i;
    }
}

// Extents of a device tile set (decides the key packing of the load path):
// out = {min x, max x, min y, max y}, preset by the caller to +inf/-inf.
__global__ void k_tile_extents(const long long* tx, const long long* ty, u64 n, long long* out) {
    long long mnx = LLONG_MAX, mxx = LLONG_MIN, mny = LLONG_MAX, mxy = LLONG_MIN;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const long long x = tx[i], y = ty[i];
        mnx = min(mnx, x);
        mxx = max(mxx, x);
        mny = min(mny, y);
        mxy = max(mxy, y);
    }
    for (int o = 16; o; o >>= 1) {
        mnx = min(mnx, __shfl_xor_sync(~0u, mnx, o));
        mxx = max(mxx, __shfl_xor_sync(~0u, mxx, o));
        mny = min(mny, __shfl_xor_sync(~0u, mny, o));
        mxy = max(mxy, __shfl_xor_sync(~0u, mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], mnx);
        atomicMax(&out[1], mxx);
        atomicMin(&out[2], mny);
        atomicMax(&out[3], mxy);
    }
}

// ---------------------------------------------------------------- launchers

static int grid_for(u64 n, int n_sm, int per_sm = 8) {
    const u64 want = (n + 255) / 256;
    const u64 cap = (u64)n_sm * per_sm;
    return (int)(want == 0 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_agglomerate(const AggLaunch& A, cudaStream_t st) {
    const int gs = grid_for(A.n_sig, A.n_sm, 16);
    Offsets off{A.offsets, A.n_offsets, A.cheb1};
    const EdgeList el{A.edges, A.edge_n};
    k_union<<<gs, 256, 0, st>>>(A.sig_key, A.n_sig_dev, A.t, A.bits_y, A.bits_x, off, A.parent, el);
    k_union_edges<<<gs, 256, 0, st>>>(el, A.n_sig_dev, A.parent);
    k_compress_reduce<<<gs, 256, 0, st>>>(A.parent, A.sig_key, A.sig_cnt, A.n_sig_dev, A.size,
                                          A.npts, A.min_key);
    k_select_roots<<<gs, 256, 0, st>>>(A.parent, A.size, A.min_key, A.n_sig_dev, A.mu,
                                       A.root_key, A.root_idx, A.ctr);
    return cudaGetLastError();
}

cudaError_t launch_order_and_label(const AggLaunch& A, u64 n_kept, cudaStream_t st) {
    if (n_kept > 0) {
        size_t bytes = A.sort_temp_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(
            A.sort_temp, bytes, A.root_key, A.root_key_sorted, A.root_idx, A.root_idx_sorted,
            (int)n_kept, 0, (int)(A.bits_x + A.bits_y), st);
        if (e != cudaSuccess) return e;
        k_assign_ids<<<grid_for(n_kept, A.n_sm), 256, 0, st>>>(A.root_idx_sorted,
                                                                &A.ctr->n_kept, A.root_cid);
    }
    k_label_tiles<<<grid_for(A.n_sig, A.n_sm, 16), 256, 0, st>>>(A.parent, A.root_cid,
                                                                 A.n_sig_dev, A.tile_cid);
    return cudaGetLastError();
}

size_t sort_pairs_temp_bytes(u64 n, int bits) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs((void*)nullptr, bytes, (const u64*)nullptr, (u64*)nullptr,
                                    (const u32*)nullptr, (u32*)nullptr, (int)n, 0, bits);
    return bytes;
}

cudaError_t sort_pairs(void* temp, size_t temp_bytes, const u64* k_in, u64* k_out,
                       const u32* v_in, u32* v_out, u64 n, int bits, cudaStream_t st) {
    size_t bytes = temp_bytes;
    return cub::DeviceRadixSort::SortPairs(temp, bytes, k_in, k_out, v_in, v_out, (int)n, 0,
                                           bits, st);
}

cudaError_t launch_load_tiles(const long long* tx, const long long* ty, const u64* cnt, u64 n,
                              long long ox, long long oy, u32 bits_y, Table t, u64* sig_key,
                              u64* sig_cnt, u32* parent, u32* size, u64* npts, u64* min_key,
                              int* root_cid, int n_sm, cudaStream_t st) {
    k_load_tiles<<<grid_for(n, n_sm), 256, 0, st>>>(tx, ty, cnt, n, ox, oy, bits_y, t, sig_key,
                                                     sig_cnt, parent, size, npts, min_key,
                                                     root_cid);
    return cudaGetLastError();
}

cudaError_t launch_tile_extents(const long long* tx, const long long* ty, u64 n, long long* out,
                                int n_sm, cudaStream_t st) {
    k_tile_extents<<<grid_for(n, n_sm, 4), 256, 0, st>>>(tx, ty, n, out);
    return cudaGetLastError();
}

}  // namespace rg
