// agglomerate_sorted.cu — K3 over the significant tiles in key order.
//
// Same contract as agglomerate.cu (connected_components agglomerate.hpp:124-170,
// the mu filter :198-199 and finalize_clusters :175-191) but the tiles are
// first radix-sorted by packed key, i.e. lexicographically by (tx, ty) — the
// canonical order of finalize_clusters. Then:
//   * neighbour discovery needs no hash probes: (x, y+1..y+r) are the next
//     entries of the same column, and column x+dx's window [y-r, y+r] is found
//     by a galloping search from the tile's own position (all L1/L2 hits:
//     neighbours in key order are close in memory);
//   * most edges join tiles a few positions apart, so a block resolves the
//     edges among its 256 consecutive tiles in a shared-memory union-find and
//     defers only the few edges leaving the window;
//   * the root of a component (smallest index) is its smallest tile, so
//     canonical cluster ids are an exclusive scan of "root with size >= mu"
//     flags — no per-root minimum and no sort of the roots;
//   * the sorted keys are the canonical output order.
// Used for delta <= 2 (at most 12 forward offsets, bounded edge list).
#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace rg {

namespace {

__device__ __forceinline__ u32 s_ld_parent(const u32* p) {
    u32 v;
    asm volatile("ld.global.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ u32 s_find(u32* parent, u32 v) {
    u32 par = s_ld_parent(parent + v);
    if (par != v) {
        u32 prev = v, next;
        while (par > (next = s_ld_parent(parent + par))) {
            parent[prev] = next;
            prev = par;
            par = next;
        }
    }
    return par;
}

__device__ __forceinline__ void s_unite(u32* parent, u32 a, u32 b) {
    u32 ra = s_find(parent, a), rb = s_find(parent, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 t = ra;
            ra = rb;
            rb = t;
        }
        const u32 old = atomicCAS(parent + ra, ra, rb);
        if (old == ra) return;
        ra = old;
    }
}

// s_unite that records the root it links under another (each root is
// linked at most once), so its counts can be folded into the final root.
__device__ __forceinline__ void s_unite_rec(u32* parent, u32 a, u32 b, u32* linked,
                                            u64* n_linked) {
    u32 ra = s_find(parent, a), rb = s_find(parent, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 t = ra;
            ra = rb;
            rb = t;
        }
        const u32 old = atomicCAS(parent + ra, ra, rb);
        if (old == ra) {
            linked[atomicAdd(n_linked, 1ull)] = ra;
            return;
        }
        ra = old;
    }
}

__device__ __forceinline__ u32 l_find(volatile u32* lp, u32 x) {
    u32 p;
    while ((p = lp[x]) != x) x = p;
    return x;
}

// Find with path halving (shared memory). Parents only ever move to smaller
// members of the same set, so a plain store of the grandparent is safe: a
// lost race only loses compression. Roots are never written here.
__device__ __forceinline__ u32 l_find_h(volatile u32* lp, u32 x) {
    u32 p = lp[x];
    while (p != x) {
        const u32 g = lp[p];
        if (g == p) return p;
        lp[x] = g;
        x = g;
        p = lp[x];
    }
    return x;
}

__device__ __forceinline__ void l_unite_h(u32* lp, u32 a, u32 b) {
    volatile u32* v = lp;
    u32 ra = l_find_h(v, a), rb = l_find_h(v, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 t = ra;
            ra = rb;
            rb = t;
        }
        const u32 old = atomicCAS(lp + ra, ra, rb);
        if (old == ra) return;
        ra = l_find_h(v, old);
        rb = l_find_h(v, rb);
    }
}

__device__ __forceinline__ void l_unite(u32* lp, u32 a, u32 b) {
    volatile u32* v = lp;
    u32 ra = l_find(v, a), rb = l_find(v, b);
    while (ra != rb) {
        if (ra < rb) {
            const u32 t = ra;
            ra = rb;
            rb = t;
        }
        const u32 old = atomicCAS(lp + ra, ra, rb);
        if (old == ra) return;
        ra = l_find(v, old);
        rb = l_find(v, rb);
    }
}

// First index j >= from with key[j] >= target (galloping, then binary).
__device__ __forceinline__ u64 gallop(const u64* key, u64 n, u64 from, u64 target) {
    if (from >= n || key[from] >= target) return from;
    u64 lo = from, step = 1, hi = from + 1;
    while (hi < n && key[hi] < target) {
        lo = hi;
        step <<= 1;
        hi = from + step;
    }
    if (hi > n) hi = n;
    // key[lo] < target; answer in (lo, hi]
    u64 a = lo + 1, b = hi;
    while (a < b) {
        const u64 m = (a + b) >> 1;
        if (key[m] < target)
            a = m + 1;
        else
            b = m;
    }
    return a;
}

}  // namespace

struct SortedEdges {
    uint2* e;
    u64 cap;
    u64* n;
};

// Window = the 256 consecutive tiles of a block.
__global__ void __launch_bounds__(256) k_sorted_union(const u64* skey, const u64* n_sig_p,
                                                      u32 bits_y, int delta, int manhattan,
                                                      u32* parent, u32* size, u64* npts,
                                                      SortedEdges el) {
    __shared__ u32 s_par[256];
    __shared__ u32 s_wcnt[8];
    __shared__ u64 s_base;
    const u64 n = *n_sig_p;
    const u32 loc = threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 ymask = (1ull << bits_y) - 1;
    const u64 span = (n + 255) / 256 * 256;
    for (u64 i = blockIdx.x * 256ull + loc; i < span; i += (u64)gridDim.x * 256) {
        const u64 base = i - loc;
        const u64 wend = base + 256;
        const bool valid = i < n;
        s_par[loc] = loc;
        __syncthreads();
        u32 ext[12];
        int n_ext = 0;
        if (valid) {
            const u64 k = skey[i];
            const u64 x = k >> bits_y, y = k & ymask;
            // same column, rows y+1 .. y+delta: the next entries
            for (u64 j = i + 1; j < n; ++j) {
                const u64 kj = skey[j];
                if ((kj >> bits_y) != x || (kj & ymask) > y + (u64)delta) break;
                if (j < wend)
                    l_unite(s_par, loc, (u32)(j - base));
                else if (n_ext < 12)
                    ext[n_ext++] = (u32)j;
            }
            // columns x+1 .. x+delta
            u64 from = i + 1;
            for (int dx = 1; dx <= delta; ++dx) {
                const u64 r = manhattan ? (u64)(delta - dx) : (u64)delta;
                const u64 nx = x + (u64)dx;
                if (nx >> (63 - bits_y)) break;  // beyond the key space
                const u64 ylo = y >= r ? y - r : 0;
                const u64 lo_key = (nx << bits_y) | ylo;
                const u64 hi_key = (nx << bits_y) | min(y + r, ymask);
                u64 j = gallop(skey, n, from, lo_key);
                from = j;
                for (; j < n && skey[j] <= hi_key; ++j) {
                    if (j < wend)
                        l_unite(s_par, loc, (u32)(j - base));
                    else if (n_ext < 12)
                        ext[n_ext++] = (u32)j;
                }
            }
        }
        __syncthreads();
        const u32 r = l_find(s_par, loc);
        if (valid) {
            parent[i] = (u32)base + r;  // <= i; sole writer of parent[i] in this kernel
            size[i] = 0;
            npts[i] = 0;
        }
        // deferred window-external edges: block-aggregated reservation
        u32 incl = (u32)n_ext;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 yv = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += yv;
        }
        if (lane == 31) s_wcnt[wid] = incl;
        __syncthreads();
        if (loc == 0) {
            u32 tot = 0;
            for (int q = 0; q < 8; ++q) {
                const u32 c = s_wcnt[q];
                s_wcnt[q] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(el.n, (u64)tot) : 0;
        }
        __syncthreads();
        u64 at = s_base + s_wcnt[wid] + incl - (u32)n_ext;
        for (int q = 0; q < n_ext; ++q, ++at)
            if (at < el.cap) el.e[at] = make_uint2((u32)base + r, ext[q]);
        __syncthreads();
    }
}

// Chebyshev delta 1 (the BASELINE setting): at most four forward neighbours
// (x, y+1) = the next entry, and (x+1, y-1..y+1) found by one galloping
// search. A diagonal edge is dropped when an orthogonal neighbour makes it
// redundant ((x+1,y+1) touches (x,y+1) and (x+1,y); (x+1,y-1) touches
// (x+1,y)). Window-local components are found by min-label propagation with
// pointer jumping in shared memory (converges in a few rounds; labels only
// decrease), then every tile is linked to its component's smallest member.
// The block's 256 keys plus the next kC1Extra (where the next column of
// the window's last tiles usually lies) are staged in shared memory, so the
// neighbour searches run on shared memory; a search that leaves the staged
// range continues in global memory.
constexpr u32 kC1Extra = 256;

__global__ void __launch_bounds__(256) k_sorted_union_c1(const u64* skey, const u64* n_sig_p,
                                                         u32 bits_y, u32* parent, u32* size,
                                                         u64* npts, SortedEdges el) {
    __shared__ u32 s_lbl[256];
    __shared__ u32 s_wcnt[8];
    __shared__ u64 s_base;
    __shared__ u64 s_key[256 + kC1Extra];
    const u64 n = *n_sig_p;
    const u32 loc = threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 ymask = (1ull << bits_y) - 1;
    const u64 span = (n + 255) / 256 * 256;
    for (u64 i = blockIdx.x * 256ull + loc; i < span; i += (u64)gridDim.x * 256) {
        const u64 base = i - loc;
        const u64 wend = base + 256;
        const bool valid = i < n;
        const u32 staged = (u32)min((u64)(256 + kC1Extra), n - base);
        for (u32 q = loc; q < 256 + kC1Extra; q += 256) s_key[q] = q < staged ? skey[base + q] : ~0ull;
        __syncthreads();
        // key at global index j (staged range from shared memory)
        auto key_at = [&](u64 j) -> u64 { return j - base < staged ? s_key[j - base] : skey[j]; };
        u32 nb[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
        if (valid) {
            const u64 k = s_key[loc];
            const u64 y = k & ymask;
            // (x, y+1); key + 1 wraps to (x+1, 0) when y is the top row
            if (y != ymask && i + 1 < n && key_at(i + 1) == k + 1) nb[0] = (u32)(i + 1);
            const u64 nxk = k + (1ull << bits_y);                          // (x+1, y)
            if ((nxk >> bits_y) == (k >> bits_y) + 1) {
                const u64 lo = y > 0 ? nxk - 1 : nxk;
                u64 j;
                if (s_key[staged - 1] >= lo) {
                    // first staged index > loc with key >= lo: gallop, then bisect
                    u32 a = loc + 1, step = 1, b = loc + 1;
                    while (b < staged && s_key[b] < lo) {
                        a = b;
                        b += step;
                        step <<= 1;
                    }
                    if (b > staged) b = staged;
                    while (a < b) {
                        const u32 m = (a + b) >> 1;
                        if (s_key[m] < lo) a = m + 1;
                        else b = m;
                    }
                    j = base + a;
                } else {
                    j = gallop(skey, n, base + staged, lo);
                }
                u32 dm = 0xffffffffu, d0 = 0xffffffffu, dp = 0xffffffffu;
                for (; j < n; ++j) {
                    const u64 kj = key_at(j);
                    if (kj > nxk + 1 || (y == ymask && kj > nxk)) break;
                    if (kj == nxk - 1 && y > 0) dm = (u32)j;
                    else if (kj == nxk) d0 = (u32)j;
                    else if (kj == nxk + 1) dp = (u32)j;
                }
                nb[2] = d0;
                if (d0 == 0xffffffffu) {
                    nb[1] = dm;
                    if (nb[0] == 0xffffffffu) nb[3] = dp;
                }
            }
        }
        s_lbl[loc] = loc;
        __syncthreads();
        while (true) {
            bool ch = false;
            u32 m = s_lbl[loc];
#pragma unroll
            for (int o = 0; o < 4; ++o)
                if (nb[o] < wend && nb[o] >= base) m = min(m, s_lbl[nb[o] - base]);
#pragma unroll
            for (int o = 0; o < 4; ++o)
                if (nb[o] < wend && nb[o] >= base && s_lbl[nb[o] - base] > m) {
                    atomicMin(&s_lbl[nb[o] - base], m);
                    ch = true;
                }
            if (m < s_lbl[loc]) {
                atomicMin(&s_lbl[loc], m);
                ch = true;
            }
            __syncthreads();
            const u32 l = s_lbl[loc];
            const u32 ll = s_lbl[l];
            if (ll < l) {
                atomicMin(&s_lbl[loc], ll);
                ch = true;
            }
            if (!__syncthreads_or(ch)) break;
        }
        const u32 r = s_lbl[loc];
        if (valid) {
            parent[i] = (u32)base + r;  // <= i; sole writer of parent[i] in this kernel
            size[i] = 0;
            npts[i] = 0;
        }
        // deferred window-external edges: block-aggregated reservation
        u32 n_ext = 0;
#pragma unroll
        for (int o = 0; o < 4; ++o) n_ext += (nb[o] != 0xffffffffu && nb[o] >= wend);
        u32 incl = n_ext;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 yv = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += yv;
        }
        if (lane == 31) s_wcnt[wid] = incl;
        __syncthreads();
        if (loc == 0) {
            u32 tot = 0;
            for (int q = 0; q < 8; ++q) {
                const u32 c = s_wcnt[q];
                s_wcnt[q] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(el.n, (u64)tot) : 0;
        }
        __syncthreads();
        u64 at = s_base + s_wcnt[wid] + incl - n_ext;
#pragma unroll
        for (int o = 0; o < 4; ++o)
            if (nb[o] != 0xffffffffu && nb[o] >= wend) {
                if (at < el.cap) el.e[at] = make_uint2((u32)base + r, nb[o]);
                ++at;
            }
        __syncthreads();
    }
}

__global__ void k_sorted_edges(SortedEdges el, u32* parent) {
    const u64 n = min(*el.n, el.cap);
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const uint2 v = el.e[i];
        s_unite(parent, v.x, v.y);
    }
}

// Flatten + per-root tile and point counts (segmented warp reduction over
// runs of equal roots; only run heads touch global memory). Counts are read
// through the sort permutation.
__global__ void k_sorted_reduce(u32* parent, const u32* perm, const u64* cnt_b,
                                const u64* n_sig_p, u32* size, u64* npts, u32* is_root,
                                u64 mu) {
    const u64 n = *n_sig_p;
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const bool valid = i < n;
        u32 r = 0xffffffffu;
        if (valid) {
            const u32 old = s_ld_parent(parent + i);
            u32 next;
            r = old;
            while (r > (next = s_ld_parent(parent + r))) r = next;
            if (r != old) parent[i] = r;
        }
        u32 c = valid ? 1u : 0u;
        u64 p = valid && cnt_b ? cnt_b[perm[i]] : 0ull;
        const u32 prev = __shfl_up_sync(kFull, r, 1);
        const bool head = lane == 0 || prev != r;
        const u32 heads = __ballot_sync(kFull, head);
        const u32 run = __popc(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 orun = __shfl_down_sync(kFull, run, o);
            const u32 oc = __shfl_down_sync(kFull, c, o);
            const u64 op = __shfl_down_sync(kFull, p, o);
            if (lane + o < 32 && orun == run) {
                c += oc;
                p += op;
            }
        }
        if (head && valid) {
            atomicAdd(size + r, c);
            atomicAdd(npts + r, p);
        }
    }
}

// Kept-root flag of sorted position i (root with >= mu tiles), evaluated
// inside the id scan: the root of a component is its smallest tile, so the
// exclusive scan of the flags in sorted order is the canonical id
// (finalize_clusters agglomerate.hpp:186-190).



// ---------------------------------------------------- single-pass scans
// (decoupled look-back helpers: common.cuh)

// Column offsets for the column-ordered K3 in one pass (replaces a column
// maximum pass, a library scan and a bucket-bounds search): col_off =
// exclusive scan of the column histogram (cols + 1 entries, the last is n),
// the longest column into *max_col, and for 2^shift-tile buckets the start
// of bucket b, rs[b] = the first column start >= b << shift (rs[nbkt] = n),
// copied to the scatter cursors rs[nbkt + 1 + b]. One block per tile.
constexpr int kCsThr = 256, kCsPer = 16, kCsTile = kCsThr * kCsPer;
__global__ void __launch_bounds__(kCsThr) k_col_scan(const u32* cnt, u64 cols, const u64* n_p,
                                                     u32 shift, u32* col_off, u32* max_col,
                                                     u32* rs, u64* status, u32* ticket) {
    __shared__ u32 s_warp[33];
    __shared__ u32 s_tile;
    __shared__ u64 s_pre;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 total_cols = cols + 1;
    const u64 c0 = (u64)tile * kCsTile + (u64)threadIdx.x * kCsPer;
    u32 v[kCsPer];
    u32 sum = 0, mx = 0;
#pragma unroll
    for (int j = 0; j < kCsPer; ++j) {
        v[j] = c0 + j < cols ? cnt[c0 + j] : 0;  // index cols is the end marker
        sum += v[j];
        mx = max(mx, v[j]);
    }
    u32 agg;
    const u32 ex = block_excl_sum<kCsThr>(sum, s_warp, &agg);
    if (threadIdx.x < 32) {
        const u64 pre = lb_prefix(status, tile, agg);
        if (threadIdx.x == 0) s_pre = pre;
    }
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_col, mx);
    __syncthreads();
    const u64 n = *n_p;
    const u64 nbkt = (n + (1ull << shift) - 1) >> shift;
    u32* cur = rs + nbkt + 1;
    u64 off = s_pre + ex;
    // column c starts at s_c; bucket b starts at c when s_{c-1} < b << shift <= s_c
    u64 prev = c0 > 0 && c0 - 1 < cols ? off - cnt[c0 - 1] : off;
#pragma unroll
    for (int j = 0; j < kCsPer; ++j) {
        const u64 c = c0 + j;
        if (c < total_cols) {
            col_off[c] = (u32)off;
            for (u64 b = c == 0 ? 0 : (prev >> shift) + 1; b < nbkt && (b << shift) <= off; ++b) {
                rs[b] = (u32)off;
                cur[b] = (u32)off;
            }
            if (c == cols) rs[nbkt] = (u32)n;
        }
        prev = off;
        off += v[j];
    }
}

// Canonical ids in one pass (replaces the kept-root library scan and the
// labelling kernel): in sorted order a tile's root is its component's
// smallest position (P2-P4 link larger roots under smaller ones), so the
// number of kept roots before a root is its cluster id (finalize_clusters
// agglomerate.hpp:186-190). Tiles whose root lies in an earlier tile wait
// for that tile's ids (tiles are taken in ticket order: the wait ends).
// (tile shapes measured on config 4, K3 in all: 256 x 16 positions 0.673 ms,
// 256 x 8: 0.663, 512 x 8: 0.655, 512 x 4: 0.678, 1024 x 4: 0.672)
#ifndef RG_IDS_THR
#define RG_IDS_THR 512
#endif
#ifndef RG_IDS_PER
#define RG_IDS_PER 8
#endif
constexpr int kLbThr = RG_IDS_THR, kLbPer = RG_IDS_PER, kLbTile = kLbThr * kLbPer;
__global__ void __launch_bounds__(kLbThr) k_sorted_ids(const u32* parent, const u32* size,
                                                       u64 mu, const u32* perm, const u64* n_sig_p,
                                                       int* tile_cid_b, int* cid_s, u32* clu_root,
                                                       Counters* ctr, u64* status, u32* done,
                                                       u32* ticket) {
    __shared__ u32 s_warp[33];
    __shared__ u32 s_tile;
    __shared__ u64 s_pre;
    __shared__ int s_cid[kLbTile];
    __shared__ u32 s_root[kLbTile];
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const u64 n = *n_sig_p;
    const u64 t0 = (u64)tile * kLbTile;
    // roots (coalesced: item j of thread t is position t0 + j * kLbThr + t)
#pragma unroll 4
    for (int j = 0; j < kLbPer; ++j) {
        const u32 li = j * kLbThr + threadIdx.x;
        u32 r = 0xffffffffu;
        if (t0 + li < n) {
            // parent is final here (read-only in this kernel): cached loads
            r = __ldg(parent + t0 + li);
            u32 nx;
            while ((nx = __ldg(parent + r)) != r) r = nx;  // linked bucket roots (P3)
        }
        s_root[li] = r;
    }
    __syncthreads();
    // kept-root flags in position order: thread t owns positions t * kLbPer ..
    u32 flags = 0, cntk = 0, roots = 0;
#pragma unroll
    for (int j = 0; j < kLbPer; ++j) {
        const u32 li = threadIdx.x * kLbPer + j;
        const bool root = t0 + li < n && s_root[li] == (u32)(t0 + li);
        const bool kept = root && __ldg(size + t0 + li) >= mu;
        flags |= (u32)kept << j;
        cntk += kept;
        roots += root;
    }
    u32 agg;
    const u32 ex = block_excl_sum<kLbThr>(cntk, s_warp, &agg);
    if (threadIdx.x < 32) {
        const u64 pre = lb_prefix(status, tile, agg);
        if (threadIdx.x == 0) s_pre = pre;
    }
    __syncthreads();
    const u64 pre = s_pre;
    u32 k = ex;
#pragma unroll
    for (int j = 0; j < kLbPer; ++j) {
        const u32 li = threadIdx.x * kLbPer + j;
        int cid = -1;
        if ((flags >> j) & 1u) {
            cid = (int)(pre + k++);
            clu_root[cid] = (u32)(t0 + li);
            cid_s[t0 + li] = cid;
        }
        s_cid[li] = cid;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(done + tile, 1u);  // this tile's root ids are visible
    }
#pragma unroll 4
    for (int j = 0; j < kLbPer; ++j) {
        const u32 li = j * kLbThr + threadIdx.x;
        const u64 i = t0 + li;
        if (i >= n) continue;
        const u32 r = s_root[li];
        int cid;
        if (r >= t0) {
            cid = s_cid[r - t0];
        } else {  // root in an earlier tile: wait for its ids
            const u32 rt = (u32)(r / kLbTile);
            while (*(volatile u32*)(done + rt) == 0) {
            }
            __threadfence();
            cid = __ldg(size + r) >= mu ? *(volatile int*)(cid_s + r) : -1;
        }
        cid_s[i] = cid;
        if (tile_cid_b) tile_cid_b[perm[i]] = cid;
    }
    roots = __reduce_add_sync(kFull, roots);
    if ((threadIdx.x & 31) == 0 && roots) atomicAdd(&ctr->n_roots, (u64)roots);
    if (t0 + kLbTile >= n && threadIdx.x == 0) ctr->n_kept = pre + agg;  // the last tile
}

// Key sort by columns (when the column field has <= kColBitsMax bits): a
// counting sort on the column (histogram, scan, scatter), then a segmented
// sort of each column by row — two passes over the data instead of the
// radix sort's five, and columns are short (tens of tiles).
#ifndef RG_COL_BITS_MAX
#define RG_COL_BITS_MAX 22
#endif
constexpr u32 kColBitsMax = RG_COL_BITS_MAX;

__global__ void k_col_hist(const u64* key, const u64* n_p, u32 bits_y, u32* cnt, u32* max_col) {
    // Consecutive tiles (bucket order) share columns: one atomic per column
    // group of a warp.
    const u64 n = *n_p;
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    u32 mx = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const bool valid = i < n;
        const u32 col = valid ? (u32)(key[i] >> bits_y) : 0xffffffffu;
        const u32 peers = __match_any_sync(kFull, col);
        if (valid && lane == __ffs(peers) - 1) {
            const u32 c = atomicAdd(cnt + col, (u32)__popc(peers)) + __popc(peers);
            mx = max(mx, c);
        }
    }
    mx = __reduce_max_sync(kFull, mx);
    if (lane == 0 && mx) atomicMax(max_col, mx);
}

// Each thread scatters kColIlp keys of a warp tile whose reservations are in
// flight together (the reservation's round trip, not bandwidth, bounds a
// one-key-per-iteration scatter).
constexpr int kColIlp = 4;
__global__ void __launch_bounds__(256) k_col_scatter(const u64* key, const u64* n_p, u32 bits_y,
                                                     u32* cursor, u64* k_out, u32* v_out) {
    const u64 n = *n_p;
    const int lane = threadIdx.x & 31;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    constexpr u64 tile = 32ull * kColIlp;
    for (u64 base = warp * tile; base < n; base += n_warps * tile) {
        u64 k[kColIlp];
        u32 col[kColIlp], peers[kColIlp], at[kColIlp];
#pragma unroll
        for (int j = 0; j < kColIlp; ++j) {
            const u64 i = base + j * 32 + lane;
            k[j] = i < n ? key[i] : 0;
            col[j] = i < n ? (u32)(k[j] >> bits_y) : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < kColIlp; ++j) peers[j] = __match_any_sync(kFull, col[j]);
#pragma unroll
        for (int j = 0; j < kColIlp; ++j) {
            const int leader = __ffs(peers[j]) - 1;
            at[j] = 0;
            if (col[j] != 0xffffffffu && lane == leader)
                at[j] = atomicAdd(cursor + col[j], (u32)__popc(peers[j]));
        }
#pragma unroll
        for (int j = 0; j < kColIlp; ++j) {
            const int leader = __ffs(peers[j]) - 1;
            const u32 pos = __shfl_sync(kFull, at[j], leader) +
                            __popc(peers[j] & ((1u << lane) - 1));
            const u64 i = base + j * 32 + lane;
            if (i < n) {
                k_out[pos] = k[j];
                v_out[pos] = (u32)i;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Bucketed column sort (default when every column holds <= kBktMaxCol tiles).
//
// The column counting sort gives every column its final range col_off[c] ..
// col_off[c+1]. Columns are grouped into buckets of about kBkt tiles: the
// bucket of a column is col_off[c] / kBkt, so a bucket is a run of whole
// columns whose sorted range [rs[b], rs[b+1]) is shorter than kBkt + the
// longest column. Then
//   P1 k_bkt_scatter: each block ranks its 8192 keys per bucket in shared
//      memory and reserves one range per (block, bucket) — about one global
//      atomic per two keys instead of one per column group of a warp;
//   P2 k_bkt_sort: one block per bucket places the bucket's keys by column in
//      shared memory, ranks each key inside its (short) column, writes the
//      sorted run, and (Chebyshev delta 1) resolves the bucket's unions in a
//      shared-memory union-find — the whole bucket is the union window;
//   P3 k_bkt_cross: the only edges P2 cannot see join the last column of a
//      bucket and the first column of the next; one warp per bucket boundary
//      unites them in the global union-find.
// Every component's root is its smallest sorted index, as in the 256-tile
// window kernels, so the reduce / id / label passes are shared.
// ---------------------------------------------------------------------------
// Bucket size 2^shift tiles and P2 block shapes: 4096-tile buckets in
// 512-thread blocks (108 KB, 2 per SM) for columns of <= 2048 tiles, or
// (RG_BKT_SHIFT=11) 2048-tile buckets in 256-thread blocks (55 KB, 4 per
// SM) when every column holds <= 1024 tiles.
// (P1 block shapes on config 4, K3 in all: 512 x 8 keys 0.673 ms, 256 x 8: 0.662,
// 512 x 4: 0.666, 1024 x 8: 0.674, 128 x 8 as 256 x 8)
#ifndef RG_P1_THREADS
#define RG_P1_THREADS 256
#endif
#ifndef RG_P1_PER
#define RG_P1_PER 8
#endif
constexpr int kP1Threads = RG_P1_THREADS;
constexpr int kP1Per = RG_P1_PER;       // keys per thread (256 x 8 = 2048 per block)
constexpr u32 kP1Tile = kP1Threads * kP1Per;
constexpr u32 kP1RankBits = 13;         // rank inside a block's tile < 8192
static_assert(kP1Tile <= (1u << kP1RankBits), "P1 tile rank field");
constexpr int kP2Items = 12;
#ifndef RG_BKT_MAX_COL
#define RG_BKT_MAX_COL 2048
#endif
constexpr u64 kBktMaxCol = RG_BKT_MAX_COL;  // 4096 + kBktMaxCol <= 512 * kP2Items
constexpr size_t p2_smem(int threads) { return (size_t)threads * kP2Items * (8 + 4 + 4 + 2); }

// (n and the bucket count are read on the device: the launch may be sized
// for an upper bound of n; `nbkt_cap` >= the bucket count lays out the
// shared memory; rs = bucket starts, then the scatter cursors, as
// k_col_scan left them)
__global__ void __launch_bounds__(kP1Threads) k_bkt_scatter(const u64* key, const u64* n_p,
                                                            u32 bits_y, const u32* col_off,
                                                            u32* rs, u32 nbkt_cap, u32 shift,
                                                            u64* k_out, u32* v_out) {
    extern __shared__ u32 sh_p1[];
    const u64 n = *n_p;
    const u32 nbkt = (u32)((n + (1ull << shift) - 1) >> shift);
    u32* cur = rs + nbkt + 1;
    u32* hist = sh_p1;
    u32* base = sh_p1 + nbkt_cap;
    for (u64 t0 = blockIdx.x * (u64)kP1Tile; t0 < n; t0 += (u64)gridDim.x * kP1Tile) {
        for (u32 b = threadIdx.x; b < nbkt; b += kP1Threads) hist[b] = 0;
        __syncthreads();
        u64 k[kP1Per];
        u32 br[kP1Per];
#pragma unroll
        for (int j = 0; j < kP1Per; ++j) {
            const u64 i = t0 + (u64)j * kP1Threads + threadIdx.x;
            k[j] = i < n ? key[i] : 0;
        }
#pragma unroll
        for (int j = 0; j < kP1Per; ++j) {
            const u64 i = t0 + (u64)j * kP1Threads + threadIdx.x;
            br[j] = 0xffffffffu;
            if (i < n) {
                const u32 b = __ldg(col_off + (k[j] >> bits_y)) >> shift;
                br[j] = (b << kP1RankBits) | atomicAdd(&hist[b], 1u);
            }
        }
        __syncthreads();
        // one reservation per (tile, bucket); a thread's reservations are
        // issued together (their round trips overlap instead of queueing)
        for (u32 b0 = threadIdx.x; b0 < nbkt; b0 += 4 * kP1Threads) {
            u32 r[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u32 b = b0 + q * kP1Threads;
                const u32 c = b < nbkt ? hist[b] : 0;
                r[q] = c ? atomicAdd(cur + b, c) : 0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const u32 b = b0 + q * kP1Threads;
                if (b < nbkt) base[b] = r[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kP1Per; ++j) {
            if (br[j] != 0xffffffffu) {
                const u32 pos = base[br[j] >> kP1RankBits] + (br[j] & ((1u << kP1RankBits) - 1));
                k_out[pos] = k[j];
                v_out[pos] = (u32)(t0 + (u64)j * kP1Threads + threadIdx.x);
            }
        }
        __syncthreads();
    }
}

// Shared memory per P2 block: keys, perm, a per-slot u32 (column cursor /
// column length, then union-find parent) and the slot's column start (u16).
template <bool kUnion, int kP2Threads, int kMinBlocks>
__global__ void __launch_bounds__(kP2Threads, kMinBlocks) k_bkt_sort(const u64* kin, const u32* vin,
                                                                     const u32* rs, const u64* n_p,
                                                                     u32 shift,
                                                                     const u32* col_off, u32 bits_y,
                                                                     u64* skey, u32* perm,
                                                                     u32* parent, u32* size) {
    const u32 nbkt = (u32)((*n_p + (1ull << shift) - 1) >> shift);
    constexpr u32 kP2Cap = kP2Threads * kP2Items;
    extern __shared__ u64 sh_p2[];
    u64* sk = sh_p2;
    u32* sp = (u32*)(sk + kP2Cap);
    u32* aux = sp + kP2Cap;
    unsigned short* cst = (unsigned short*)(aux + kP2Cap);
    const u32 tid = threadIdx.x;
    for (u32 b = blockIdx.x; b < nbkt; b += gridDim.x) {
        const u32 r0 = rs[b], r1 = rs[b + 1];
        const u32 m = r1 - r0;
        // (a bucket holds whole columns, < 4096 + the longest column: a launch
        // that did not wait for the longest column's length must not trust it;
        // the host sees max_col with the final counters and redoes K3 then)
        if (m > kP2Cap) continue;
        for (u32 j = tid; j < m; j += kP2Threads) aux[j] = 0;
        // all of this thread's keys, perms and column starts in flight together
        u64 kk[kP2Items];
        u32 pp[kP2Items], cs[kP2Items];
#pragma unroll
        for (int q = 0; q < kP2Items; ++q) {
            const u32 j = tid + q * kP2Threads;
            if (j < m) {
                kk[q] = kin[r0 + j];
                pp[q] = vin[r0 + j];
            }
        }
#pragma unroll
        for (int q = 0; q < kP2Items; ++q) {
            const u32 j = tid + q * kP2Threads;
            if (j < m) cs[q] = __ldg(col_off + (kk[q] >> bits_y)) - r0;
        }
        __syncthreads();
        // place by column (order inside a column arbitrary); the cursor ends
        // as the column's length
#pragma unroll
        for (int q = 0; q < kP2Items; ++q) {
            const u32 j = tid + q * kP2Threads;
            if (j < m) {
                const u32 slot = cs[q] + atomicAdd(&aux[cs[q]], 1u);
                sk[slot] = kk[q];
                sp[slot] = pp[q];
                cst[slot] = (unsigned short)cs[q];
            }
        }
        __syncthreads();
        // rank inside the column (columns are short: at most kBktMaxCol);
        // rows compared as u32 words, four per step
#pragma unroll
        for (int q = 0; q < kP2Items; ++q) {
            const u32 j = tid + q * kP2Threads;
            if (j < m) {
                const u64 k = sk[j];
                const u32 s = cst[j], e = s + aux[s];
                u32 rank = 0;
                if (bits_y <= 32) {
                    const u32* lo = reinterpret_cast<const u32*>(sk);
                    const u32 y = (u32)k;
                    u32 t = s;
                    for (; t + 4 <= e; t += 4)
                        rank += (lo[2 * t] < y) + (lo[2 * t + 2] < y) + (lo[2 * t + 4] < y) +
                                (lo[2 * t + 6] < y);
                    for (; t < e; ++t) rank += lo[2 * t] < y;
                } else {
                    for (u32 t = s; t < e; ++t) rank += sk[t] < k;
                }
                kk[q] = k;
                pp[q] = sp[j];
                cs[q] = s + rank;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kP2Items; ++q) {
            const u32 j = tid + q * kP2Threads;
            if (j < m) {
                sk[cs[q]] = kk[q];
                sp[cs[q]] = pp[q];  // cst[] is unchanged: same column
            }
        }
        __syncthreads();
        for (u32 j = tid; j < m; j += kP2Threads) {
            skey[r0 + j] = sk[j];
            perm[r0 + j] = sp[j];
        }
        if (kUnion) {
            __syncthreads();
            // Chebyshev delta 1 inside the bucket: (x, y+1) is the next
            // entry of the same column; column x+1, when it is in this
            // bucket, is the run right after column x. Diagonals made
            // redundant by an orthogonal neighbour are skipped (see
            // k_sorted_union_c1), which leaves at most two forward partners
            // per tile. Partners are found first (the searches stay
            // converged) and packed into sp: two 16-bit local indices,
            // 0xffff = none. Column x+1 in the next bucket is P3's.
            // A vertical run (consecutive rows of one column) is one set from
            // the start: every tile's initial parent is its run's first
            // tile, so only the horizontal / diagonal edges need unions.
            for (u32 j = tid; j < m; j += kP2Threads) {
                const u64 k = sk[j];
                const u32 s = cst[j], e = s + aux[s];
                const bool up = j + 1 < e && sk[j + 1] == k + 1;
                u32 h = j;
                while (h > s && sk[h - 1] == sk[h] - 1) --h;
                u32 pa = 0xffffu, pb = 0xffffu;
                const u64 nxk = k + (1ull << bits_y);
                if (e < m && (sk[e] >> bits_y) == (nxk >> bits_y)) {
                    const u32 ne = e + aux[e];
                    const u64 y = k & ((1ull << bits_y) - 1);
                    const u64 lo = y > 0 ? nxk - 1 : nxk;
                    u32 a = e, bb = ne;
                    while (a < bb) {
                        const u32 mid = (a + bb) >> 1;
                        if (sk[mid] < lo) a = mid + 1;
                        else bb = mid;
                    }
                    u32 dm = 0xffffu, d0 = 0xffffu, dp = 0xffffu;
                    const u32 stop = min(ne, a + 3);
                    for (u32 t = a; t < stop; ++t) {
                        const u64 kt = sk[t];
                        if (kt == nxk - 1 && y > 0) dm = t;
                        else if (kt == nxk) d0 = t;
                        else if (kt == nxk + 1) dp = t;
                    }
                    if (d0 != 0xffffu) {
                        if (pa == 0xffffu) pa = d0;
                        else pb = d0;
                    } else {
                        if (dm != 0xffffu) {
                            if (pa == 0xffffu) pa = dm;
                            else pb = dm;
                        }
                        if (dp != 0xffffu && !up) {
                            if (pa == 0xffffu) pa = dp;
                            else pb = dp;
                        }
                    }
                }
                sp[j] = pa | (pb << 16);
                cst[j] = (unsigned short)h;  // only this thread reads cst[j] here
            }
            __syncthreads();
            for (u32 j = tid; j < m; j += kP2Threads) aux[j] = cst[j];
            __syncthreads();
            // warp-uniform trip counts with a reconvergence point per
            // round: divergent find loops must not split the warp for the
            // rest of the bucket
            for (u32 j0 = 0; j0 < m; j0 += kP2Threads) {
                const u32 j = j0 + tid;
                if (j < m) {
                    const u32 e = sp[j];
                    if ((e & 0xffffu) != 0xffffu) l_unite_h(aux, j, e & 0xffffu);
                    if ((e >> 16) != 0xffffu) l_unite_h(aux, j, e >> 16);
                }
                __syncwarp();
            }
            __syncthreads();
            // flatten; tiles per bucket-local root (sp is free now: perm is
            // written, partners consumed). Points per cluster are not part of
            // the clustering (Cluster agglomerate.hpp:18-23 has none): they
            // are summed on demand by rg_get_clusters.
            for (u32 j = tid; j < m; j += kP2Threads) sp[j] = 0;
            __syncthreads();
            for (u32 j0 = 0; j0 < m; j0 += kP2Threads) {
                const u32 j = j0 + tid;
                if (j < m) {
                    const u32 r = l_find_h(aux, j);
                    parent[r0 + j] = r0 + r;
                    atomicAdd(&sp[r], 1u);
                }
                __syncwarp();
            }
            __syncthreads();
            for (u32 j = tid; j < m; j += kP2Threads)
                if (aux[j] == j) size[r0 + j] = sp[j];
        }
        __syncthreads();
    }
}

// Edges between the last column of bucket b and the first column of bucket
// b+1 (Chebyshev delta 1, all three offsets; no elision needed).
__global__ void k_bkt_cross(const u64* skey, const u32* rs, const u64* n_p, u32 shift,
                            const u32* col_off, u64 cols, u32 bits_y, u32* parent, u32* linked,
                            u64* n_linked) {
    const u32 nbkt = (u32)((*n_p + (1ull << shift) - 1) >> shift);
    const int lane = threadIdx.x & 31;
    const u64 ymask = (1ull << bits_y) - 1;
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    for (u64 b = warp; b + 1 < nbkt; b += n_warps) {
        const u32 re = rs[b + 1];
        if (re == rs[b]) continue;
        const u64 xl = skey[re - 1] >> bits_y;
        if (xl + 1 >= cols) continue;
        const u32 ns = col_off[xl + 1], ne = col_off[xl + 2];
        if (ne == ns) continue;  // column x+1 empty
        for (u32 t = col_off[xl] + lane; t < re; t += 32) {
            const u64 k = skey[t];
            const u64 y = k & ymask;
            const u64 nxk = k + (1ull << bits_y);
            const u64 lo = y > 0 ? nxk - 1 : nxk;
            u32 a = ns, bb = ne;
            while (a < bb) {
                const u32 mid = (a + bb) >> 1;
                if (skey[mid] < lo) a = mid + 1;
                else bb = mid;
            }
            for (u32 q = a; q < ne; ++q) {
                const u64 kq = skey[q];
                if (kq > nxk + 1 || (kq == nxk + 1 && y == ymask)) break;
                s_unite_rec(parent, t, q, linked, n_linked);
            }
        }
    }
}

// Fold the tile count of every bucket-local root that P3 linked
// under another root into its final root (the final root's own count is
// already there; a linked root receives nothing, so its count is its own).
__global__ void k_bkt_merge(const u32* linked, const u64* n_linked, u32* parent, u32* size,
                            u64* npts) {
    const u64 n = *n_linked;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const u32 ra = linked[i];
        const u32 f = s_find(parent, ra);
        atomicAdd(size + f, size[ra]);
    }
}

// Points per cluster on demand (after the bucketed K3, which leaves npts
// unset): npts[root of cluster k] = sum of its tiles' counts. Runs of equal
// ids within a warp are pre-summed.
__global__ void k_cluster_npts(const int* cid_s, const u32* perm, const u64* cnt_b, u64 n,
                               const u32* clu_root, u64* npts) {
    const int lane = threadIdx.x & 31;
    const u64 span = (n + 31) / 32 * 32;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < span;
         i += (u64)gridDim.x * blockDim.x) {
        const int c = i < n ? cid_s[i] : -1;
        u64 p = c >= 0 ? cnt_b[perm[i]] : 0ull;
        const int prev = __shfl_up_sync(kFull, c, 1);
        const bool head = lane == 0 || prev != c;
        const u32 heads = __ballot_sync(kFull, head);
        const u32 run = __popc(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 orun = __shfl_down_sync(kFull, run, o);
            const u64 op = __shfl_down_sync(kFull, p, o);
            if (lane + o < 32 && orun == run) p += op;
        }
        if (head && c >= 0) atomicAdd(npts + clu_root[c], p);
    }
}

cudaError_t launch_cluster_npts(const int* cid_s, const u32* perm, const u64* cnt_b, u64 n,
                                const u32* clu_root, u64 n_kept, u64* npts, int n_sm,
                                cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    // clusters' roots are sorted positions < n: clear them all
    if ((e = cudaMemsetAsync(npts, 0, n * sizeof(u64), st)) != cudaSuccess) return e;
    (void)n_kept;
    if (n == 0) return cudaSuccess;
    const u64 want = (n + 255) / 256;
    const int g = (int)std::min<u64>(want, (u64)n_sm * 16);
    k_cluster_npts<<<g, 256, 0, st>>>(cid_s, perm, cnt_b, n, clu_root, npts);
    return cudaGetLastError();
}

static int grid_for_s(u64 n, int n_sm, int per_sm) {
    const u64 want = (n + 255) / 256;
    const u64 cap = (u64)n_sm * per_sm;
    return (int)(want == 0 ? 1 : (want < cap ? want : cap));
}

u64 sorted_columns(u32 bits_x) { return bits_x <= kColBitsMax ? (1ull << bits_x) : 0; }

size_t sorted_temp_bytes(u64 n, int bits, u32 bits_x) {
    size_t a = 0, b = 0, c = 0, d = 0;
    cub::DeviceRadixSort::SortPairs((void*)nullptr, a, (const u64*)nullptr, (u64*)nullptr,
                                    (const u32*)nullptr, (u32*)nullptr, (int)n, 0, bits);
    cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const u32*)nullptr, (u32*)nullptr, (int)n);
    const u64 cols = sorted_columns(bits_x);
    if (cols) {
        cub::DeviceScan::ExclusiveSum((void*)nullptr, c, (const u32*)nullptr, (u32*)nullptr,
                                      (int)(cols + 1));
        cub::DeviceSegmentedSort::SortPairs((void*)nullptr, d, (const u64*)nullptr,
                                            (u64*)nullptr, (const u32*)nullptr, (u32*)nullptr,
                                            (int)n, (int)cols, (const u32*)nullptr,
                                            (const u32*)nullptr);
    }
    const u64 tiles = std::max<u64>((n + kLbTile - 1) / kLbTile, (cols + kCsTile) / kCsTile) + 1;
    const size_t lb = 16 + tiles * 12;  // look-back scans: ticket, status words, done flags
    return std::max(std::max(std::max(a, b), std::max(c, d)), lb);
}

// Look-back scratch at the start of the temp buffer, cleared before a scan.
struct LbScratch {
    u32* ticket;
    u64* status;
    u32* done;
};
static LbScratch lb_scratch(void* temp, u64 tiles, cudaStream_t st) {
    LbScratch r;
    r.ticket = (u32*)temp;
    r.status = (u64*)((char*)temp + 16);
    r.done = (u32*)(r.status + tiles);
    cudaMemsetAsync(temp, 0, 16 + tiles * 12, st);
    return r;
}

// Columns longer than this reach CUB's large-segment path, which sorts all 64
// key bits per segment and is slow
// (config 5's walks: 2.7 ms); such inputs take the full radix sort instead.
#ifndef RG_SEG_MAX_COLUMN
#define RG_SEG_MAX_COLUMN 128
#endif
constexpr u64 kSegSortMaxColumn = RG_SEG_MAX_COLUMN;

u64 sorted_bucket_max_column() { return kBktMaxCol; }

cudaError_t launch_agglomerate_sorted(const SortedLaunch& L, cudaStream_t st) {
    if (L.n_sig == 0) return cudaSuccess;
    cudaError_t e;
    size_t bytes = L.temp_bytes;
    const u64 cols = sorted_columns(L.key_bits - L.bits_y);
    constexpr u32 shift = 12;  // 4096-tile buckets
    if (cols && L.col_cnt) {
        cudaMemsetAsync(&L.ctr->max_col, 0, sizeof(u64), st);
        if (!L.col_hist_ready) {  // (K2 builds the histogram on the prune path)
            cudaMemsetAsync(L.col_cnt, 0, (cols + 1) * sizeof(u32), st);
            k_col_hist<<<grid_for_s(L.n_sig, L.n_sm, 16), 256, 0, st>>>(
                L.sig_key, L.n_sig_dev, L.bits_y, L.col_cnt, (u32*)&L.ctr->max_col);
        }
        // column offsets, longest column and bucket starts in one pass
        const u64 tiles = (cols + kCsTile) / kCsTile;
        const LbScratch lb = lb_scratch(L.temp, tiles, st);
        k_col_scan<<<(int)tiles, kCsThr, 0, st>>>(L.col_cnt, cols, L.n_sig_dev, shift, L.col_off,
                                                  (u32*)&L.ctr->max_col, L.flag, lb.status,
                                                  lb.ticket);
    }
    const bool c1 = L.delta == 1 && !L.manhattan;
    static const int variant = [] {
        const char* v = std::getenv("RG_K3_SORT");
        return v && v[0] == 's' ? 1 : (v && v[0] == 'r' ? 2 : 0);
    }();
    // Without the host read (L.speculate): every launch is sized for the
    // bound L.n_sig, the kernels read the exact count on the device, and the
    // bucketed path is taken on the assumption that no column is longer than
    // kBktMaxCol; the caller checks max_col (and K1's stop flag) in the
    // counters it reads at the end of the call and redoes K3 otherwise.
    const bool spec = L.speculate && c1 && cols && L.col_cnt && variant == 0 &&
                      (size_t)(((L.n_sig + (1ull << shift) - 1) >> shift) + 1) * 8 <= 96 * 1024;
    if (L.speculated) *L.speculated = spec;
    if (spec) {
        // nothing to wait for
    } else if (L.check_k1_stop) {  // K1's counters ride along (its stop check was deferred)
        if ((e = cudaMemcpyAsync(L.host_ctr, L.ctr, sizeof(Counters), cudaMemcpyDeviceToHost,
                                 st)) != cudaSuccess)
            return e;
    } else if ((e = cudaMemcpyAsync(&L.host_ctr->n_sig, &L.ctr->n_sig,
                                    sizeof(Counters) - offsetof(Counters, n_sig),
                                    cudaMemcpyDeviceToHost, st)) != cudaSuccess) {
        return e;
    }
    if (!spec && (e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if (!spec && L.check_k1_stop && L.host_ctr->stopped) {
        if (L.launches) *L.launches = cols && L.col_cnt ? (L.col_hist_ready ? 1 : 2) : 0;
        return cudaErrorNotReady;
    }
    const u64 n = spec ? L.n_sig : L.host_ctr->n_sig;  // (an upper bound when speculating)
    if (!spec && std::getenv("RG_DEBUG"))
        std::fprintf(stderr, "[rg] K3 sorted: n=%llu max_col=%llu\n", (unsigned long long)n,
                     (unsigned long long)L.host_ctr->max_col);
    if (n == 0) {
        if (L.launches) *L.launches = cols && L.col_cnt ? (L.col_hist_ready ? 1 : 2) : 0;
        return cudaSuccess;
    }
    const int gs = grid_for_s(n, L.n_sm, 16);
    int launches = cols && L.col_cnt ? (L.col_hist_ready ? 1 : 2) : 0;  // col_hist, col_scan
    const u64 mcol = spec ? 0 : L.host_ctr->max_col;
    const u32 nbkt = (u32)((n + (1ull << shift) - 1) >> shift);
    bool bucket_counts = false;  // per-root counts already final (bucketed Chebyshev-1 path)
    if (cols && L.col_cnt && variant == 0 && mcol <= kBktMaxCol &&
        (size_t)nbkt * 8 <= 96 * 1024) {  // L.flag holds >= 1024 and >= n entries
        // bucketed column sort (+ fused bucket-local unions for Chebyshev 1);
        // k_col_scan left the bucket starts and the scatter cursors in flag
        u32* rs = L.flag;  // nbkt + 1 region starts, then nbkt scatter cursors
        const size_t sm1 = (size_t)nbkt * 2 * sizeof(u32);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_bkt_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 96 * 1024 + 1024);
            cudaFuncSetAttribute(k_bkt_sort<true, 512, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p2_smem(512));
            cudaFuncSetAttribute(k_bkt_sort<false, 512, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p2_smem(512));
            attr = true;
        }
        const u64 t1 = (n + kP1Tile - 1) / kP1Tile;
        const int g1 = (int)std::min<u64>(t1, (u64)L.n_sm * (2048 / kP1Threads));
        k_bkt_scatter<<<g1, kP1Threads, sm1, st>>>(L.sig_key, L.n_sig_dev, L.bits_y, L.col_off, rs,
                                                   nbkt, shift, L.ktmp, L.iota);
        const int g2 = (int)std::min<u64>(nbkt, (u64)L.n_sm * 2);
        auto p2 = [&](auto kernel, int threads) {
            kernel<<<g2, threads, p2_smem(threads), st>>>(L.ktmp, L.iota, rs, L.n_sig_dev, shift,
                                                          L.col_off, L.bits_y, L.skey, L.perm,
                                                          L.parent, L.size);
        };
        if (c1) {
            p2(k_bkt_sort<true, 512, 2>, 512);
            launches += 2;  // scatter, sort
            if (nbkt > 1) {
                u32* linked = reinterpret_cast<u32*>(L.edges);  // >= 2n u32 entries
                cudaMemsetAsync(&L.ctr->n_edges, 0, sizeof(u64), st);
                k_bkt_cross<<<(int)std::min<u64>((nbkt + 7) / 8, (u64)L.n_sm * 8), 256, 0, st>>>(
                    L.skey, rs, L.n_sig_dev, shift, L.col_off, cols, L.bits_y, L.parent, linked,
                    &L.ctr->n_edges);
                k_bkt_merge<<<L.n_sm, 256, 0, st>>>(linked, &L.ctr->n_edges, L.parent, L.size,
                                                    L.npts);
                launches += 2;
            }
            bucket_counts = true;
            if (L.npts_deferred) *L.npts_deferred = true;
        } else {
            p2(k_bkt_sort<false, 512, 2>, 512);
            launches += 2;
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (!c1) {
            SortedEdges el{L.edges, L.edge_cap, &L.ctr->n_edges};
            cudaMemsetAsync(&L.ctr->n_edges, 0, sizeof(u64), st);
            k_sorted_union<<<gs, 256, 0, st>>>(L.skey, L.n_sig_dev, L.bits_y, L.delta,
                                               L.manhattan, L.parent, L.size, L.npts, el);
            k_sorted_edges<<<gs, 256, 0, st>>>(el, L.parent);
            launches += 2;
        }
    } else {
        if (cols && L.col_cnt && variant != 2 && L.host_ctr->max_col <= kSegSortMaxColumn) {
            cudaMemcpyAsync(L.col_cnt, L.col_off, (cols + 1) * sizeof(u32),
                            cudaMemcpyDeviceToDevice, st);
            k_col_scatter<<<gs, 256, 0, st>>>(L.sig_key, L.n_sig_dev, L.bits_y, L.col_cnt, L.ktmp,
                                              L.iota);
            bytes = L.temp_bytes;
            e = cub::DeviceSegmentedSort::SortPairs(L.temp, bytes, L.ktmp, L.skey, L.iota, L.perm,
                                                    (int)n, (int)cols, L.col_off, L.col_off + 1,
                                                    st);
            if (e != cudaSuccess) return e;
            launches += 5;  // scatter, segmented sort (4)
        } else {
            e = launch_iota(L.iota, n, L.n_sm, st);
            if (e != cudaSuccess) return e;
            e = cub::DeviceRadixSort::SortPairs(L.temp, bytes, L.sig_key, L.skey, L.iota, L.perm,
                                                (int)n, 0, (int)L.key_bits, st);
            if (e != cudaSuccess) return e;
            launches += 1 + 2 * (((int)L.key_bits + 7) / 8) + 1;  // iota + onesweep passes
        }
        SortedEdges el{L.edges, L.edge_cap, &L.ctr->n_edges};
        cudaMemsetAsync(&L.ctr->n_edges, 0, sizeof(u64), st);
        if (c1)
            k_sorted_union_c1<<<gs, 256, 0, st>>>(L.skey, L.n_sig_dev, L.bits_y, L.parent, L.size,
                                                  L.npts, el);
        else
            k_sorted_union<<<gs, 256, 0, st>>>(L.skey, L.n_sig_dev, L.bits_y, L.delta,
                                               L.manhattan, L.parent, L.size, L.npts, el);
        k_sorted_edges<<<gs, 256, 0, st>>>(el, L.parent);
        launches += 2;
    }
    if (!bucket_counts) {  // flatten + per-root counts (the bucketed union did both)
        k_sorted_reduce<<<gs, 256, 0, st>>>(L.parent, L.perm, L.sig_cnt, L.n_sig_dev, L.size,
                                            L.npts, L.flag, L.mu);
        ++launches;
    }
    {
        // (four short passes instead - count, scan, root ids, labels - with
        // ballot bitmaps measured 128 us against this kernel's 119 us)
        const u64 tiles = (n + kLbTile - 1) / kLbTile;
        const LbScratch lb = lb_scratch(L.temp, tiles, st);
        k_sorted_ids<<<(int)tiles, kLbThr, 0, st>>>(L.parent, L.size, L.mu, L.perm, L.n_sig_dev,
                                                    L.tile_cid_b, L.cid_s, L.clu_root, L.ctr,
                                                    lb.status, lb.done, lb.ticket);
        launches += 1;
    }
    if (L.launches) *L.launches = launches;
    return cudaGetLastError();
}

}  // namespace rg
