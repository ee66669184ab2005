// contract.cu — K1 (contraction) and K2 (compaction) for sm_100a.
//
// K1 replaces the reference's hot loop TileAccumulator::ingest
// (accumulator.hpp:120-134: Bounds::contains core.hpp:33-35 ->
// project_unchecked core.hpp:136-139 -> TileCounts::add accumulator.hpp:33-50).
//
// Work decomposition. Points are processed in rows of 32 (one point per lane,
// one coalesced 512-byte warp load) grouped into segments of consecutive
// rows. Warps pull segments from a global ticket counter (the next ticket is
// prefetched one segment ahead so the atomic's latency is hidden), so hot
// spots (config 5's blob) and cold regions load-balance dynamically.
//
// Aggregation. Per row the warp groups equal keys with __match_any_sync; each
// distinct key's leader lane merges the group's count into a per-warp
// direct-mapped write-back cache in shared memory (128 entries; slot
// ownership per row is arbitrated through a shared-memory owner byte, so no
// shared-memory atomics are needed). Entries reach the HBM table only when
// evicted or at the end, so a run of points from one cluster costs one global
// RED per distinct tile rather than one per point.
//
// Growth without a device-side rehash in the loop. The reference grows its
// table at 70% load (accumulator.hpp:34,84-94). Here each launch gives every
// warp a budget of new keys (host-computed from the table's free space); a
// warp whose (claimed keys + cached entries) reaches its budget records where
// it stopped and exits. The host then rehashes into a larger table and
// resumes exactly the unprocessed rows, so results are identical to a single
// pass regardless of how often the table grew.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "internal.h"

namespace rg {

constexpr int kWarpsPerBlock = 8;
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr int kCacheSlots = 128;
constexpr int kBatch = 4;

struct K1Params {
    const double* xy;
    u64 n;
    u64 n_rows;
    u64 rows_per_seg;
    u64 n_seg;
    Grid g;
    Table t;
    Counters* ctr;
    const Partial* partial_in;
    u64 n_partial_in;
    Partial* partial_out;
    u64 budget;
};

__device__ __forceinline__ u32 cache_slot(u64 key) {
    return (u32)((key * 0xD6E8FEB86659FD93ull) >> (64 - 7));
}

template <bool kAligned>
__device__ __forceinline__ void load_point(const double* xy, u64 idx, u64 n, u64 pol,
                                           double& x, double& y) {
    if (idx < n) {
        if (kAligned) {
            const double2 v = ld_point_stream(reinterpret_cast<const double2*>(xy) + idx, pol);
            x = v.x;
            y = v.y;
        } else {
            x = xy[2 * idx];
            y = xy[2 * idx + 1];
        }
    } else {
        x = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not in bounds
        y = x;
    }
}

template <bool kAligned>
__global__ void __launch_bounds__(kThreads) k_contract(K1Params P) {
    __shared__ u64 s_key[kWarpsPerBlock][kCacheSlots];
    __shared__ u64 s_cnt[kWarpsPerBlock][kCacheSlots];
    __shared__ unsigned char s_owner[kWarpsPerBlock][kCacheSlots];

    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    u64* ckey = s_key[wib];
    u64* ccnt = s_cnt[wib];
    unsigned char* owner = s_owner[wib];
    for (int i = lane; i < kCacheSlots; i += 32) ckey[i] = kEmpty;
    __syncwarp();

    const Grid& g = P.g;
    const u64 pol = evict_first_policy();
    u64 claimed = 0;  // warp-uniform: keys this warp claimed in the table
    u32 occ = 0;      // warp-uniform: occupied cache entries
    u64 n_in = 0, n_out = 0;  // per lane
    bool stopped = false;

    // Work queue: first the partial segments of a previous (stopped)
    // launch, then fresh tickets.
    auto fetch = [&](u64& seg, u64& row0) -> bool {
        if (P.n_partial_in) {
            u64 pt = 0;
            if (lane == 0) pt = atomicAdd(&P.ctr->partial_ticket, 1ull);
            pt = __shfl_sync(kFull, pt, 0);
            if (pt < P.n_partial_in) {
                seg = P.partial_in[pt].segment;
                row0 = P.partial_in[pt].next_row;
                return true;
            }
        }
        u64 t = 0;
        if (lane == 0) t = atomicAdd(&P.ctr->ticket, 1ull);
        t = __shfl_sync(kFull, t, 0);
        if (t >= P.n_seg) return false;
        seg = t;
        row0 = t * P.rows_per_seg;
        return true;
    };
    auto record_partial = [&](u64 seg, u64 row) {
        if (lane == 0) {
            const u64 at = atomicAdd(&P.ctr->n_partial, 1ull);
            P.partial_out[at].segment = seg;
            P.partial_out[at].next_row = row;
        }
    };

    u64 seg, row0;
    bool have = fetch(seg, row0);
    while (have && !stopped) {
        const u64 row_end = min((seg + 1) * P.rows_per_seg, P.n_rows);
        for (u64 r = row0; r < row_end; r += kBatch) {
            double xs[kBatch], ys[kBatch];
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                const u64 row = r + b;
                const u64 idx = row * 32 + lane;
                load_point<kAligned>(P.xy, row < row_end ? idx : P.n, P.n, pol, xs[b], ys[b]);
            }
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                const u64 row = r + b;
                if (row >= row_end) break;
                const u64 idx = row * 32 + lane;
                const bool valid = idx < P.n;
                const bool inb = in_bounds(g, xs[b], ys[b]);
                n_in += inb;
                n_out += (valid && !inb);
                const u64 key = inb ? pack_key(g, xs[b], ys[b]) : kEmpty;
                const u32 peers = __match_any_sync(kFull, key);
                const bool leader = inb && (lane == __ffs(peers) - 1);
                const u32 cs = cache_slot(key);
                if (leader) owner[cs] = (unsigned char)lane;
                __syncwarp();
                u32 delta = 0;  // low 16: claimed keys, high 16: new cache entries
                if (leader) {
                    const u64 cnt = __popc(peers);
                    if (owner[cs] == lane) {
                        const u64 ek = ckey[cs];
                        if (ek == key) {
                            ccnt[cs] += cnt;
                        } else {
                            if (ek != kEmpty) {
                                delta += table_add(P.t, ek, ccnt[cs]) ? 1u : 0u;
                            } else {
                                delta += 1u << 16;
                            }
                            ckey[cs] = key;
                            ccnt[cs] = cnt;
                        }
                    } else {
                        delta += table_add(P.t, key, cnt) ? 1u : 0u;
                    }
                }
                __syncwarp();
                const u32 sum = __reduce_add_sync(kFull, delta);
                claimed += sum & 0xffffu;
                occ += sum >> 16;
                if (claimed + occ >= P.budget) {
                    // Out of budget: hand the rest of this segment back.
                    if (row + 1 < row_end) record_partial(seg, row + 1);
                    stopped = true;
                    break;
                }
            }
            if (stopped) break;
        }
        if (!stopped) have = fetch(seg, row0);
    }

    // Write back the cache.
    u32 fl = 0;
    for (int i = lane; i < kCacheSlots; i += 32) {
        const u64 k = ckey[i];
        if (k != kEmpty) fl += table_add(P.t, k, ccnt[i]) ? 1u : 0u;
    }
    claimed += __reduce_add_sync(kFull, fl);

    // Counters: one atomic per warp.
    const u64 wi = __reduce_add_sync(kFull, (u32)n_in);  // < 2^32 per warp per launch
    const u64 wo = __reduce_add_sync(kFull, (u32)n_out);
    if (lane == 0) {
        if (wi) atomicAdd(&P.ctr->ingested, wi);
        if (wo) atomicAdd(&P.ctr->skipped, wo);
        if (claimed) atomicAdd(&P.ctr->used, claimed);
        if (stopped) atomicAdd(&P.ctr->stopped, 1ull);
    }
}

// Fill a table with {EMPTY, 0}.
__global__ void k_table_clear(Slot* slots, u64 n) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        Slot s;
        s.key = kEmpty;
        s.count = 0;
        slots[i] = s;
    }
}

// Rehash (TileCounts::grow accumulator.hpp:84-94) or merge
// (TileAccumulator::merge accumulator.hpp:137-154): fold every occupied slot
// of `src` into `dst`. Returns newly claimed keys in *claimed.
__global__ void k_table_fold(const Slot* src, u64 n_src, Table dst, u64* claimed) {
    u32 local = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n_src;
         i += (u64)gridDim.x * blockDim.x) {
        u64 k, v;
        ld_slot(src + i, k, v);
        if (k != kEmpty) local += table_add(dst, k, v) ? 1u : 0u;
    }
    const u32 w = __reduce_add_sync(kFull, local);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(claimed, (u64)w);
}

// Strict policy pre-pass: smallest index of an out-of-bounds point.
__global__ void k_first_oob(const double* xy, u64 n, Grid g, u64* first) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (!in_bounds(g, x, y)) {
            atomicMin(first, i);
            return;  // later indices of this thread are larger
        }
    }
}

// K2: TileAccumulator::prune accumulator.hpp:160-174 — keep count >= tau.
// Each significant slot gets a dense index (block-aggregated append), its
// key/count are written to the compact arrays, the slot's value word becomes
// SIG_BIT | index and the union-find parent is initialised.
constexpr int kK2Items = 4;
__global__ void __launch_bounds__(256) k_compact(Table t, u64 cap, u64 tau, u64* sig_key,
                                                 u64* sig_cnt, u32* parent, Counters* ctr) {
    __shared__ u32 s_warp[8];
    __shared__ u64 s_base;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const u64 per_block = 256ull * kK2Items;
    for (u64 base = blockIdx.x * per_block; base < cap; base += (u64)gridDim.x * per_block) {
        u64 k[kK2Items], v[kK2Items];
        u32 nsig = 0;
#pragma unroll
        for (int j = 0; j < kK2Items; ++j) {
            const u64 i = base + j * 256 + threadIdx.x;
            if (i < cap) {
                ld_slot(t.slots + i, k[j], v[j]);
            } else {
                k[j] = kEmpty;
                v[j] = 0;
            }
            nsig += (k[j] != kEmpty && v[j] >= tau);
        }
        // block-exclusive scan of nsig
        u32 incl = nsig;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[wib] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            u32 tot = 0;
            for (int w = 0; w < 8; ++w) {
                const u32 c = s_warp[w];
                s_warp[w] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(&ctr->n_sig, (u64)tot) : 0;
        }
        __syncthreads();
        u64 pos = s_base + s_warp[wib] + incl - nsig;
#pragma unroll
        for (int j = 0; j < kK2Items; ++j) {
            if (k[j] != kEmpty && v[j] >= tau) {
                const u64 i = base + j * 256 + threadIdx.x;
                sig_key[pos] = k[j];
                sig_cnt[pos] = v[j];
                parent[pos] = (u32)pos;
                t.slots[i].count = kSigBit | pos;
                ++pos;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers

static int g_k1_blocks_per_sm[2] = {0, 0};

int contract_max_warps(int n_sm) {
    if (!g_k1_blocks_per_sm[1]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k1_blocks_per_sm[1], k_contract<true>,
                                                      kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_k1_blocks_per_sm[0], k_contract<false>,
                                                      kThreads, 0);
        if (g_k1_blocks_per_sm[1] < 1) g_k1_blocks_per_sm[1] = 1;
        if (g_k1_blocks_per_sm[0] < 1) g_k1_blocks_per_sm[0] = 1;
    }
    return g_k1_blocks_per_sm[1] * n_sm * kWarpsPerBlock;
}

cudaError_t launch_contract(const ContractLaunch& L, cudaStream_t st) {
    K1Params P;
    P.xy = L.xy;
    P.n = L.n;
    P.n_rows = (L.n + 31) / 32;
    P.rows_per_seg = L.rows_per_seg;
    P.n_seg = (P.n_rows + L.rows_per_seg - 1) / L.rows_per_seg;
    P.g = L.g;
    P.t = L.t;
    P.ctr = L.ctr;
    P.partial_in = L.partial_in;
    P.n_partial_in = L.n_partial_in;
    P.partial_out = L.partial_out;
    P.budget = L.budget;
    const int blocks = (int)((L.warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const bool aligned = ((uintptr_t)L.xy & 15) == 0;
    if (aligned)
        k_contract<true><<<blocks, kThreads, 0, st>>>(P);
    else
        k_contract<false><<<blocks, kThreads, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_table_clear(Slot* slots, u64 n, int n_sm, cudaStream_t st) {
    const u64 want = (n + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? (want ? want : 1) : (u64)n_sm * 16);
    k_table_clear<<<blocks, 256, 0, st>>>(slots, n);
    return cudaGetLastError();
}

cudaError_t launch_table_fold(const Slot* src, u64 n_src, Table dst, u64* claimed, int n_sm,
                              cudaStream_t st) {
    const u64 want = (n_src + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? (want ? want : 1) : (u64)n_sm * 16);
    k_table_fold<<<blocks, 256, 0, st>>>(src, n_src, dst, claimed);
    return cudaGetLastError();
}

cudaError_t launch_first_oob(const double* xy, u64 n, Grid g, u64* first, int n_sm,
                             cudaStream_t st) {
    const u64 want = (n + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 8 ? (want ? want : 1) : (u64)n_sm * 8);
    k_first_oob<<<blocks, 256, 0, st>>>(xy, n, g, first);
    return cudaGetLastError();
}

cudaError_t launch_compact(Table t, u64 cap, u64 tau, u64* sig_key, u64* sig_cnt, u32* parent,
                           Counters* ctr, int n_sm, cudaStream_t st) {
    const u64 per_block = 256ull * kK2Items;
    const u64 want = (cap + per_block - 1) / per_block;
    const int blocks = (int)(want < (u64)n_sm * 8 ? (want ? want : 1) : (u64)n_sm * 8);
    k_compact<<<blocks, 256, 0, st>>>(t, cap, tau, sig_key, sig_cnt, parent, ctr);
    return cudaGetLastError();
}

}  // namespace rg
