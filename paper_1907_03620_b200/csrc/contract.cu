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
// Staging. Each warp keeps a ring of rows in flight with per-lane 16-byte
// cp.async copies (L2 evict-first). A TMA bulk-copy ring (one elected lane,
// one cp.async.bulk + mbarrier per 2-row stage) is built too (RG_K1=tma);
// it measured slower (K1).
//
// Aggregation. Every lane looks its tile up in a per-warp direct-mapped
// write-back cache in shared memory (128 entries, slot = position in an
// 8 x 16-tile window, so the tiles of one cluster never evict each other); a
// hit is one shared-memory increment. Misses of a whole batch of rows are
// resolved together: one missing point per slot wins it (owner byte),
// evicts the old entry into a staging list and installs its tile; the
// staging list is written to the HBM table 32 entries at a time by the
// whole warp (CAS-first claims, RED adds). A run of points from one cluster
// therefore costs about one global update per distinct tile.
//
// Growth without a device-side rehash in the loop. The reference grows its
// table at 70% load (accumulator.hpp:34,84-94). Here each launch gives every
// warp a budget of new keys (host-computed from the table's free space); a
// warp whose (claimed keys + cached entries) reaches its budget records where
// it stopped and exits. The host then rehashes into a larger table and
// resumes exactly the unprocessed rows, so results are identical to a single
// pass regardless of how often the table grew.
#include <cub/device/device_radix_sort.cuh>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace rg {

#ifndef RG_K1_WARPS
#define RG_K1_WARPS 4
#endif
constexpr int kWarpsPerBlock = RG_K1_WARPS;
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr int kCacheSlots = 128;
#ifndef RG_K1_BATCH
#define RG_K1_BATCH 2
#endif
#ifndef RG_K1_MINBLOCKS
#define RG_K1_MINBLOCKS 8
#endif
constexpr int kBatch = RG_K1_BATCH;  // rows per batch; the next batch is prefetched while one is processed

struct K1Params {
    const double* xy;
    u64 n;
    u64 n_rows;
    u64 rows_per_seg;  // multiple of kBatch
    u64 n_seg;
    Grid g;
    Table t;
    Counters* ctr;
    const Partial* partial_in;
    u64 n_partial_in;
    Partial* partial_out;
    u32 budget;  // per-warp bound on (claimed keys + cached entries)
};

// Per-warp shared state of K1.
// Staging list: flushed once more than kStageCap - 32 entries wait (a row
// adds at most 32).
#ifndef RG_K1_STAGE
#define RG_K1_STAGE (64 + 32 * RG_K1_BATCH)
#endif
constexpr u32 kStageCap = RG_K1_STAGE;

typedef u32 CacheCount;  // bounded by the per-segment overflow check in k_contract

struct WarpSmem {
    u64 ckey[kCacheSlots];          // direct-mapped write-back cache: cache keys
    CacheCount ccnt[kCacheSlots];   //                                 counts
    u64 skey[kStageCap];     // staged (table key, count) pairs bound for the HBM table
    u32 scnt[kStageCap];     // (cache counts stay below 2^31 + 8192, see k_contract)
    unsigned char owner[kCacheSlots];
};

struct K1State {
    u32 pot;      // warp-uniform: bound on claimed keys + cache entries + staged entries
    u32 slen;     // warp-uniform: staged entries (some may be placeholders)
    u32 claims;   // per lane: keys this lane claimed in the table
    u64 added;    // per lane: points this lane added to the table (= ingested, by conservation)
};

// Flush the staging list with every lane active: one table_add per entry,
// lanes in parallel (the divergent, latency-bound part of a miss is paid
// once per 32 misses instead of once per row). Placeholder entries (a miss
// that filled an empty cache slot reserved one) carry kEmpty and are skipped.
template <bool kC128 = false>
__device__ __forceinline__ void flush_stage(const Table& t, WarpSmem& w, K1State& s, int lane) {
    u32 c = 0, ph = 0;
    for (u32 e = lane; e < s.slen; e += 32) {
        const u64 k = w.skey[e];
        if (k != kEmpty) {
#ifdef RG_K1_NOFLUSH  // experiment: drop evictions (results are wrong)
            c += (w.scnt[e] == 12345) ? 1u : 0u;
#else
            // (claim-heavy inputs install key and count with one 128-bit CAS)
            c += (kC128 ? table_add_cas128(t, k, w.scnt[e]) : table_add_cas(t, k, w.scnt[e])) ? 1u : 0u;
#endif
            s.added += w.scnt[e];
        } else {
            ++ph;
        }
    }
    // (claimed keys) | (placeholders << 16); slen <= kStageCap
    const u32 r = __reduce_add_sync(kFull, c | (ph << 16));
    s.claims += c;
    // a placeholder's cache entry stays in the cache: it keeps its unit
    s.pot = s.pot - (s.slen - (r >> 16)) + (r & 0xffffu);
    s.slen = 0;
    __syncwarp();
}

#ifdef RG_K1_ROWWISE
// One batch of kBatch rows already in registers (one point per lane per
// row). Every lane looks its tile up in the per-warp cache; a hit adds 1
// with a shared-memory reduction (fire-and-forget: the warp does not wait,
// and lanes of one tile serialise inside the shared-memory atomic unit
// instead of in a match/leader/add chain). Misses are resolved per slot:
// one missing lane wins the slot, evicts the old occupant into the staging
// list (or leaves a placeholder if the slot was empty) and installs its key
// with count 0; then every missing lane whose key now owns its slot adds
// 1, and the others (a different key won the slot in this row) stage
// (key, 1) themselves.
template <bool kNarrow, bool kPf, bool kC128>
__device__ __forceinline__ bool process_batch(const Grid& g, const Table& t, const double* x,
                                              const double* y, WarpSmem& w, K1State& s,
                                              int lane, u32 lt_mask, u32 budget) {
    using K = KeyOps<kNarrow>;
    u64 key[kBatch];
    u32 cs[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
        key[b] = K::cache_key(g, x[b], y[b]);
        cs[b] = K::slot(key[b], g.bits_y);
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
        const bool valid = key[b] != kEmpty;
        const bool hit = valid && w.ckey[cs[b]] == key[b];
        if (hit) atomicAdd(&w.ccnt[cs[b]], 1u);
        const bool miss = valid && !hit;
        const u32 missmask = ballot(miss);
        if (missmask) {
            if (miss) w.owner[cs[b]] = (unsigned char)lane;
            __syncwarp();
            const bool win = miss && w.owner[cs[b]] == lane;
            u64 sk = kEmpty, sc = 0;
            if (win) {
                sk = K::table_key(w.ckey[cs[b]], g.bits_y);  // kEmpty: placeholder
                sc = w.ccnt[cs[b]];
                w.ckey[cs[b]] = key[b];
                w.ccnt[cs[b]] = 0;
            }
            __syncwarp();
            bool lose = false;
            if (miss) {
                if (w.ckey[cs[b]] == key[b]) {
                    atomicAdd(&w.ccnt[cs[b]], 1u);
                } else {
                    lose = true;
                    sk = K::table_key(key[b], g.bits_y);
                    sc = 1;
                }
            }
            // each winner and each loser adds one to (cache + staged entries)
            const u32 smask = ballot(win || lose);
            if (win || lose) {
                const u32 pos = s.slen + __popc(smask & lt_mask);
                w.skey[pos] = sk;
                w.scnt[pos] = sc;
            }
            const u32 ns = __popc(smask);
            s.slen += ns;
            s.pot += ns;
            __syncwarp();
            if (s.slen > kStageCap - 32 * kBatch) flush_stage<kC128>(t, w, s, lane);
        }
    }
    return s.pot >= budget;
}
#else
// One batch of kBatch rows already in registers (one point per lane per
// row). Every lane looks its tiles up in the per-warp cache; a hit adds 1
// with a shared-memory increment (fire-and-forget: the warp does not wait,
// and lanes of one tile are aggregated in the shared-memory atomic unit).
// The lookups are branch-free: the bounds test stays a predicate (an
// out-of-bounds point's key is never materialised or compared against the
// sentinel; its slot is still a valid index). Misses of ALL rows of the batch
// are then resolved together, per slot: one missing (lane, row) wins the
// slot, evicts the old occupant into the staging list (or leaves a
// placeholder if the slot was empty) and installs its key with count 0;
// every missing point whose key now owns its slot adds 1, the others stage
// (key, 1). Each winner and each loser adds one staged entry.
template <bool kNarrow, bool kPf, bool kC128>
__device__ __forceinline__ bool process_batch(const Grid& g, const Table& t, const double* x,
                                              const double* y, WarpSmem& w, K1State& s,
                                              int lane, u32 lt_mask, u32 budget) {
    using K = KeyOps<kNarrow>;
    u64 key[kBatch];
    u32 cs[kBatch];
    bool miss[kBatch];
    bool valid[kBatch];
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
        key[r] = K::raw_key(g, x[r], y[r]);
        valid[r] = in_bounds(g, x[r], y[r]);
        cs[r] = K::slot(key[r], g.bits_y);
    }
    bool any = false;
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
        const u64 ck = w.ckey[cs[r]];
        const bool hit = (ck == key[r]) & valid[r];
        if (hit) atomicAdd(&w.ccnt[cs[r]], 1u);
        miss[r] = valid[r] & !hit;
        any |= miss[r];
    }
    if (!__any_sync(kFull, any)) return false;  // pot only grows on the miss path
#pragma unroll
    for (int r = 0; r < kBatch; ++r)
        if (miss[r]) w.owner[cs[r]] = (unsigned char)(r * 32 + lane);
    __syncwarp();
    u64 sk[kBatch];
    u32 sc[kBatch];
    bool win[kBatch];
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
        win[r] = miss[r] && w.owner[cs[r]] == (unsigned char)(r * 32 + lane);
        sk[r] = kEmpty;
        sc[r] = 0;
        if (win[r]) {
            sk[r] = K::table_key(w.ckey[cs[r]], g.bits_y);  // kEmpty: placeholder
            sc[r] = w.ccnt[cs[r]];
            w.ckey[cs[r]] = key[r];
            w.ccnt[cs[r]] = 0;
            // The evicted tile waits in the staging list for the next flush
            // (at most 64 entries away). For tables up to 256 MB its home
            // slot's sector is fetched into L2 now, so the flush's CAS does
            // not wait on DRAM (config 3: K1 0.354 -> 0.320 ms); with config
            // 4's 537 MB table the same prefetch costs 8 % (1.56 -> 1.68 ms),
            // as does prefetching when a tile enters the cache.
            if (kPf && sk[r] != kEmpty) prefetch_slot(t, sk[r]);
        }
    }
    __syncwarp();
    u32 pos = s.slen;
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
        bool lose = false;
        if (miss[r]) {
            if (w.ckey[cs[r]] == key[r]) {
                atomicAdd(&w.ccnt[cs[r]], 1u);
            } else {
                lose = true;
                sk[r] = K::table_key(key[r], g.bits_y);
                sc[r] = 1;
            }
        }
        const bool stage = win[r] | lose;
        const u32 m = ballot(stage);
        if (stage) {
            const u32 at = pos + __popc(m & lt_mask);
            w.skey[at] = sk[r];
            w.scnt[at] = sc[r];
        }
        pos += __popc(m);
    }
    s.pot += pos - s.slen;
    s.slen = pos;
    __syncwarp();
    if (s.slen > kStageCap - 32 * kBatch) flush_stage<kC128>(t, w, s, lane);
    return s.pot >= budget;
}
#endif  // RG_K1_ROWWISE


// ------------------------------------------------------- TMA bulk staging
// One elected lane arms a stage's mbarrier with the byte count and issues
// ONE bulk copy (cp.async.bulk, the TMA's non-tensor form, L2 evict-first)
// for the whole stage; the warp waits on the mbarrier phase. This replaces
// 32 per-lane LDGSTS + commit/wait per row.
__device__ __forceinline__ u32 smem_u32(const void* p) {
    return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, u32 bytes, u64* bar,
                                          u64 pol) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
#ifndef RG_MBAR_HINT
#define RG_MBAR_HINT 0x989680
#endif
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    // the suspend-time hint lets the scheduler park the warp until the phase
    // completes instead of spinning on the barrier (issue slots)
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(RG_MBAR_HINT)
        : "memory");
}

#ifndef RG_K1_RING
#define RG_K1_RING 4
#endif
constexpr int kRing = RG_K1_RING;  // rows in flight per warp (multiple of kBatch)
#ifndef RG_K1_UNROLL
#define RG_K1_UNROLL 2
#endif
constexpr int kK1Unroll = RG_K1_UNROLL;  // batches per trip of run_segment's loop

// One segment of nr rows starting at `base` (this lane's point of the first
// row). kFullRows: every point of every row exists (all segments but
// possibly the last), so loads need no per-lane checks. `valid` = points of
// the segment (only read when !kFullRows). Each lane copies its own point
// into its own ring column, so no cross-lane synchronisation is needed
// around the ring. Returns the row index at which the warp ran out of
// budget, or nr.
template <bool kAligned, bool kNarrow, bool kFullRows, bool kPf, bool kC128>
__device__ __forceinline__ u32 run_segment(const double2* base, const double* xy_base, u32 nr,
                                           u32 valid, double2 (*ring)[32], const Grid& g,
                                           const Table& t, WarpSmem& w, K1State& st, int lane,
                                           u32 lt_mask, u64 pol, u32 budget) {
    auto issue = [&](u32 row) {
        if (row < nr) {
            const u32 idx = row * 32 + lane;
            if (kFullRows || idx < valid) {
                double2* dst = &ring[row % kRing][lane];
                if (kAligned) {
                    cp_async16(dst, base + row * 32, pol);
                } else {
                    dst->x = xy_base[2 * (u64)idx];
                    dst->y = xy_base[2 * (u64)idx + 1];
                }
            }
        }
        cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < kRing; ++k) issue(k);
#pragma unroll kK1Unroll
    for (u32 j = 0; j < nr; j += kBatch) {
        cp_async_wait<kRing - kBatch>();
        double x[kBatch], y[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const u32 row = j + b;
            if (kFullRows || (row < nr && row * 32 + lane < valid)) {
                const double2 v = ring[row % kRing][lane];
                x[b] = v.x;
                y[b] = v.y;
            } else {
                x[b] = y[b] = __longlong_as_double(0x7ff8000000000000ll);
            }
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) issue(j + kRing + b);
#ifdef RG_K1_STREAM_ONLY  // experiment: the load path alone (results are wrong)
#pragma unroll
        for (int b = 0; b < kBatch; ++b) st.added += (x[b] + y[b] > 1e300) ? 1 : 0;
        const bool over = false;
#else
        const bool over = process_batch<kNarrow, kPf, kC128>(g, t, x, y, w, st, lane, lt_mask, budget);
#endif
        if (over) return j + kBatch < nr ? j + kBatch : nr;
    }
    return nr;
}

// run_segment with TMA bulk staging (16-byte aligned points): the ring is
// kStages stages of kBatch rows; lane 0 refills a stage with one bulk copy
// once every lane has read it. `phase` carries the stages' mbarrier parities
// across segments. Same return convention as run_segment.
constexpr int kStages = kRing / kBatch;
template <bool kNarrow, bool kPf, bool kC128>
__device__ __forceinline__ u32 run_segment_tma(const double2* src, u32 nr, u32 valid,
                                               double2 (*ring)[32], u64* bar, u32& phase,
                                               const Grid& g, const Table& t, WarpSmem& w,
                                               K1State& st, int lane, u32 lt_mask, u64 pol,
                                               u32 budget) {
    const u32 nb = (nr + kBatch - 1) / kBatch;
    auto issue = [&](u32 b) {  // lane 0 only
        const u32 first = b * (kBatch * 32);
        const u32 cnt = min((u32)(kBatch * 32), valid - first);
        bulk_load(ring[(b % kStages) * kBatch], src + first, cnt * 16u, &bar[b % kStages], pol);
    };
    if (lane == 0)
        for (u32 b = 0; b < (u32)kStages && b < nb; ++b) issue(b);
    u32 done_b = nb;
    for (u32 b = 0; b < nb; ++b) {
        const u32 s = b % kStages;
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        double x[kBatch], y[kBatch];
#pragma unroll
        for (int r = 0; r < kBatch; ++r) {
            const u32 idx = b * (kBatch * 32) + r * 32 + lane;
            const double2 v = ring[s * kBatch + r][lane];
            x[r] = idx < valid ? v.x : __longlong_as_double(0x7ff8000000000000ll);
            y[r] = v.y;
        }
        __syncwarp();  // every lane has read the stage: it may be refilled
        if (lane == 0 && b + kStages < nb) {
#ifndef RG_K1_NOFENCE
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
            issue(b + kStages);
        }
        if (process_batch<kNarrow, kPf, kC128>(g, t, x, y, w, st, lane, lt_mask, budget)) {
            done_b = b + 1;
            break;
        }
    }
    // stages still in flight after a budget stop
    for (u32 b = done_b; b < nb && b < done_b + kStages; ++b) {
        const u32 s = b % kStages;
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
    }
    return done_b < nb ? done_b * kBatch : nr;
}

template <bool kAligned, bool kNarrow, bool kTma, bool kPf = false, bool kC128 = false>
// (the 128-bit claim variant is held to the others' 9 blocks per SM: the
// launch is sized for the slowest variant's residency)
__global__ void __launch_bounds__(kThreads, kC128 ? 9 : RG_K1_MINBLOCKS) k_contract(K1Params P) {
    __shared__ WarpSmem s_warp[kWarpsPerBlock];
    __shared__ __align__(16) double2 s_ring[kWarpsPerBlock][kRing][32];
    __shared__ u64 s_bar[kWarpsPerBlock][kStages];

    const int lane = threadIdx.x & 31;
    const u32 lt_mask = (1u << lane) - 1;
    WarpSmem& w = s_warp[threadIdx.x >> 5];
    double2 (*ring)[32] = s_ring[threadIdx.x >> 5];
    for (int i = lane; i < kCacheSlots; i += 32) {
        w.ckey[i] = kEmpty;
        w.ccnt[i] = 0;
    }
    u64* bar = s_bar[threadIdx.x >> 5];
    u32 phase = 0;
    if (kTma && lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncwarp();

    const Grid g = P.g;
    const Table t = P.t;
    const u64 pol = evict_first_policy();
    const double2* pts = reinterpret_cast<const double2*>(P.xy);
    K1State st{0, 0, 0, 0};
    u64 n_valid = 0;  // warp-uniform: points examined
    bool stopped = false;

    // Work queue: partial segments of a previous (stopped) launch first, then
    // fresh tickets; the next ticket is requested while the current segment
    // is processed.
    u64 pending = ~0ull;  // prefetched ticket (lane 0's copy is authoritative)
    auto fetch = [&](u64& seg, u64& row0, bool& from_ticket) -> bool {
        if (P.n_partial_in) {
            u64 pt = 0;
            if (lane == 0) pt = atomicAdd(&P.ctr->partial_ticket, 1ull);
            pt = __shfl_sync(kFull, pt, 0);
            if (pt < P.n_partial_in) {
                seg = P.partial_in[pt].segment;
                row0 = P.partial_in[pt].next_row;
                from_ticket = false;
                return true;
            }
        }
        u64 tk = pending;
        if (tk == ~0ull) {
            if (lane == 0) tk = atomicAdd(&P.ctr->ticket, 1ull);
        }
        tk = __shfl_sync(kFull, tk, 0);
        pending = ~0ull;
        if (tk >= P.n_seg) return false;
        seg = tk;
        row0 = tk * P.rows_per_seg;
        from_ticket = true;
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
    bool from_ticket;
    bool have = fetch(seg, row0, from_ticket);
    while (have) {
        const u64 row_end = min((seg + 1) * P.rows_per_seg, P.n_rows);
        if (lane == 0 && (from_ticket || P.n_partial_in == 0))
            pending = atomicAdd(&P.ctr->ticket, 1ull);
        // 32-bit cache counts: a segment adds at most 32 * rows_per_seg
        // (<= 8192) to an entry, so moving large counts out here keeps
        // every entry below 2^31 + 8192.
        {
            u32 gc = 0;
            for (int i = lane; i < kCacheSlots; i += 32) {
                if (w.ccnt[i] >= 0x80000000u) {
                    const u64 k = KeyOps<kNarrow>::table_key(w.ckey[i], g.bits_y);
                    gc += table_add_cas(t, k, w.ccnt[i]) ? 1u : 0u;
                    st.added += w.ccnt[i];
                    w.ccnt[i] = 0;
                }
            }
            st.claims += gc;
            st.pot += __reduce_add_sync(kFull, gc);  // the entry stays cached too
            __syncwarp();
        }
        const u32 nr = (u32)(row_end - row0);
        const u64 p0 = row0 * 32;
        const u32 valid = (u32)min(P.n - p0, (u64)nr * 32);
        const double2* base = pts + p0 + lane;
        const double* xy_base = P.xy + 2 * p0;
        u32 done;
        if (kTma)
            done = run_segment_tma<kNarrow, kPf, kC128>(pts + p0, nr, valid, ring, bar, phase, g, t, w, st,
                                            lane, lt_mask, pol, P.budget);
        else if (valid == nr * 32 && nr % kBatch == 0)
            done = run_segment<kAligned, kNarrow, true, kPf, kC128>(base, xy_base, nr, valid, ring, g, t, w,
                                                        st, lane, lt_mask, pol, P.budget);
        else
            done = run_segment<kAligned, kNarrow, false, kPf, kC128>(base, xy_base, nr, valid, ring, g, t, w,
                                                         st, lane, lt_mask, pol, P.budget);
        if (!kTma) cp_async_wait<0>();
        n_valid += min((u64)done * 32, (u64)valid);
        if (done < nr || st.pot >= P.budget) {
            if (done < nr) record_partial(seg, row0 + done);
            // hand back the prefetched ticket too
            const u64 tk = __shfl_sync(kFull, pending, 0);
            if (tk != ~0ull && tk < P.n_seg) record_partial(tk, tk * P.rows_per_seg);
            stopped = true;
            break;
        }
        have = fetch(seg, row0, from_ticket);
    }

    // Write back staged entries and the cache.
    flush_stage<kC128>(t, w, st, lane);
    for (int i = lane; i < kCacheSlots; i += 32) {
        const u64 k = KeyOps<kNarrow>::table_key(w.ckey[i], g.bits_y);
        if (k != kEmpty) {
            st.claims += table_add_cas(t, k, w.ccnt[i]) ? 1u : 0u;
            st.added += w.ccnt[i];
        }
    }

    // Counters: one atomic per warp. Every in-bounds point reached the table
    // through exactly one table_add, so the added counts are the ingested
    // points (conservation, test_accumulator.cpp:88-99).
    const u32 wc = __reduce_add_sync(kFull, st.claims);
    u64 wi = st.added;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wi += __shfl_xor_sync(kFull, wi, o);
    if (lane == 0) {
        if (wi) atomicAdd(&P.ctr->ingested, wi);
        if (n_valid > wi) atomicAdd(&P.ctr->skipped, n_valid - wi);
        if (wc) atomicAdd(&P.ctr->used, (u64)wc);
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

// Fold (key, count) pairs into a table (merge of pre-aggregated counts, e.g.
// received from other ranks). Adds the claimed keys and the summed counts.
__global__ void k_pairs_fold(const u64* keys, const u64* cnts, u64 n, Table dst, u64* claimed,
                             u64* points) {
    u32 local = 0;
    u64 pts = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n;
         i += (u64)gridDim.x * blockDim.x) {
        local += table_add(dst, keys[i], cnts[i]) ? 1u : 0u;
        pts += cnts[i];
    }
    const u32 w = __reduce_add_sync(kFull, local);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pts += __shfl_xor_sync(kFull, pts, o);
    if ((threadIdx.x & 31) == 0) {
        if (w) atomicAdd(claimed, (u64)w);
        if (pts) atomicAdd(points, pts);
    }
}

// Occupied slots -> (key, count) arrays (block-aggregated append).
__global__ void __launch_bounds__(256) k_export(const Slot* slots, u64 cap, u64* keys, u64* cnts,
                                                u64* n_out) {
    __shared__ u32 s_w[8];
    __shared__ u64 s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int kItems = 8;
    for (u64 base = blockIdx.x * 256ull * kItems; base < cap; base += (u64)gridDim.x * 256 * kItems) {
        u64 k[kItems], v[kItems];
        u32 c = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const u64 i = base + (u64)j * 256 + threadIdx.x;
            k[j] = kEmpty;
            v[j] = 0;
            if (i < cap) ld_slot(slots + i, k[j], v[j]);
            c += k[j] != kEmpty;
        }
        u32 incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += y;
        }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            u32 t = 0;
            for (int q = 0; q < 8; ++q) {
                const u32 x = s_w[q];
                s_w[q] = t;
                t += x;
            }
            s_base = t ? atomicAdd(n_out, (u64)t) : 0;
        }
        __syncthreads();
        u64 at = s_base + s_w[wid] + incl - c;
#pragma unroll
        for (int j = 0; j < kItems; ++j)
            if (k[j] != kEmpty) {
                keys[at] = k[j];
                cnts[at] = v[j];
                ++at;
            }
        __syncthreads();
    }
}

cudaError_t launch_pairs_fold(const u64* keys, const u64* cnts, u64 n, Table dst, u64* claimed,
                              u64* points, int n_sm, cudaStream_t st) {
    const u64 want = (n + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? (want ? want : 1) : (u64)n_sm * 16);
    k_pairs_fold<<<blocks, 256, 0, st>>>(keys, cnts, n, dst, claimed, points);
    return cudaGetLastError();
}

cudaError_t launch_export(const Slot* slots, u64 cap, u64* keys, u64* cnts, u64* n_out, int n_sm,
                          cudaStream_t st) {
    const u64 want = (cap + 2047) / 2048;
    const int blocks = (int)(want < (u64)n_sm * 8 ? (want ? want : 1) : (u64)n_sm * 8);
    k_export<<<blocks, 256, 0, st>>>(slots, cap, keys, cnts, n_out);
    return cudaGetLastError();
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
// Each significant slot gets a dense index, its key/count are written to the
// compact arrays, the slot's value word becomes SIG_BIT | index and the
// union-find parent is initialised. A warp streams 32 x kK2Items consecutive
// slots per step (coalesced 16-byte loads, all in flight together) and only
// stages the slot numbers of significant entries in shared memory; every
// >= 256 staged entries it reserves output space with one atomic and writes
// them out contiguously (the slots are re-read from L1/L2). Waiting on the
// reservation is paid once per 256 outputs instead of once per step.
#ifndef RG_K2_ITEMS
#define RG_K2_ITEMS 4
#endif
constexpr int kK2Items = RG_K2_ITEMS;
#ifndef RG_K2_FLUSH
#define RG_K2_FLUSH 128
#endif
constexpr u32 kK2Flush = RG_K2_FLUSH;  // staged entries that trigger a write-out
constexpr int kK2Stage = kK2Flush + 32 * kK2Items;

struct K2Out {
    u64* sig_key;
    u64* sig_cnt;
    u32* parent;
    // per-root accumulators of agglomeration, initialised here
    u32* size;
    u64* npts;
    u64* min_key;
    int* root_cid;
    u32* col_cnt;  // sorted K3: per-column tile counts (key >> bits_y), or null
    u32 bits_y;
    u32* slot_of;  // sorted K3: table slot of each significant tile (the table is not rewritten)
};

__device__ __forceinline__ void k2_flush(const Table& t, const u32* s_idx, u32 n, const K2Out& o,
                                         Counters* ctr, int lane) {
    u64 at = 0;
    if (lane == 0) at = atomicAdd(&ctr->n_sig, (u64)n);
    at = __shfl_sync(kFull, at, 0);
    for (u32 e = lane; e < n; e += 32) {
        const u32 i = s_idx[e];
        u64 k, v;
        ld_slot(t.slots + i, k, v);
        const u64 pos = at + e;
        o.sig_key[pos] = k;
        o.sig_cnt[pos] = v;
        if (o.size) {  // hash-probe K3 only (the sorted K3 initialises its own)
            o.parent[pos] = (u32)pos;
            o.size[pos] = 0;
            o.npts[pos] = 0;
            o.min_key[pos] = kEmpty;
            o.root_cid[pos] = -1;
        }
        if (o.slot_of)
            o.slot_of[pos] = i;  // the table's SIG marks are written when K4 needs them
        else
            t.slots[i].count = kSigBit | pos;
    }
    if (o.col_cnt) {
        // column histogram of the sorted K3 (replaces its k_col_hist pass):
        // flushed slots come in table order, so a warp's keys share a few
        // 4x4 blocks and columns; one RED per distinct column of a warp
        for (u32 e0 = 0; e0 < n; e0 += 32) {
            const u32 e = e0 + lane;
            const u32 col = e < n ? (u32)(o.sig_key[at + e] >> o.bits_y) : 0xffffffffu;
            const u32 peers = __match_any_sync(kFull, col);
            if (col != 0xffffffffu && lane == __ffs(peers) - 1)
                red_add_u32(o.col_cnt + col, (u32)__popc(peers));
        }
    }
    __syncwarp();
}

// window_fix agglomerate.hpp:212-246 — a tile is significant when some 2x2
// window containing it holds >= tau points. The windows containing tile t are
// the four anchored at t + (ax, ay), ax, ay in {-1, 0}, so the decision for
// t needs only the counts of its 3x3 neighbourhood: one thread per occupied
// slot, eight table lookups, one flag byte. (The reference marks every
// occupied tile of each window it evaluates; the set of marked tiles is the
// same, since every window containing t is one of t's own four.)
__global__ void __launch_bounds__(256) k_window_mark(Table t, u64 cap, u64 tau, u32 bits_x,
                                                     u8* keep) {
    const long long xlim = 1ll << bits_x, ylim = 1ll << t.bits_y;
    const u64 ymask = (1ull << t.bits_y) - 1;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < cap;
         i += (u64)gridDim.x * blockDim.x) {
        u64 k, v;
        ld_slot(t.slots + i, k, v);
        if (k == kEmpty) continue;
        const long long kx = (long long)(k >> t.bits_y), ky = (long long)(k & ymask);
        u64 c[3][3];
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx)
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy) {
                u64 w = 0;
                const long long nx = kx + dx, ny = ky + dy;
                if (dx == 0 && dy == 0) {
                    w = v;
                } else if (nx >= 0 && nx < xlim && ny >= 0 && ny < ylim) {
                    const u64 f = table_find(t, ((u64)nx << t.bits_y) | (u64)ny);
                    w = f == kEmpty ? 0 : f;
                }
                c[dx + 1][dy + 1] = w;
            }
        bool any = false;
#pragma unroll
        for (int ax = 0; ax <= 1; ++ax)
#pragma unroll
            for (int ay = 0; ay <= 1; ++ay)
                any |= c[ax][ay] + c[ax + 1][ay] + c[ax][ay + 1] + c[ax + 1][ay + 1] >= tau;
        keep[i] = any;
    }
}

// keep == nullptr: count >= tau (prune); else the window_fix flags.
__global__ void __launch_bounds__(256) k_compact(Table t, u64 cap, u64 tau, const u8* keep,
                                                 K2Out out, Counters* ctr) {
    __shared__ u32 s_stage[8][kK2Stage];
    const int lane = threadIdx.x & 31;
    u32* s_idx = s_stage[threadIdx.x >> 5];
    const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
    const u64 n_warps = ((u64)gridDim.x * blockDim.x) >> 5;
    constexpr u64 per_warp = 32ull * kK2Items;
    u32 slen = 0;  // warp-uniform
    for (u64 base = warp * per_warp; base < cap; base += n_warps * per_warp) {
        u64 k[kK2Items], v[kK2Items];
#pragma unroll
        for (int j = 0; j < kK2Items; ++j) {
            const u64 i = base + j * 32 + lane;
            if (i < cap) {
                ld_slot(t.slots + i, k[j], v[j]);
                if (keep) v[j] = keep[i] ? tau : 0;  // predicate only; k2_flush re-reads
            } else {
                k[j] = kEmpty;
                v[j] = 0;
            }
        }
        u32 nsig = 0;
#pragma unroll
        for (int j = 0; j < kK2Items; ++j) nsig += (k[j] != kEmpty && v[j] >= tau);
        u32 incl = nsig;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        const u32 total = __shfl_sync(kFull, incl, 31);
        u32 p = slen + incl - nsig;
#pragma unroll
        for (int j = 0; j < kK2Items; ++j)
            if (k[j] != kEmpty && v[j] >= tau) s_idx[p++] = (u32)(base + j * 32 + lane);
        slen += total;
        __syncwarp();
        if (slen >= kK2Flush) {
            k2_flush(t, s_idx, slen, out, ctr, lane);
            slen = 0;
        }
    }
    if (slen) k2_flush(t, s_idx, slen, out, ctr, lane);
}

// K2, one pass per tile (default): a block takes the next tile of
// kK2LbThr x kK2LbPer slots from a ticket, loads all of its slots (four
// 16-byte loads in flight per thread), counts the significant ones,
// reserves the tile's output range with one atomic and writes key, count
// and slot index straight from registers. No re-read of the table (the
// staged variant above re-reads every flushed slot).
#ifndef RG_K2_THR
#define RG_K2_THR 256
#endif
#ifndef RG_K2_PER
#define RG_K2_PER 4  // (256 x 8: 166 us, 256 x 4: 145 us, 256 x 2: 176 us, 128 x 4: 164 us, 512 x 8: 174 us, 1024 x 8: 196 us)
#endif
constexpr int kK2LbThr = RG_K2_THR, kK2LbPer = RG_K2_PER;
constexpr u64 kK2LbTile = (u64)kK2LbThr * kK2LbPer;
__global__ void __launch_bounds__(kK2LbThr) k_compact_lb(Table t, u64 cap, u64 tau, const u8* keep,
                                                         K2Out o, Counters* ctr, u64* status,
                                                         u32* ticket) {
    __shared__ u32 s_warp[33];
    __shared__ u32 s_tile;
    __shared__ u64 s_pre;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const u32 tile = s_tile;
    const int lane = threadIdx.x & 31;
    const u64 base = (u64)tile * kK2LbTile;
    u64 k[kK2LbPer], v[kK2LbPer];
#pragma unroll
    for (int j = 0; j < kK2LbPer; ++j) {
        const u64 i = base + (u64)j * kK2LbThr + threadIdx.x;  // striped: coalesced
        k[j] = kEmpty;
        v[j] = 0;
        if (i < cap) ld_slot(t.slots + i, k[j], v[j]);
    }
    u32 flags = 0;
#pragma unroll
    for (int j = 0; j < kK2LbPer; ++j) {
        const u64 i = base + (u64)j * kK2LbThr + threadIdx.x;
        const bool sig = k[j] != kEmpty && (keep ? (i < cap && keep[i] != 0) : v[j] >= tau);
        flags |= (u32)sig << j;
    }
    u32 agg;
    const u32 ex = block_excl_sum<kK2LbThr>((u32)__popc(flags), s_warp, &agg);
    // one reservation per tile (the output order is free: K3 sorts). A
    // decoupled look-back here measured 370 us: with ~1,200 tiles in
    // flight the look-back walked hundreds of predecessors per tile.
    if (threadIdx.x == 0) s_pre = agg ? atomicAdd(&ctr->n_sig, (u64)agg) : 0;
    __syncthreads();
    u64 pos = s_pre + ex;
#pragma unroll
    for (int j = 0; j < kK2LbPer; ++j) {
        const bool sig = (flags >> j) & 1u;
        if (sig) {
            const u32 i = (u32)(base + (u64)j * kK2LbThr + threadIdx.x);
            o.sig_key[pos] = k[j];
            o.sig_cnt[pos] = v[j];
            if (o.size) {  // hash-probe K3 only (the sorted K3 initialises its own)
                o.parent[pos] = (u32)pos;
                o.size[pos] = 0;
                o.npts[pos] = 0;
                o.min_key[pos] = kEmpty;
                o.root_cid[pos] = -1;
            }
            if (o.slot_of)
                o.slot_of[pos] = i;  // the table's SIG marks are written when K4 needs them
            else
                t.slots[i].count = kSigBit | pos;
            ++pos;
        }
        if (o.col_cnt) {
            // column histogram of the sorted K3: a warp's 32 slots of row j
            // share a few 4x4 blocks, so one RED per distinct column
            const u32 col = sig ? (u32)(k[j] >> o.bits_y) : 0xffffffffu;
            const u32 peers = __match_any_sync(kFull, col);
            if (sig && lane == __ffs(peers) - 1) red_add_u32(o.col_cnt + col, (u32)__popc(peers));
        }
    }
}

// K2 over (key, count) pairs instead of the table: after a partitioned
// contraction into an empty table every work unit's pairs are final counts
// (one unit per partition), so prune (accumulator.hpp:160-174) is a filter
// of the pair slabs - 150 MB for config 4 instead of the 537 MB table -
// and does not wait for the pairs' insertion into the table, which runs
// beside K2 and K3 on another stream. One block per unit; a reservation
// atomic per 1024 pairs; the column histogram as in k_compact_lb. The
// table slots of the significant tiles are not known here (k_find_slots
// looks them up if SIG marks are ever needed).
__global__ void __launch_bounds__(256) k_compact_pairs(const uint4* units, const u32* dcnt,
                                                       u32 n_units, const u64* pkey,
                                                       const u32* pcnt, u64 tau, K2Out o,
                                                       Counters* ctr) {
    __shared__ u32 s_warp[33];
    __shared__ u64 s_pre;
    const int lane = threadIdx.x & 31;
    constexpr int kPer = 4;
    for (u32 u = blockIdx.x; u < n_units; u += gridDim.x) {
        const u64 lo = units[u].x;
        const u32 d = dcnt[u];
        for (u32 i0 = 0; i0 < d; i0 += 256 * kPer) {
            u64 k[kPer];
            u32 v[kPer];
            u32 flags = 0;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const u32 i = i0 + j * 256 + threadIdx.x;
                k[j] = kEmpty;
                v[j] = 0;
                if (i < d) {
                    k[j] = pkey[lo + i];
                    v[j] = pcnt[lo + i];
                }
                flags |= (u32)(i < d && v[j] >= tau) << j;
            }
            u32 agg;
            const u32 ex = block_excl_sum<256>((u32)__popc(flags), s_warp, &agg);
            if (threadIdx.x == 0) s_pre = agg ? atomicAdd(&ctr->n_sig, (u64)agg) : 0;
            __syncthreads();
            u64 pos = s_pre + ex;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const bool sig = (flags >> j) & 1u;
                if (sig) {
                    o.sig_key[pos] = k[j];
                    o.sig_cnt[pos] = v[j];
                    ++pos;
                }
                if (o.col_cnt) {
                    const u32 col = sig ? (u32)(k[j] >> o.bits_y) : 0xffffffffu;
                    const u32 peers = __match_any_sync(kFull, col);
                    if (sig && lane == __ffs(peers) - 1)
                        red_add_u32(o.col_cnt + col, (u32)__popc(peers));
                }
            }
            __syncthreads();
        }
    }
}

// Table slot of every significant tile (for the SIG marks, after a K2 that
// did not scan the table).
__global__ void k_find_slots(Table t, const u64* sig_key, u64 n, u32* slot_of) {
    for (u64 pos = blockIdx.x * (u64)blockDim.x + threadIdx.x; pos < n;
         pos += (u64)gridDim.x * blockDim.x) {
        const u64 key = sig_key[pos];
        Probe p(key, t);
        while (true) {
            const u64 k = ld_key(t.slots + p.slot());
            if (k == key || k == kEmpty) break;  // (every significant tile is in the table)
            p.next(t);
        }
        slot_of[pos] = (u32)p.slot();
    }
}

cudaError_t launch_compact_pairs(const uint4* units, const u32* dcnt, u32 n_units, const u64* pkey,
                                 const u32* pcnt, u64 tau, u64* sig_key, u64* sig_cnt,
                                 u32* col_cnt, u32 bits_y, Counters* ctr, int n_sm,
                                 cudaStream_t st) {
    if (n_units == 0) return cudaSuccess;
    const K2Out o{sig_key, sig_cnt, nullptr, nullptr, nullptr, nullptr, nullptr, col_cnt, bits_y,
                  nullptr};
    const u32 blocks = n_units < (u32)n_sm * 16 ? n_units : (u32)n_sm * 16;
    k_compact_pairs<<<(int)blocks, 256, 0, st>>>(units, dcnt, n_units, pkey, pcnt, tau, o, ctr);
    return cudaGetLastError();
}

cudaError_t launch_find_slots(Table t, const u64* sig_key, u64 n, u32* slot_of, int n_sm,
                              cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const u64 want = (n + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? want : (u64)n_sm * 16);
    k_find_slots<<<blocks, 256, 0, st>>>(t, sig_key, n, slot_of);
    return cudaGetLastError();
}

// Deferred SIG marks (sorted K3 path): the count word of significant tile
// pos becomes SIG | pos (dense index, as K2 writes it on the hash path) or
// SIG | (cluster id + 1) (K4's lookups then need no second load).
__global__ void k_mark_sig(Table t, const u32* slot_of, const int* cid, u64 n) {
    for (u64 pos = blockIdx.x * (u64)blockDim.x + threadIdx.x; pos < n;
         pos += (u64)gridDim.x * blockDim.x)
        t.slots[slot_of[pos]].count = kSigBit | (cid ? (u64)(u32)(cid[pos] + 1) : pos);
}

cudaError_t launch_mark_sig(Table t, const u32* slot_of, const int* cid, u64 n, int n_sm,
                            cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const u64 want = (n + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? want : (u64)n_sm * 16);
    k_mark_sig<<<blocks, 256, 0, st>>>(t, slot_of, cid, n);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- launchers

static int g_k1_warps_per_sm = 0;

// Resident warps per SM of the slowest K1 variant: the launch is persistent
// (one wave), and the per-warp new-key budget bounds how far the table can
// overshoot its load target (see ingest_device in api.cu).
int contract_max_warps(int n_sm) {
    if (!g_k1_warps_per_sm) {
        int b[7] = {0, 0, 0, 0, 0, 0, 0};
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[0], k_contract<true, true, false>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[1], k_contract<true, false, false>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[2], k_contract<false, true, false>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[3], k_contract<false, false, false>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[4], k_contract<true, true, true>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[5], k_contract<true, true, false, true>, kThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[6], k_contract<true, true, false, false, true>, kThreads, 0);
        int m = b[0];
        for (int i = 1; i < 7; ++i) m = b[i] < m ? b[i] : m;
        g_k1_warps_per_sm = (m < 1 ? 1 : m) * kWarpsPerBlock;
    }
    return g_k1_warps_per_sm * n_sm;
}

int contract_batch_rows() { return kBatch; }
int contract_block_warps() { return kWarpsPerBlock; }

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
    P.budget = (u32)(L.budget < (1ull << 30) ? L.budget : (1ull << 30));
    static const int pf_mode = [] {  // RG_K1_PREFETCH=0 / =1 forces it (A/B)
        const char* v = std::getenv("RG_K1_PREFETCH");
        return v ? (std::strcmp(v, "0") == 0 ? 0 : 1) : -1;
    }();
    const u64 table_bytes = (L.t.bmask + 1) * kBucketSlots * sizeof(Slot);
    const bool prefetch = pf_mode >= 0 ? pf_mode != 0 : table_bytes <= (256ull << 20);
    const int blocks = (int)((L.warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
    const bool aligned = ((uintptr_t)L.xy & 15) == 0;
    // RG_K1=tma selects the TMA bulk-copy ring (measured slower than the
    // per-lane cp.async ring: DESIGN.md, K1)
    static const bool tma = [] {
        const char* v = std::getenv("RG_K1");
        return v && std::strcmp(v, "tma") == 0;
    }();
    if (aligned && L.narrow && tma)
        k_contract<true, true, true><<<blocks, kThreads, 0, st>>>(P);
    else if (aligned && L.narrow && L.claim128)
        k_contract<true, true, false, false, true><<<blocks, kThreads, 0, st>>>(P);
    else if (aligned && L.narrow && prefetch)
        k_contract<true, true, false, true><<<blocks, kThreads, 0, st>>>(P);
    else if (aligned && L.narrow)
        k_contract<true, true, false><<<blocks, kThreads, 0, st>>>(P);
    else if (aligned)
        k_contract<true, false, false><<<blocks, kThreads, 0, st>>>(P);
    else if (L.narrow)
        k_contract<false, true, false><<<blocks, kThreads, 0, st>>>(P);
    else
        k_contract<false, false, false><<<blocks, kThreads, 0, st>>>(P);
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

u64 compact_lb_words(u64 cap) { return (cap + kK2LbTile - 1) / kK2LbTile + 2; }

cudaError_t launch_compact(Table t, u64 cap, u64 tau, const u8* keep, u64* sig_key, u64* sig_cnt,
                           u32* parent, u32* size, u64* npts, u64* min_key, int* root_cid,
                           u32* col_cnt, u32* slot_of, Counters* ctr, int n_sm,
                           cudaStream_t st, u64* lb_scratch) {
#ifndef RG_K2_BPS
#define RG_K2_BPS 16
#endif
    const u64 per_block = 256ull * kK2Items;
    const u64 want = (cap + per_block - 1) / per_block;
    const u64 mx = (u64)n_sm * RG_K2_BPS;
    const int blocks = (int)(want < mx ? (want ? want : 1) : mx);
    const K2Out o{sig_key, sig_cnt, parent, size, npts, min_key, root_cid, col_cnt, t.bits_y,
                  slot_of};
    static const bool staged = [] {  // RG_K2=staged: the reservation-based K2 (A/B)
        const char* v = std::getenv("RG_K2");
        return v && std::strcmp(v, "staged") == 0;
    }();
    if (lb_scratch && !staged) {
        const u64 tiles = (cap + kK2LbTile - 1) / kK2LbTile;
        cudaError_t e = cudaMemsetAsync(lb_scratch, 0, (tiles + 2) * sizeof(u64), st);
        if (e != cudaSuccess) return e;
        k_compact_lb<<<(int)tiles, kK2LbThr, 0, st>>>(t, cap, tau, keep, o, ctr, lb_scratch + 2,
                                                      (u32*)lb_scratch);
        return cudaGetLastError();
    }
    k_compact<<<blocks, 256, 0, st>>>(t, cap, tau, keep, o, ctr);
    return cudaGetLastError();
}

cudaError_t launch_window_mark(Table t, u64 cap, u64 tau, u32 bits_x, u8* keep, int n_sm,
                               cudaStream_t st) {
    const u64 want = (cap + 255) / 256;
    const int blocks = (int)(want < (u64)n_sm * 16 ? (want ? want : 1) : (u64)n_sm * 16);
    k_window_mark<<<blocks, 256, 0, st>>>(t, cap, tau, bits_x, keep);
    return cudaGetLastError();
}

}  // namespace rg
