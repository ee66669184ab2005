// common.cuh — device-side data layout shared by all RASTER kernels.
//
// Tile keys. The reference identifies a tile by raster::Tile{int64 x, int64 y}
// with lexicographic order (core.hpp:48-54). On the device a tile is one
// 64-bit packed key
//      key = (tx - origin_x) << bits_y | (ty - origin_y)
// with both fields non-negative and bits_x + bits_y <= 63, so unsigned key
// order == lexicographic Tile order and the all-ones word can never be a key
// (it is the EMPTY sentinel). For ingested points origin = (min_column,
// min_row) of the canvas (core.hpp:117-122); monotonicity of IEEE
// round-to-nearest multiplication guarantees every in-bounds point lands in
// [origin, origin + 2^bits).
//
// Hash table. One open-addressed table of 16-byte slots {u64 key, u64 count}
// in HBM replaces TileCounts (accumulator.hpp:23-99). It is bucketed for
// spatial locality: the grid is cut into 4x4-tile blocks, a block hashes to a
// bucket of 16 slots (256 B, two cache lines) and a tile's slot inside the
// bucket is its in-block position XOR a per-block hash nibble (so inputs
// whose tiles share an in-block position, e.g. lattices, still spread over
// all 16 slots). Collisions probe bucket by bucket at the same in-bucket
// slot; after a full cycle of buckets the slot advances, so every slot is
// reachable and the global load bound is the only fill limit. A cluster's
// tiles share one or a few buckets: contraction updates, neighbour probes
// during agglomeration and per-point lookups touch a handful of lines instead
// of one random line per tile, and compaction (which scans slot order) emits
// spatially adjacent tiles next to each other.
// Keys are claimed with a 64-bit CAS and never change afterwards, so probes
// may use plain (L1-cacheable) loads; counts are bumped with RED.ADD.64.
// After pruning, the count word of a significant slot is overwritten with
// SIG_BIT | dense_index so neighbour lookups and per-point labelling resolve
// a key to its significant-tile index with one probe.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rg {

typedef unsigned long long u64;
typedef unsigned int u32;
typedef unsigned char u8;

constexpr u64 kEmpty = ~0ull;
constexpr u64 kSigBit = 1ull << 63;
constexpr u32 kFull = 0xffffffffu;

struct __align__(16) Slot {
    u64 key;
    u64 count;
};

// Point-set slot of the dedupe mode: the bit patterns of a canonical point
// (never NaN, so {~0, ~0} marks an empty slot).
struct __align__(16) PtKey {
    u64 x, y;
};
struct PointSet {
    PtKey* slots;
    u64 mask;  // capacity - 1 (power of two)
};

// Projection + packing parameters (host computes scale = pow(10, p) with the
// same libm as the reference, core.hpp:95; the device never calls pow).
struct Grid {
    double scale;
    double x_min, x_max, y_min, y_max;
    long long origin_x, origin_y;
    u32 bits_y;
    u32 bits_x;
    int ox32, oy32;  // origin_x / origin_y truncated (narrow canvases): a plain
                     // 32-bit constant operand in the projection, no reload
};

#ifndef RG_BLOCK_BITS
#define RG_BLOCK_BITS 2
#endif
constexpr u32 kBlockBits = RG_BLOCK_BITS;       // 2: 4x4-tile blocks
constexpr u32 kBucketSlots = 1u << (2 * kBlockBits);  // 16 slots per bucket

struct Table {
    Slot* slots;
    u64 bmask;     // buckets - 1 (bucket count is a power of two)
    u32 shift;     // 64 - log2(buckets)
    u32 bits_y;    // key packing of the keys stored in this table (>= kBlockBits)
};

// Probe sequence of a key: Fibonacci hashing of the block coordinate picks
// the home bucket and (next bits) the nibble that scrambles the in-bucket
// slot. The reference's TileHash (core.hpp:56-68) only affects probe order,
// never results.
struct Probe {
    u64 b0, b;
    u32 pos;
    Probe() = default;
    __device__ __forceinline__ Probe(u64 key, const Table& t) {
        const u64 ky = key & ((1ull << t.bits_y) - 1);
        const u64 block =
            ((key >> (t.bits_y + kBlockBits)) << (t.bits_y - kBlockBits)) | (ky >> kBlockBits);
        const u64 h = block * 0x9E3779B97F4A7C15ull;
        b0 = b = h >> t.shift;
        const u32 kx = (u32)(key >> t.bits_y) & ((1u << kBlockBits) - 1);
        const u32 kyl = (u32)key & ((1u << kBlockBits) - 1);
        pos = ((kx << kBlockBits) | kyl) ^ ((u32)(h >> (t.shift - 2 * kBlockBits)) & (kBucketSlots - 1));
    }
    __device__ __forceinline__ u64 slot() const { return (b << (2 * kBlockBits)) | pos; }
    __device__ __forceinline__ void next(const Table& t) {
        b = (b + 1) & t.bmask;
        if (b == b0) pos = (pos + 1) & (kBucketSlots - 1);
    }
};

// Bounds::contains core.hpp:33-35 — closed interval; NaN compares false.
__device__ __forceinline__ bool in_bounds(const Grid& g, double x, double y) {
    return x >= g.x_min && x <= g.x_max && y >= g.y_min && y <= g.y_max;
}

// project_unchecked core.hpp:136-139: (int64)floor(x * s). __dmul_rn is the
// IEEE double product (no FMA contraction can apply to a lone multiply, but
// the intrinsic makes it explicit); cvt.rmi.s64.f64 floors and converts in
// one instruction, identical to floor-then-cast for in-range values.
__device__ __forceinline__ u64 pack_key(const Grid& g, double x, double y) {
    const long long tx = __double2ll_rd(__dmul_rn(x, g.scale));
    const long long ty = __double2ll_rd(__dmul_rn(y, g.scale));
    return ((u64)(tx - g.origin_x) << g.bits_y) | (u64)(ty - g.origin_y);
}

__device__ __forceinline__ u64 ld_key(const Slot* s) {
    u64 v;
    asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(&s->key));
    return v;
}

__device__ __forceinline__ void ld_slot(const Slot* s, u64& key, u64& val) {
    asm volatile("ld.global.v2.u64 {%0, %1}, [%2];" : "=l"(key), "=l"(val) : "l"(s));
}

__device__ __forceinline__ void red_add(u64* p, u64 v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_add_u32(u32* p, u32 v) {
    asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming 128-bit load of one point (read once: keep it out of L1 and
// mark it evict-first in L2 so the hash table stays resident).
__device__ __forceinline__ u64 evict_first_policy() {
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ double2 ld_point_stream(const double2* p, u64 pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// Insert-or-add into the HBM table. Returns true when this call claimed a new
// slot (a new distinct tile). TileCounts::add accumulator.hpp:33-50.
__device__ __forceinline__ bool table_add(const Table& t, u64 key, u64 cnt) {
    Probe p(key, t);
    while (true) {
        Slot* s = t.slots + p.slot();
        u64 k = ld_key(s);
        if (k == key) {
            red_add(&s->count, cnt);
            return false;
        }
        if (k == kEmpty) {
            const u64 old = atomicCAS(&s->key, kEmpty, key);
            if (old == kEmpty) {
                red_add(&s->count, cnt);
                return true;
            }
            if (old == key) {
                red_add(&s->count, cnt);
                return false;
            }
        }
        p.next(t);
    }
}

// table_add for keys that are usually new (K1's evictions): the claim is
// attempted first, so a new key costs one L2 round trip (the CAS) instead of
// a load followed by the CAS; an existing key costs the CAS's read of it.
__device__ __forceinline__ bool table_add_cas(const Table& t, u64 key, u64 cnt) {
    Probe p(key, t);
    while (true) {
        Slot* s = t.slots + p.slot();
        const u64 old = atomicCAS(&s->key, kEmpty, key);
        if (old == kEmpty || old == key) {
            red_add(&s->count, cnt);
            return old == kEmpty;
        }
        p.next(t);
    }
}

// table_add_cas with one 128-bit CAS that installs key and count together
// ({EMPTY, 0} is the cleared state): a new key costs a single atomic and no
// RED. Faster where most keys are new (KP3's pair inserts, config 5's noise);
// slower for K1's evictions on config 4 (1.586 against 1.550 ms), which keep
// the 64-bit claim.
__device__ __forceinline__ bool table_add_cas128(const Table& t, u64 key, u64 cnt) {
    Probe p(key, t);
    Slot want, empty;
    want.key = key;
    want.count = cnt;
    empty.key = kEmpty;
    empty.count = 0;
    while (true) {
        Slot* s = t.slots + p.slot();
        const Slot old = atomicCAS(s, empty, want);
        if (old.key == kEmpty && old.count == 0) return true;
        if (old.key == key) {
            red_add(&s->count, cnt);
            return false;
        }
        if (old.key == kEmpty) {  // defensive: an empty key with a count takes the 64-bit claim
            const u64 o2 = atomicCAS(&s->key, kEmpty, key);
            if (o2 == kEmpty || o2 == key) {
                red_add(&s->count, cnt);
                return o2 == kEmpty;
            }
        }
        p.next(t);
    }
}

// L2 prefetch of a key's home slot (no register result: fire and forget).
__device__ __forceinline__ void prefetch_slot(const Table& t, u64 key) {
    const Probe p(key, t);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(t.slots + p.slot()));
}

// Lookup: returns the slot's value word, or kEmpty when the key is absent.
// TileCounts::count_of accumulator.hpp:53-61.
__device__ __forceinline__ u64 table_find(const Table& t, u64 key) {
    Probe p(key, t);
    while (true) {
        u64 k, v;
        ld_slot(t.slots + p.slot(), k, v);
        if (k == key) return v;
        if (k == kEmpty) return kEmpty;
        p.next(t);
    }
}

// Claim a slot for a key known to be absent (rehash / load paths); returns
// the slot index.
__device__ __forceinline__ u64 table_claim(const Table& t, u64 key) {
    Probe p(key, t);
    while (true) {
        const u64 i = p.slot();
        const u64 old = atomicCAS(&t.slots[i].key, kEmpty, key);
        if (old == kEmpty || old == key) return i;
        p.next(t);
    }
}

// Cache keys. In the narrow case (every canvas column/row index fits int32,
// checked on the host) the per-warp cache works on the unpacked pair
// (kx << 32 | ky): building it costs no shift, its slot is two bit
// operations, and the table's packed key (kx << bits_y | ky) is formed only
// when an entry leaves the cache. Otherwise the packed key is used
// throughout. Out-of-bounds points get kEmpty (a valid pair has kx < 2^31).
template <bool kNarrow>
struct KeyOps;

template <>
struct KeyOps<true> {
    __device__ static __forceinline__ u64 cache_key(const Grid& g, double x, double y) {
        const int tx = __double2int_rd(__dmul_rn(x, g.scale));
        const int ty = __double2int_rd(__dmul_rn(y, g.scale));
        const u32 kx = (u32)(tx - g.ox32);
        const u32 ky = (u32)(ty - g.oy32);
        return in_bounds(g, x, y) ? (((u64)kx << 32) | ky) : kEmpty;
    }
    // The key without the bounds select (any value for an out-of-bounds
    // point: callers carry the bounds predicate separately).
    __device__ static __forceinline__ u64 raw_key(const Grid& g, double x, double y) {
        const int tx = __double2int_rd(__dmul_rn(x, g.scale));
        const int ty = __double2int_rd(__dmul_rn(y, g.scale));
        return ((u64)(u32)(tx - g.ox32) << 32) | (u32)(ty - g.oy32);
    }
    // Direct-mapped by position in an 8 x 16-tile window (low 3 column bits,
    // low 4 row bits): the few tiles of one cluster never evict each other.
    __device__ static __forceinline__ u32 slot(u64 ck, u32) {
        return (((u32)(ck >> 32) & 7u) << 4) | ((u32)ck & 15u);
    }
    __device__ static __forceinline__ u64 table_key(u64 ck, u32 bits_y) {
        return ck == kEmpty ? kEmpty : (((ck >> 32) << bits_y) | (u32)ck);
    }
};

template <>
struct KeyOps<false> {
    __device__ static __forceinline__ u64 cache_key(const Grid& g, double x, double y) {
        const u64 k = pack_key(g, x, y);
        return in_bounds(g, x, y) ? k : kEmpty;
    }
    __device__ static __forceinline__ u64 raw_key(const Grid& g, double x, double y) {
        return pack_key(g, x, y);
    }
    __device__ static __forceinline__ u32 slot(u64 k, u32 bits_y) {
        return (((u32)(k >> bits_y) & 7u) << 4) | ((u32)k & 15u);
    }
    __device__ static __forceinline__ u64 table_key(u64 k, u32) { return k; }
};

__device__ __forceinline__ u32 match_any64(u64 v) {
    u32 m;
    asm volatile("match.any.sync.b64 %0, %1, 0xffffffff;" : "=r"(m) : "l"(v));
    return m;
}

__device__ __forceinline__ u32 ballot(bool p) {
    u32 m;
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n vote.sync.ballot.b32 %0, q, 0xffffffff;\n}"
        : "=r"(m)
        : "r"((u32)p));
    return m;
}

// Asynchronous 16-byte global->shared copy (LDGSTS), L1-bypassing, with an
// L2 evict-first policy: the points are read exactly once.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, u64 pol) {
    const u32 s = (u32)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Device-side counters of one context (one cache line each to avoid false
// sharing between the hot ones).
struct Counters {
    u64 ticket;          // next work segment (K1 / K4 dynamic scheduling)
    u64 pad0[15];
    u64 used;            // distinct keys in the table
    u64 ingested;        // in-bounds points
    u64 skipped;         // out-of-bounds points
    u64 stopped;         // warps that exhausted their new-key budget
    u64 n_partial;       // partially processed segments recorded
    u64 partial_ticket;  // next partial segment to resume
    u64 pad1[10];
    u64 n_sig;           // significant tiles (K2)
    u64 n_roots;         // components
    u64 n_kept;          // clusters after the mu filter
    u64 first_oob;       // strict policy: smallest out-of-bounds index
    u64 n_edges;         // deferred union edges (K3)
    u64 max_col;         // largest column of significant tiles (sorted K3)
    u64 pad2[10];
};

struct Partial {
    u64 segment;
    u64 next_row;
};

// ---------------------------------------------------- single-pass scans (K2, K3)
// Decoupled look-back (one pass, no library scan): a block takes the next
// tile from a ticket, publishes its aggregate, reads its predecessors'
// published values back to the first inclusive prefix, and publishes its
// own inclusive prefix. Status word: flag (2 bits) << 62 | value.
constexpr u64 kLbAgg = 1ull << 62, kLbPre = 2ull << 62, kLbVal = (1ull << 62) - 1;

__device__ __forceinline__ void lb_store(u64* p, u64 v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 lb_load(const u64* p) {
    u64 v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by one whole warp: the exclusive prefix of `tile` given its
// aggregate. The warp inspects 32 predecessors at a time (each lane waits
// until its predecessor has published something), adds up aggregates back to
// the nearest inclusive prefix, and publishes its own inclusive prefix.
__device__ __forceinline__ u64 lb_prefix(u64* status, u32 tile, u64 agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(status, kLbPre | agg);
        return 0;
    }
    if (lane == 0) lb_store(status + tile, kLbAgg | agg);
    u64 pre = 0;
    for (long long j = (long long)tile - 1;; j -= 32) {
        const long long idx = j - lane;
        u64 v = kLbPre;  // before tile 0: an inclusive prefix of 0
        if (idx >= 0)
            while (((v = lb_load(status + idx)) >> 62) == 0) {
            }
        const u32 pm = __ballot_sync(kFull, (v >> 62) == 2);
        // lanes up to the nearest inclusive prefix (all 32 when none)
        const int last = pm ? __ffs(pm) - 1 : 31;
        u64 x = lane <= last ? (v & kLbVal) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        pre += x;
        if (pm) break;
    }
    if (lane == 0) lb_store(status + tile, kLbPre | (pre + agg));
    return pre;
}

// Block-wide exclusive sum of one u32 per thread (kThr threads); the block
// total through *total.
template <int kThr>
__device__ __forceinline__ u32 block_excl_sum(u32 v, u32* s_warp, u32* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const u32 w = lane < kThr / 32 ? s_warp[lane] : 0;
        u32 wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u32 y = __shfl_up_sync(kFull, wi, d);
            if (lane >= d) wi += y;
        }
        if (lane < kThr / 32) s_warp[lane] = wi - w;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    *total = s_warp[32];
    return s_warp[wid] + incl - v;
}



}  // namespace rg
