// partition.cu — contraction for inputs without spatial order (sm_100a).
//
// Same contract as K1 (TileAccumulator::ingest accumulator.hpp:120-134:
// Bounds::contains core.hpp:33-35 -> project_unchecked core.hpp:136-139 ->
// TileCounts::add accumulator.hpp:33-50), for inputs whose consecutive
// points do not share tiles (the reference generator shuffles its output,
// datagen.hpp:224-226). K1's per-warp cache then misses on almost every
// point and each point costs a CAS and a RED on a random table slot. Here
// the points are instead partitioned by tile so that every tile's points
// meet in one block's shared memory:
//
//   KP0 k_part_hist    stream the points once; per 64 Ki-point tile, a
//                      shared-memory histogram of the 2048 partitions;
//   (scan)             partition-major exclusive scan of the histograms:
//                      every (partition, tile) run gets its exact place;
//   KP1 k_part_scatter stream the points again; in 16 Ki-point rounds,
//                      order them by partition in shared memory and write
//                      each point's 32-bit residual key in runs (no global
//                      atomics);
//   KP2 k_part_agg     one block per work unit (up to 256 Ki points of one
//                      partition) counts its residuals in a shared-memory
//                      hash table (16 Ki slots; more rounds when a unit has
//                      more tiles) and writes its (key, count) pairs into
//                      its own slab;
//   KP3 k_part_insert  folds the pairs into the HBM table (one CAS + RED per
//                      distinct tile of a unit), after the host has grown
//                      the table to fit them.
//
// Config 4 in a random order: 9.2 ms per step against 21.7 ms with K1 (whose
// cache then misses on every point). Ordered inputs keep K1 (an order probe
// in api.cu decides).
//
// A partition is the low 11 bits of a bijective mix of the packed key
// (multiply by an odd constant mod 2^B, then xor-shift by ceil(B/2)); the
// other B-11 bits are the residual, so the key is recovered exactly. A unit
// holds at most 256 Ki points, so 32 rounds of 12 Ki tiles always suffice;
// the per-point fallback (a unit KP2 flags as overflowed, whose points KP3
// adds one by one) is exercised with RG_PART_MAX_ROUNDS=1 in the tests.
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.h"

namespace rg {

namespace {

constexpr u32 kPBits = 11;
constexpr u32 kParts = 1u << kPBits;
constexpr u64 kPTile = 65536;          // points per histogram tile
constexpr int kPThreads = 512;
constexpr int kPSub = 8;               // points per thread per sub-chunk
constexpr u32 kPSubN = kPThreads * kPSub;
constexpr u32 kAggSlots = 1u << 14;    // shared-memory hash table (KP2)
constexpr u32 kAggMax = 12288;         // distinct tiles per round (75 % load)
constexpr u32 kMaxRounds = 64;
constexpr u32 kOverflow = 0xffffffffu;

struct Mix {
    u64 mul, inv, mask;
    u32 shift;
};

__device__ __forceinline__ u64 mix(const Mix& m, u64 k) {
    const u64 h = (k * m.mul) & m.mask;
    return h ^ (h >> m.shift);
}

__device__ __forceinline__ u64 unmix(const Mix& m, u64 h) {
    h ^= h >> m.shift;  // 2 * shift >= B: the xor-shift is its own inverse
    return (h * m.inv) & m.mask;
}

// Point load that stays in L2 for a second read (KP1's placement pass).
__device__ __forceinline__ double2 ld_point_keep(const double2* p, u64 pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ bool point_key(const Grid& g, double2 v, u64& key) {
    key = pack_key(g, v.x, v.y);
    return in_bounds(g, v.x, v.y);
}

// KP0: per-tile partition histograms, stored partition-major (M[p * T + t]).
__global__ void __launch_bounds__(kPThreads) k_part_hist(const double2* xy, u64 n, Grid g, Mix m,
                                                         u32* hist_pt, u64 T, Counters* ctr) {
    __shared__ u32 hist[kParts];
    const u64 pol = evict_first_policy();
    u64 in = 0, out = 0;
    for (u64 t = blockIdx.x; t < T; t += gridDim.x) {
        for (u32 i = threadIdx.x; i < kParts; i += kPThreads) hist[i] = 0;
        __syncthreads();
        const u64 p0 = t * kPTile, p1 = min(n, p0 + kPTile);
        for (u64 b = p0; b < p1; b += 4 * kPThreads) {
            double2 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const u64 i = b + j * kPThreads + threadIdx.x;
                v[j] = i < p1 ? ld_point_stream(xy + i, pol)
                              : make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                u64 k;
                if (point_key(g, v[j], k)) {
                    atomicAdd(&hist[(u32)mix(m, k) & (kParts - 1)], 1u);
                    ++in;
                } else if (b + j * kPThreads + threadIdx.x < p1) {
                    ++out;  // out of bounds or NaN: skipped (accumulator.hpp:122-128)
                }
            }
        }
        __syncthreads();
        for (u32 p = threadIdx.x; p < kParts; p += kPThreads) hist_pt[p * T + t] = hist[p];
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        in += __shfl_xor_sync(kFull, in, o);
        out += __shfl_xor_sync(kFull, out, o);
    }
    if ((threadIdx.x & 31) == 0 && in) atomicAdd(&ctr->ingested, in);
    if ((threadIdx.x & 31) == 0 && out) atomicAdd(&ctr->skipped, out);
}

// Block-wide exclusive scan of kParts counters (kParts / kThr per thread).
template <int kThr>
__device__ __forceinline__ void block_scan_parts(const u32* in, u32* out, u32* wsum) {
    constexpr int kI = kParts / kThr;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 v[kI], s = 0;
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        v[j] = in[kI * threadIdx.x + j];
        s += v[j];
    }
    u32 incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        u32 w = lane < kThr / 32 ? wsum[lane] : 0, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kThr / 32) wsum[lane] = wi - w;
    }
    __syncthreads();
    u32 ex = wsum[wid] + incl - s;
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        out[kI * threadIdx.x + j] = ex;
        ex += v[j];
    }
}

// KP1 stages kSubN points per round (2 x 8192): points are read twice per
// round (histogram, then placement; the second read hits L2), so that each
// partition's run of residuals averages 8 entries (one 32-byte sector) and
// the O(partitions) bookkeeping is paid once per 16 Ki points.
#ifndef RG_KP1_THREADS
#define RG_KP1_THREADS 1024
#endif
#ifndef RG_KP1_STEPS
#define RG_KP1_STEPS 2
#endif
#ifndef RG_KP1_BLOCKS
#define RG_KP1_BLOCKS 1
#endif
constexpr int kP1Thr = RG_KP1_THREADS;
constexpr u32 kP1SubN = kP1Thr * kPSub;  // points per pass step
constexpr u32 kSubN = RG_KP1_STEPS * kP1SubN;
constexpr size_t kScatterSmem = (5 * kParts + kSubN + kP1Thr / 32) * 4 + kSubN * 2;
static_assert(kParts % kP1Thr == 0 && kParts % kPThreads == 0, "partition scan layout");

// KP1: every in-bounds point's residual, written at its partition's place.
__global__ void __launch_bounds__(kP1Thr, RG_KP1_BLOCKS) k_part_scatter(const double2* xy, u64 n, Grid g,
                                                            Mix m, const u32* off_pt, u64 T,
                                                            u32* res) {
    extern __shared__ u32 sh_sc[];  // kScatterSmem bytes
    u32* cur = sh_sc;               // next global position per partition (this tile)
    u32* hist = cur + kParts;       // this round's points per partition
    u32* loff = hist + kParts;      // exclusive prefix of hist
    u32* lcur = loff + kParts;      // placement cursors
    u32* pend = lcur + kParts;      // end of each partition's global range
    u32* stage = pend + kParts;
    u32* wsum = stage + kSubN;
    unsigned short* spart = (unsigned short*)(wsum + kP1Thr / 32);
    const u64 pol = evict_first_policy();
    u64 pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    for (u64 t = blockIdx.x; t < T; t += gridDim.x) {
        for (u32 p = threadIdx.x; p < kParts; p += kP1Thr) {
            cur[p] = off_pt[p * T + t];
            pend[p] = off_pt[(p + 1) * T];  // (p + 1) * T = kParts * T: the total
        }
        const u64 p0 = t * kPTile, p1 = min(n, p0 + kPTile);
        for (u64 q0 = p0; q0 < p1; q0 += kSubN) {
            const u64 q1 = min(p1, q0 + kSubN);
            for (u32 p = threadIdx.x; p < kParts; p += kP1Thr) hist[p] = 0;
            __syncthreads();
            for (u64 b = q0; b < q1; b += kP1SubN) {  // pass a: histogram
                double2 v[kPSub];
#pragma unroll
                for (int j = 0; j < kPSub; ++j) {
                    const u64 i = b + j * kP1Thr + threadIdx.x;
                    v[j] = i < q1 ? ld_point_keep(xy + i, pol_keep)  // kept in L2 for pass b
                                  : make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
                }
#pragma unroll
                for (int j = 0; j < kPSub; ++j) {
                    u64 k;
                    if (point_key(g, v[j], k)) atomicAdd(&hist[(u32)mix(m, k) & (kParts - 1)], 1u);
                }
            }
            __syncthreads();
            block_scan_parts<kP1Thr>(hist, loff, wsum);
            __syncthreads();
            for (u32 p = threadIdx.x; p < kParts; p += kP1Thr) lcur[p] = loff[p];
            __syncthreads();
            for (u64 b = q0; b < q1; b += kP1SubN) {  // pass b: placement
                double2 v[kPSub];
#pragma unroll
                for (int j = 0; j < kPSub; ++j) {
                    const u64 i = b + j * kP1Thr + threadIdx.x;
                    v[j] = i < q1 ? ld_point_stream(xy + i, pol)
                                  : make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
                }
#pragma unroll
                for (int j = 0; j < kPSub; ++j) {
                    u64 k;
                    if (point_key(g, v[j], k)) {
                        const u64 h = mix(m, k);
                        const u32 part = (u32)h & (kParts - 1);
                        const u32 at = atomicAdd(&lcur[part], 1u);
                        stage[at] = (u32)(h >> kPBits);
                        spart[at] = (unsigned short)part;
                    }
                }
            }
            __syncthreads();
            const u32 cnt = loff[kParts - 1] + hist[kParts - 1];
            for (u32 i = threadIdx.x; i < cnt; i += kP1Thr) {
                const u32 part = spart[i];
                const u32 at = cur[part] + (i - loff[part]);
                // KP0 counted exactly these points; the guard only matters if
                // the buffer changed between the two passes (a caller race)
                if (at < pend[part]) res[at] = stage[i];
            }
            __syncthreads();
            for (u32 p = threadIdx.x; p < kParts; p += kP1Thr) cur[p] += hist[p];
            __syncthreads();
        }
    }
}

// Round of a residual when a unit's tiles do not fit one shared-memory
// table: rounds split the residuals by a hash, R rounds (a power of two).
__device__ __forceinline__ u32 round_of(u32 r, u32 R) { return ((r * 0x85EBCA6Bu) >> 16) & (R - 1); }

// Insert `c` occurrences of residual r into the shared-memory table.
__device__ __forceinline__ void agg_insert(u32* skey, u32* scnt, u32* occ, u32* over, u32 r,
                                           u32 c) {
    const u32 k = r + 1;
    u32 s = (r * 0x9E3779B1u) >> (32 - 14);
    for (u32 probes = 0;; ++probes) {
        if (probes == kAggSlots) {  // full table: the unit is redone in more rounds
            *over = 1;
            return;
        }
        const u32 cur = skey[s];
        if (cur == k) {
            atomicAdd(&scnt[s], c);
            return;
        }
        if (cur == 0) {
            const u32 old = atomicCAS(&skey[s], 0u, k);
            if (old == 0) {
                atomicAdd(&scnt[s], c);
                if (atomicAdd(occ, 1u) >= kAggMax) *over = 1;
                return;
            }
            if (old == k) {
                atomicAdd(&scnt[s], c);
                return;
            }
        }
        s = (s + 1) & (kAggSlots - 1);
    }
}

// KP2: count a work unit's residuals (at most kUnit points of one
// partition; a hot partition is split into several units, whose pairs KP3
// adds up) in a shared-memory hash table, and write its (key, count) pairs
// into the unit's own slab of the pair arrays (pair index space = residual
// index space, so slabs never overlap: a unit has at most as many distinct
// tiles as points). A unit whose tiles overflow one table is redone in R
// rounds (doubling), each taking the residuals of one hash class; dcnt[u]
// is the unit's number of pairs (kOverflow past max_rounds: KP3 then adds
// its points one by one).
constexpr int kAggThreads = 1024;
static_assert(kAggThreads % 32 == 0, "whole warps");
__global__ void __launch_bounds__(kAggThreads, 1) k_part_agg(const u32* res, const uint4* units,
                                                             u32 n_units, Mix m, u32 max_rounds,
                                                             u32* dcnt, u64* pkey, u32* pcnt) {
    extern __shared__ u32 sh_agg[];
    u32* skey = sh_agg;  // residual + 1, 0 = empty
    u32* scnt = sh_agg + kAggSlots;
    __shared__ u32 occ, over, wpos;
    for (u32 u = blockIdx.x; u < n_units; u += gridDim.x) {
        const uint4 w = units[u];
        const u32 lo = w.x, hi = w.y, p = w.z;
        u32 R = 1, total = 0;
        while (true) {
            bool ok = true;
            total = 0;
            for (u32 rr = 0; rr < R && ok; ++rr) {
                for (u32 i = threadIdx.x; i < kAggSlots; i += kAggThreads) {
                    skey[i] = 0;
                    scnt[i] = 0;
                }
                if (threadIdx.x == 0) {
                    occ = 0;
                    over = 0;
                    wpos = 0;
                }
                __syncthreads();
                constexpr int kPf = 8;  // residuals per thread in flight
                for (u32 i0 = lo; i0 < hi; i0 += kAggThreads * kPf) {
                    // warp-uniform exit (no barrier inside the loop)
                    if (__any_sync(kFull, *(volatile u32*)&over != 0)) break;
                    u32 rv[kPf];
#pragma unroll
                    for (int j = 0; j < kPf; ++j) {
                        const u32 i = i0 + j * kAggThreads + threadIdx.x;
                        rv[j] = i < hi ? res[i] : 0xffffffffu;
                    }
#pragma unroll
                    for (int j = 0; j < kPf; ++j) {
                        const u32 r = rv[j];
                        if (r != 0xffffffffu && (R == 1 || round_of(r, R) == rr))
                            agg_insert(skey, scnt, &occ, &over, r, 1u);
                    }
                }
                __syncthreads();
                if (over) {
                    ok = false;
                } else {
                    const u64 o = (u64)lo + total;
                    for (u32 i = threadIdx.x; i < kAggSlots; i += kAggThreads) {
                        if (skey[i]) {
                            const u64 at = o + atomicAdd(&wpos, 1u);
                            pkey[at] = unmix(m, ((u64)(skey[i] - 1) << kPBits) | p);
                            pcnt[at] = scnt[i];
                        }
                    }
                    total += occ;
                }
                __syncthreads();
            }
            if (ok || R >= max_rounds) {
                if (!ok) total = kOverflow;
                break;
            }
            R *= 2;
        }
        if (threadIdx.x == 0) dcnt[u] = total;
        __syncthreads();
    }
}

// KP3: fold each unit's pairs into the table (one block per unit, so the CAS
// round trips of a block overlap).
__global__ void __launch_bounds__(256) k_part_insert(const uint4* units, u32 n_units,
                                                     const u32* dcnt, const u64* pkey,
                                                     const u32* pcnt, Table t, Counters* ctr) {
    u32 claims = 0;
    for (u32 u = blockIdx.x; u < n_units; u += gridDim.x) {
        const u32 d = dcnt[u];
        if (d == kOverflow) continue;
        const u64 lo = units[u].x;
        for (u32 i = threadIdx.x; i < d; i += blockDim.x)
            claims += table_add_cas(t, pkey[lo + i], pcnt[lo + i]) ? 1u : 0u;
    }
    claims = __reduce_add_sync(kFull, claims);
    if ((threadIdx.x & 31) == 0 && claims) atomicAdd(&ctr->used, (u64)claims);
}

__global__ void k_part_insert_raw(const u32* res, u32 b0, u32 b1, u32 p, Mix m, Table t,
                                  Counters* ctr) {
    u32 claims = 0;
    for (u64 i = b0 + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < b1;
         i += (u64)gridDim.x * blockDim.x)
        claims += table_add(t, unmix(m, ((u64)res[i] << kPBits) | p), 1) ? 1u : 0u;
    claims = __reduce_add_sync(__activemask(), claims);
    if ((threadIdx.x & 31) == 0 && claims) atomicAdd(&ctr->used, (u64)claims);
}

// Order probe: distinct tiles among 2048 consecutive points, per sample.
__global__ void __launch_bounds__(256) k_order_probe(const double2* xy, u64 n, Grid g, u64 stride,
                                                     u64* out) {
    __shared__ u64 keys[4096];
    __shared__ u32 distinct, valid;
    for (u32 i = threadIdx.x; i < 4096; i += 256) keys[i] = kEmpty;
    if (threadIdx.x == 0) distinct = valid = 0;
    __syncthreads();
    const u64 b = blockIdx.x * stride;
    for (u32 j = threadIdx.x; j < 2048; j += 256) {
        const u64 i = b + j;
        if (i >= n) break;
        u64 k;
        if (!point_key(g, xy[i], k)) continue;
        atomicAdd(&valid, 1u);
        u32 s = (u32)((k * 0x9E3779B97F4A7C15ull) >> 52);
        while (true) {
            const u64 old = atomicCAS(&keys[s], kEmpty, k);
            if (old == kEmpty) {
                atomicAdd(&distinct, 1u);
                break;
            }
            if (old == k) break;
            s = (s + 1) & 4095;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(out, (u64)distinct);
        atomicAdd(out + 1, (u64)valid);
    }
}

Mix make_mix(u32 bits) {
    Mix m;
    m.mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    m.mul = 0x9E3779B97F4A7C15ull & m.mask;
    m.mul |= 1;  // odd: invertible mod 2^bits
    u64 inv = m.mul;  // Newton: inv = inv * (2 - mul * inv), doubling correct bits
    for (int i = 0; i < 6; ++i) inv *= 2 - m.mul * inv;
    m.inv = inv & m.mask;
    m.shift = (bits + 1) / 2;
    return m;
}

}  // namespace

bool partition_ingest_supported(u32 key_bits, u64 n) {
    return key_bits >= 20 && key_bits <= 42 && n < (1ull << 31);
}

constexpr u32 kUnit = 1u << 18;  // points per KP2 work unit (hot partitions are split)

u64 max_units(u64 n) { return kParts + n / kUnit + 2; }

// scratch: residuals (4 B / point), per-(partition, tile) counts and
// offsets, partition bases, work units with their rounds / distinct counts /
// pair offsets, scan temp.
size_t partition_scratch_bytes(u64 n, size_t* scan_temp) {
    const u64 T = (n + kPTile - 1) / kPTile;
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum((void*)nullptr, tb, (const u32*)nullptr, (u32*)nullptr,
                                  (int)(kParts * T + 1));
    *scan_temp = tb;
    const u64 U = max_units(n);
    return n * 4 + 2 * (kParts * T + 1) * 4 + (kParts + 1) * 4 + U * 16 + 2 * U * 4 +
           (U + 1) * 8 + tb + 4096;
}

u32 partition_count() { return kParts; }

cudaError_t launch_order_probe(const double* xy, u64 n, Grid g, u64* out, int n_sm,
                               cudaStream_t st) {
    (void)n_sm;
    const u64 samples = 64;
    const u64 stride = n / samples;
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(u64), st);
    if (e != cudaSuccess) return e;
    k_order_probe<<<(int)samples, 256, 0, st>>>(reinterpret_cast<const double2*>(xy), n, g,
                                                stride, out);
    return cudaGetLastError();
}

namespace {
struct Carve {
    u32 *res, *hist, *off, *base, *rounds, *dcnt;
    uint4* units;
    u64* pair_off;
    void* temp;
};
Carve carve(void* scratch, u64 n) {
    const u64 T = (n + kPTile - 1) / kPTile;
    const u64 U = max_units(n);
    Carve c;
    char* w = (char*)scratch;
    c.res = (u32*)w;
    w += n * 4;
    c.hist = (u32*)w;
    w += (kParts * T + 1) * 4;
    c.off = (u32*)w;
    w += (kParts * T + 1) * 4;
    c.base = (u32*)w;
    w += (kParts + 1) * 4;
    w = (char*)(((uintptr_t)w + 15) & ~(uintptr_t)15);
    c.units = (uint4*)w;
    w += U * 16;
    c.rounds = (u32*)w;
    w += U * 4;
    c.dcnt = (u32*)w;
    w += U * 4;
    w = (char*)(((uintptr_t)w + 7) & ~(uintptr_t)7);
    c.pair_off = (u64*)w;
    w += (U + 1) * 8;
    c.temp = (void*)(((uintptr_t)w + 255) & ~(uintptr_t)255);
    return c;
}
}  // namespace

// Phase 1: KP0, scan, work units (host), KP1, KP2 counting; fills the plan
// (units, distinct counts, pair offsets, points of overflowed units).
cudaError_t launch_partition_count(const PartitionLaunch& L, cudaStream_t st, PartitionPlan* plan) {
    const u64 n = L.n;
    const u64 T = (n + kPTile - 1) / kPTile;
    const Mix m = make_mix(L.key_bits);
    const Carve c = carve(L.scratch, n);
    const double2* xy = reinterpret_cast<const double2*>(L.xy);
    cudaError_t e;
    if ((e = cudaMemsetAsync(c.hist + kParts * T, 0, 4, st)) != cudaSuccess) return e;
    const int g0 = (int)std::min<u64>(T, (u64)L.n_sm * 4);
    k_part_hist<<<g0, kPThreads, 0, st>>>(xy, n, L.g, m, c.hist, T, L.ctr);
    size_t tb = L.scan_temp;
    if ((e = cub::DeviceScan::ExclusiveSum(c.temp, tb, c.hist, c.off, (int)(kParts * T + 1), st)) !=
        cudaSuccess)
        return e;
    // partition bases: off[p * T] (the total is off[kParts * T])
    if ((e = cudaMemcpy2DAsync(c.base, 4, c.off, T * 4, 4, kParts + 1, cudaMemcpyDeviceToDevice,
                               st)) != cudaSuccess)
        return e;
    static bool attr = false;
    const int sm2 = (int)(2 * kAggSlots * sizeof(u32));
    if (!attr) {
        cudaFuncSetAttribute(k_part_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kScatterSmem);
        cudaFuncSetAttribute(k_part_agg, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
        attr = true;
    }
    // (a direct variant - one block per 64 Ki-point tile storing each
    // residual straight to its run with a shared-memory cursor, relying on
    // L2 to merge the 4-byte stores - measured 13.8 ms: 7.85 GB of DRAM
    // writes for 2 GB of residuals)
    k_part_scatter<<<(int)std::min<u64>(T, (u64)L.n_sm * RG_KP1_BLOCKS), kP1Thr, kScatterSmem, st>>>(
        xy, n, L.g, m, c.off, T, c.res);
    std::vector<u32> base(kParts + 1);
    if ((e = cudaMemcpyAsync(base.data(), c.base, (kParts + 1) * 4, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    plan->units.clear();
    for (u32 p = 0; p < kParts; ++p)
        for (u32 lo = base[p]; lo < base[p + 1]; lo += kUnit)
            plan->units.push_back(make_uint4(lo, std::min(base[p + 1], lo + kUnit), p, 0));
    const u32 U = (u32)plan->units.size();
    plan->dcnt.assign(U, 0);
    plan->pair_off.assign(U + 1, 0);
    plan->raw_points = 0;
    if (U == 0) return cudaSuccess;
    if ((e = cudaMemcpyAsync(c.units, plan->units.data(), U * sizeof(uint4), cudaMemcpyHostToDevice,
                             st)) != cudaSuccess)
        return e;
    static const u32 max_rounds = [] {  // RG_PART_MAX_ROUNDS: test knob for the raw path
        const char* v = std::getenv("RG_PART_MAX_ROUNDS");
        const int r = v ? std::atoi(v) : 0;
        return r >= 1 && r <= (int)kMaxRounds ? (u32)r : kMaxRounds;
    }();
    const int g2 = (int)std::min<u32>(U, (u32)L.n_sm);
    k_part_agg<<<g2, kAggThreads, sm2, st>>>(c.res, c.units, U, m, max_rounds, c.dcnt, L.pkey,
                                             L.pcnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(plan->dcnt.data(), c.dcnt, U * 4, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
        return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    for (u32 u = 0; u < U; ++u) {
        const bool ov = plan->dcnt[u] == kOverflow;
        plan->pair_off[u + 1] = plan->pair_off[u] + (ov ? 0 : plan->dcnt[u]);
        if (ov) plan->raw_points += plan->units[u].y - plan->units[u].x;
    }
    return cudaSuccess;
}

// Phase 2: KP3 folding the pairs (and the raw points of overflowed units)
// into the table.
cudaError_t launch_partition_insert(const PartitionLaunch& L, Table t, const PartitionPlan& plan,
                                    cudaStream_t st) {
    const u64 n = L.n;
    const Mix m = make_mix(L.key_bits);
    const Carve c = carve(L.scratch, n);
    const u32 U = (u32)plan.units.size();
    if (U == 0) return cudaSuccess;
    k_part_insert<<<(int)std::min<u32>(U, (u32)L.n_sm * 8), 256, 0, st>>>(c.units, U, c.dcnt,
                                                                          L.pkey, L.pcnt, t,
                                                                          L.ctr);
    for (u32 u = 0; u < U; ++u)
        if (plan.dcnt[u] == kOverflow)
            k_part_insert_raw<<<L.n_sm, 256, 0, st>>>(c.res, plan.units[u].x, plan.units[u].y,
                                                     plan.units[u].z, m, t, L.ctr);
    return cudaGetLastError();
}

}  // namespace rg
