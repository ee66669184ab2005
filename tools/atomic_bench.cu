// Microbenchmark: random 64-bit atomics (CAS-then-add, as a hash-table
// insert) into a region of a given size. Used to size the partitioned
// contraction design (L2-resident vs HBM-resident table regions).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mix(u64 v) {
    v ^= v >> 30; v *= 0xbf58476d1ce4e5b9ull; v ^= v >> 27; v *= 0x94d049bb133111ebull; return v ^ (v >> 31);
}
__global__ void k(u64* slots, u64 mask, u64 n, int mode) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 h = mix(i);
        const u64 s = (h & mask) * 2;
        if (mode == 0) {
            atomicAdd(slots + s + 1, 1ull);
        } else {
            const u64 key = (h >> 20) | 1;
            const u64 old = atomicCAS(slots + s, 0ull, key);
            (void)old;
            atomicAdd(slots + s + 1, 1ull);
        }
    }
}
int main() {
    const u64 n = 500000000ull;
    for (int mode = 0; mode < 2; ++mode)
        for (u64 region_slots : {1ull << 17, 1ull << 20, 1ull << 22, 1ull << 25}) {
            u64* d;
            cudaMalloc(&d, region_slots * 16);
            cudaMemset(d, 0, region_slots * 16);
            k<<<148 * 16, 256>>>(d, region_slots - 1, n / 10, mode);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<148 * 16, 256>>>(d, region_slots - 1, n, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("mode %s region %llu slots (%.1f MB): %.2f ms = %.1f G ops/s\n", mode ? "cas+add" : "add",
                   region_slots, region_slots * 16 / 1e6, ms, n / ms / 1e6);
            cudaFree(d);
        }
    return 0;
}
