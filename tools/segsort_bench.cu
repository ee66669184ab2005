// Microbenchmark: CUB segmented sort of config-4-shaped data (8.75M items in
// 360K segments of ~24) with 64-bit vs 32-bit keys.
#include <cstdio>
#include <vector>
#include <random>
#include <cub/device/device_segmented_sort.cuh>
typedef unsigned long long u64;
typedef unsigned int u32;
template <typename K>
float run(const std::vector<u32>& off, int n, int segs) {
    std::vector<K> hk(n);
    std::vector<u32> hv(n);
    std::mt19937_64 r(1);
    for (int i = 0; i < n; ++i) { hk[i] = (K)(r() & 0x3ffff); hv[i] = i; }
    K *k, *k2; u32 *v, *v2, *o;
    cudaMalloc(&k, n * sizeof(K)); cudaMalloc(&k2, n * sizeof(K));
    cudaMalloc(&v, n * 4); cudaMalloc(&v2, n * 4); cudaMalloc(&o, (segs + 1) * 4);
    cudaMemcpy(k, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice);
    cudaMemcpy(v, hv.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(o, off.data(), (segs + 1) * 4, cudaMemcpyHostToDevice);
    size_t tb = 0;
    cub::DeviceSegmentedSort::SortPairs(nullptr, tb, k, k2, v, v2, n, segs, o, o + 1);
    void* t; cudaMalloc(&t, tb);
    cub::DeviceSegmentedSort::SortPairs(t, tb, k, k2, v, v2, n, segs, o, o + 1);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) cub::DeviceSegmentedSort::SortPairs(t, tb, k, k2, v, v2, n, segs, o, o + 1);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaFree(k); cudaFree(k2); cudaFree(v); cudaFree(v2); cudaFree(o); cudaFree(t);
    return ms / 10;
}
int main() {
    const int segs = 360000;
    std::mt19937_64 r(7);
    std::poisson_distribution<int> p(24.3);
    std::vector<u32> off(segs + 1, 0);
    for (int s = 0; s < segs; ++s) off[s + 1] = off[s] + p(r);
    const int n = off[segs];
    printf("n=%d segs=%d\n", n, segs);
    printf("u64 keys: %.1f us\n", run<u64>(off, n, segs) * 1e3);
    printf("u32 keys: %.1f us\n", run<u32>(off, n, segs) * 1e3);
    return 0;
}
