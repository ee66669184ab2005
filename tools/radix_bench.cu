// Microbenchmark: CUB radix sort pairs at config-4 size (8.75M): column-only
// u32 keys (19 bits) vs full u64 keys (37 bits), u32 values.
#include <cstdio>
#include <vector>
#include <random>
#include <cub/device/device_radix_sort.cuh>
typedef unsigned long long u64;
typedef unsigned int u32;
template <typename K>
float run(int n, int bits) {
    std::vector<K> hk(n); std::vector<u32> hv(n);
    std::mt19937_64 r(1);
    for (int i = 0; i < n; ++i) { hk[i] = (K)(r() & ((1ull << bits) - 1)); hv[i] = i; }
    K *k, *k2; u32 *v, *v2;
    cudaMalloc(&k, n * sizeof(K)); cudaMalloc(&k2, n * sizeof(K)); cudaMalloc(&v, n * 4); cudaMalloc(&v2, n * 4);
    cudaMemcpy(k, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice);
    cudaMemcpy(v, hv.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k, k2, v, v2, n, 0, bits);
    void* t; cudaMalloc(&t, tb);
    cub::DeviceRadixSort::SortPairs(t, tb, k, k2, v, v2, n, 0, bits);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) cub::DeviceRadixSort::SortPairs(t, tb, k, k2, v, v2, n, 0, bits);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}
int main() {
    const int n = 8750000;
    printf("u32 keys 19 bits: %.1f us\n", run<u32>(n, 19) * 1e3);
    printf("u32 keys 32 bits: %.1f us\n", run<u32>(n, 32) * 1e3);
    printf("u64 keys 37 bits: %.1f us\n", run<u64>(n, 37) * 1e3);
    printf("u64 keys 1M 37 bits: %.1f us\n", run<u64>(1000000, 37) * 1e3);
    return 0;
}
