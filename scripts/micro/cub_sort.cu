// Micro-benchmark (comparison point only, not on the product path): CUB's
// onesweep radix sort of (u32 group, i32 attr) pairs at the C2 batch shape,
// to compare per-pass cost with the engine's placement passes.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <cub/cub.cuh>

int main() {
    const int n = 1 << 24;
    std::vector<uint32_t> hk(n);
    std::vector<int32_t> hv(n);
    std::mt19937_64 rng(7);
    // Zipf s=1.0 over 10K groups by inverse CDF
    const int G = 10000;
    std::vector<double> cdf(G);
    double acc = 0;
    for (int i = 0; i < G; ++i) { acc += 1.0 / (i + 1); cdf[i] = acc; }
    std::uniform_real_distribution<double> u(0, acc);
    for (int i = 0; i < n; ++i) {
        const double x = u(rng);
        hk[i] = (uint32_t)(std::lower_bound(cdf.begin(), cdf.end(), x) - cdf.begin());
        hv[i] = (int32_t)(rng() & 0xffff);
    }
    uint32_t *k0, *k1; int32_t *v0, *v1;
    cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, n, 0, 14);
    void* tmp; cudaMalloc(&tmp, tmp_bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int bits_list[] = {7, 8, 14, 16};
    for (int bits : bits_list) {
        for (int i = 0; i < 3; ++i) cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits);
        const int N = 20;
        cudaEventRecord(a);
        for (int i = 0; i < N; ++i) cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, n, 0, bits);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("cub SortPairs n=%d bits=%d: %.1f us per sort\n", n, bits, ms * 1000 / N);
    }
    return 0;
}
