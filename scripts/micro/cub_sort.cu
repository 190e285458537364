// Reference point only (not product code): CUB onesweep radix sort times for the
// two sorts of the binning stage at the headline workload sizes.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cub/device/device_radix_sort.cuh>
template <class K>
float bench(int64_t n, int bits, int maxkey) {
    std::vector<K> hk(n); std::vector<uint32_t> hv(n);
    std::mt19937 rng(1);
    for (int64_t i = 0; i < n; ++i) { hk[i] = K(rng() % maxkey); hv[i] = uint32_t(i); }
    K *k0, *k1; uint32_t *v0, *v1;
    cudaMalloc(&k0, n * sizeof(K)); cudaMalloc(&k1, n * sizeof(K));
    cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice);
    cub::DoubleBuffer<K> dk(k0, k1); cub::DoubleBuffer<uint32_t> dv(v0, v1);
    size_t tmp = 0; cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, n, 0, bits);
    void* t; cudaMalloc(&t, tmp);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
        cudaMemcpy(k0, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice);
        dk = cub::DoubleBuffer<K>(k0, k1); dv = cub::DoubleBuffer<uint32_t>(v0, v1);
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, n, 0, bits);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(t);
    return best;
}
int main() {
    printf("cub tile sort   17.3M u16 keys (13 bits) + u32 vals: %.3f ms\n", bench<uint16_t>(17300000, 13, 8160));
    printf("cub depth sort  3M u32 keys (32 bits) + u32 vals:    %.3f ms\n", bench<uint32_t>(3000000, 32, 0x7fffffff));
    printf("cub depth sort  3M u32 keys (26 bits) + u32 vals:    %.3f ms\n", bench<uint32_t>(3000000, 26, 1 << 26));
    return 0;
}
