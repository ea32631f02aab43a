// Calibration only (not product): CUB DeviceRadixSort time for the two sorts at C2 sizes.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main() {
    const int V = 1000000, P = 3569504;
    std::mt19937_64 g(1);
    std::vector<unsigned long long> k64(V); std::vector<unsigned> k32(P), v(P);
    for (int i = 0; i < V; ++i) { double d = 1.1 + 1.8 * (g() >> 11) * 0x1.0p-53; memcpy(&k64[i], &d, 8); }
    for (int i = 0; i < P; ++i) { k32[i] = g() % 8160; v[i] = i; }
    unsigned long long *dk, *dk2; unsigned *dv, *dv2, *dk3, *dk4;
    cudaMalloc(&dk, 8*V); cudaMalloc(&dk2, 8*V); cudaMalloc(&dv, 4*P); cudaMalloc(&dv2, 4*P); cudaMalloc(&dk3, 4*P); cudaMalloc(&dk4, 4*P);
    cudaMemcpy(dk, k64.data(), 8*V, cudaMemcpyHostToDevice);
    cudaMemcpy(dk3, k32.data(), 4*P, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), 4*P, cudaMemcpyHostToDevice);
    size_t t1 = 0, t2 = 0; void* tmp;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, dk, dk2, dv, dv2, V, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, dk3, dk4, dv, dv2, P, 0, 13);
    cudaMalloc(&tmp, t1 > t2 ? t1 : t2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bits : {64, 53, 32}) {
      for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t1, dk, dk2, dv, dv2, V, 0, bits);
        cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        if (it == 2) printf("depth sort V=%d bits=%d: %.1f us\n", V, bits, ms * 1000);
      }
    }
    unsigned *k32a; cudaMalloc(&k32a, 4*V);
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t1, k32a, dk4, dv, dv2, V, 0, 32);
        cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        if (it == 2) printf("32-bit key sort V=%d: %.1f us\n", V, ms * 1000);
    }
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(tmp, t2, dk3, dk4, dv, dv2, P, 0, 13);
        cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
        if (it == 2) printf("tile sort P=%d bits=13: %.1f us\n", P, ms * 1000);
    }
    return 0;
}
