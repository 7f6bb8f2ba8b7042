// Microbenchmark (sm_100a): CUB device radix sort of float-derived 32-bit keys, for scale.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

int main() {
    const int P = 8, n1 = 1 << 20;
    const int n = P * n1;
    std::vector<uint32_t> h(n);
    uint32_t x = 12345;
    for (int i = 0; i < n; i++) {  // smooth-ish positive floats mapped to keys
        x = x * 1664525u + 1013904223u;
        float f = 0.5f + 0.3f * ((x >> 8) / 16777216.0f - 0.5f);
        uint32_t u; memcpy(&u, &f, 4);
        h[i] = u | 0x80000000u;
    }
    uint32_t *a, *b;
    cudaMalloc(&a, 4 * n); cudaMalloc(&b, 4 * n);
    cudaMemcpy(a, h.data(), 4 * n, cudaMemcpyHostToDevice);
    std::vector<int> off(P + 1);
    for (int i = 0; i <= P; i++) off[i] = i * n1;
    int *doff; cudaMalloc(&doff, 4 * (P + 1));
    cudaMemcpy(doff, off.data(), 4 * (P + 1), cudaMemcpyHostToDevice);
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, a, b, n);
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb2, a, b, n, P, doff, doff + 1);
    void *tmp; cudaMalloc(&tmp, std::max(tb, tb2));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        cub::DeviceRadixSort::SortKeys(tmp, tb, a, b, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("DeviceRadixSort %d keys: %.1f us\n", n, ms * 1e3);
        cudaEventRecord(e0);
        for (int p = 0; p < P; p++) cub::DeviceRadixSort::SortKeys(tmp, tb, a + p * n1, b + p * n1, n1);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("DeviceRadixSort %d x %d keys: %.1f us\n", P, n1, ms * 1e3);
        cudaEventRecord(e0);
        cub::DeviceSegmentedRadixSort::SortKeys(tmp, tb2, a, b, n, P, doff, doff + 1);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("DeviceSegmentedRadixSort %d segs: %.1f us\n", P, ms * 1e3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
