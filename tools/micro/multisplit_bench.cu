// Microbenchmark (sm_100a): cost of warp multisplit primitives on random 8-bit digits.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/msb tools/micro/multisplit_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}
__device__ __forceinline__ unsigned peers_ballot(uint32_t d) {
    unsigned p = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const bool bit = (d >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        p &= bit ? bal : ~bal;
    }
    return p;
}
template <int MODE>
__global__ void kern(uint32_t *out, int iters, int spread) {
    __shared__ uint32_t h[256 * 8];
    for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t acc = 0, x = blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5;
    for (int it = 0; it < iters; it++) {
        x = hash(x + it);
        const uint32_t d = spread ? (x & 255u) : ((x & 3u) + 100u);
        if (MODE == 0) acc += __match_any_sync(0xffffffffu, d);
        else if (MODE == 1) acc += peers_ballot(d);
        else if (MODE == 2) atomicAdd(&h[warp * 256 + d], 1u);
        else acc += d;  // baseline: hash only
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = acc + h[threadIdx.x];
}
int main() {
    uint32_t *out;
    cudaMalloc(&out, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    const char *names[] = {"match.any", "8-ballot peers", "smem atomicAdd per-warp", "hash only"};
    for (int spread = 0; spread < 2; spread++)
    for (int m = 0; m < 4; m++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (m == 0) kern<0><<<blocks, threads>>>(out, iters, spread);
            if (m == 1) kern<1><<<blocks, threads>>>(out, iters, spread);
            if (m == 2) kern<2><<<blocks, threads>>>(out, iters, spread);
            if (m == 3) kern<3><<<blocks, threads>>>(out, iters, spread);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double keys = (double)blocks * threads * iters;
            if (rep) printf("%-26s digits=%s  %.3f ms  %.1f Gkeys/s  %.2f clk/warp-op/SM\n", names[m],
                            spread ? "uniform256" : "4 values ", ms, keys / ms / 1e6,
                            ms * 1e-3 * 1.9e9 * 148 / (keys / 32));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
