// Shared-memory load throughput on this GPU (the projectors' on-chip roofline):
// every thread issues conflict-free LDS.64 (a half-warp reads 16 consecutive 8-byte words)
// in an unrolled loop.  Read the achieved rate with ncu (l1tex__data_pipe_lsu_wavefronts_mem_shared
// per sm__cycles_elapsed; profiles/r1_smem_roofline.txt): the program itself prints only the time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_bw tools/micro/smem_bw_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) smem_lds64(float *out, int iters, long long *clk) {
    __shared__ float2 buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_float2((float)i, 1.0f);
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    unsigned a = base + 8u * (threadIdx.x & 127);
    float2 acc = make_float2(0.f, 0.f);
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
            float2 v;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a + 1024u * u));
            acc.x += v.x;
            acc.y += v.y;
        }
        a ^= 8u;  // keep the addresses live (still conflict-free)
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    if (acc.x == 12345.f) out[threadIdx.x] = acc.y;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    float *out;
    long long *clk;
    cudaMalloc(&out, 4096);
    const int per_sm = 4, blocks = sms * per_sm, iters = 4096;
    cudaMalloc(&clk, sizeof(long long) * blocks);
    smem_lds64<<<blocks, 256>>>(out, 16, clk);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    smem_lds64<<<blocks, 256>>>(out, iters, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    long long *h = new long long[blocks];
    cudaMemcpy(h, clk, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    long long cmax = 0;
    for (int b = 0; b < blocks; b++) cmax = h[b] > cmax ? h[b] : cmax;
    printf("{\"sms\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"sm_clocks_max\": %lld}\n", sms, per_sm, ms, cmax);
    return 0;
}
