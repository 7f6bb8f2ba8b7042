// Kernel-boundary cost inside a CUDA graph, with and without programmatic dependent launch
// (PDL): a chain of NK dependent kernels, each streaming `n` floats (y = a*x + y), captured
// into a graph and replayed.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void axpy(const float *__restrict__ x, float *__restrict__ y, long long n, float a, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = a * x[i] + y[i];
    if (pdl == 2) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
    const int NK = 40;
    for (long long n : {1LL << 16, 1LL << 20, 1LL << 22}) {
        float *x, *y;
        cudaMalloc(&x, n * 4); cudaMalloc(&y, n * 4);
        cudaMemset(x, 0, n * 4); cudaMemset(y, 0, n * 4);
        cudaStream_t s; cudaStreamCreate(&s);
        const int blocks = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
        for (int pdl = 0; pdl < 3; pdl++) {
            cudaGraph_t g; cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < NK; k++) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = blocks; cfg.blockDim = 256; cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
                cudaLaunchKernelEx(&cfg, axpy, (const float *)x, y, n, 1.0f, pdl);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int w = 0; w < 5; w++) cudaGraphLaunch(ge, s);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            for (int r = 0; r < 50; r++) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("n=%lld pdl=%d  %.2f us per kernel  (%s)\n", n, pdl, ms * 1e3 / 50 / NK,
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
        }
        cudaFree(x); cudaFree(y);
    }
    return 0;
}
