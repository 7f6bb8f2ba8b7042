// vec.cu -- see vec.cuh.
#include "vec.cuh"

namespace tq {

namespace {
constexpr int VT = 256;  // threads
constexpr int VE = 4;    // elements per thread
}

int vec_blocks(long long n) { return ceil_div(n, (long long)VT * VE); }

template <typename T>
__global__ void __launch_bounds__(VT) cg_update_xr(T *x, T *r, const T *p, const T *q, long long n,
                                                   double *scal, double *partial, int part_stride,
                                                   unsigned *counter) {
    __shared__ double red[VT / 32 + 1];
    __shared__ bool last;
    const int node = blockIdx.y;
    const long long base = (long long)node * n;
    double *sc = scal + (long long)node * S_NSLOT;
    const double alpha = sc[S_ALPHA];
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < VE; e++) {
        const long long i = (long long)blockIdx.x * VT * VE + e * VT + threadIdx.x;
        if (i < n) {
            const long long g = base + i;
            x[g] = (T)((double)x[g] + alpha * (double)p[g]);
            const T rv = (T)((double)r[g] - alpha * (double)q[g]);
            r[g] = rv;
            dot += (double)rv * (double)rv;
        }
    }
    const double bs = block_sum<VT>(dot, red);
    double *part = partial + (long long)node * part_stride;
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block_of_group(counter + node, gridDim.x, &last)) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += VT) s += part[b];
        s = block_sum<VT>(s, red);
        if (threadIdx.x == 0) {
            const double rr = sc[S_RR];
            sc[S_RRNEW] = s;
            sc[S_BETA] = rr > 0.0 ? s / rr : 0.0;
            sc[S_RR] = s;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(VT) cg_update_p(T *p, const T *r, long long n, const double *scal) {
    const int node = blockIdx.y;
    const long long base = (long long)node * n;
    const double beta = scal[(long long)node * S_NSLOT + S_BETA];
#pragma unroll
    for (int e = 0; e < VE; e++) {
        const long long i = (long long)blockIdx.x * VT * VE + e * VT + threadIdx.x;
        if (i < n) {
            const long long g = base + i;
            p[g] = (T)((double)r[g] + beta * (double)p[g]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(VT) norm2_kernel(const T *x, long long n, double *scal, double *partial,
                                                   int part_stride, unsigned *counter) {
    __shared__ double red[VT / 32 + 1];
    __shared__ bool last;
    const int node = blockIdx.y;
    const long long base = (long long)node * n;
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < VE; e++) {
        const long long i = (long long)blockIdx.x * VT * VE + e * VT + threadIdx.x;
        if (i < n) {
            const double v = (double)x[base + i];
            dot += v * v;
        }
    }
    const double bs = block_sum<VT>(dot, red);
    double *part = partial + (long long)node * part_stride;
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block_of_group(counter + node, gridDim.x, &last)) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += VT) s += part[b];
        s = block_sum<VT>(s, red);
        if (threadIdx.x == 0) scal[(long long)node * S_NSLOT + S_NORM] = s;
    }
}

template <typename A, typename B>
__global__ void convert_kernel(const A *src, B *dst, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (B)src[i];
}

void launch_cg_update_xr(int prec, void *x, void *r, const void *p, const void *q, long long n,
                         int L, double *scal, double *partial, int part_stride, unsigned *counter,
                         cudaStream_t st) {
    dim3 grid(vec_blocks(n), L);
    if (prec == 0)
        cg_update_xr<float><<<grid, VT, 0, st>>>((float *)x, (float *)r, (const float *)p,
                                                 (const float *)q, n, scal, partial, part_stride, counter);
    else
        cg_update_xr<double><<<grid, VT, 0, st>>>((double *)x, (double *)r, (const double *)p,
                                                  (const double *)q, n, scal, partial, part_stride, counter);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_cg_update_p(int prec, void *p, const void *r, long long n, int L, const double *scal,
                        cudaStream_t st) {
    dim3 grid(vec_blocks(n), L);
    if (prec == 0) cg_update_p<float><<<grid, VT, 0, st>>>((float *)p, (const float *)r, n, scal);
    else cg_update_p<double><<<grid, VT, 0, st>>>((double *)p, (const double *)r, n, scal);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_norm2(int prec, const void *x, long long n, int L, double *scal, double *partial,
                  int part_stride, unsigned *counter, cudaStream_t st) {
    dim3 grid(vec_blocks(n), L);
    if (prec == 0)
        norm2_kernel<float><<<grid, VT, 0, st>>>((const float *)x, n, scal, partial, part_stride, counter);
    else
        norm2_kernel<double><<<grid, VT, 0, st>>>((const double *)x, n, scal, partial, part_stride, counter);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_convert(int sp, const void *src, int dp, void *dst, long long n, cudaStream_t st) {
    if (n == 0) return;
    const int blocks = (int)std::min<long long>(4096, (n + 255) / 256);
    if (sp == 0 && dp == 0) convert_kernel<float, float><<<blocks, 256, 0, st>>>((const float *)src, (float *)dst, n);
    else if (sp == 0 && dp == 1) convert_kernel<float, double><<<blocks, 256, 0, st>>>((const float *)src, (double *)dst, n);
    else if (sp == 1 && dp == 0) convert_kernel<double, float><<<blocks, 256, 0, st>>>((const double *)src, (float *)dst, n);
    else convert_kernel<double, double><<<blocks, 256, 0, st>>>((const double *)src, (double *)dst, n);
    TQ_CHECK_CUDA(cudaGetLastError());
}

}  // namespace tq
