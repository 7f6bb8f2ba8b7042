// vec.cu -- see vec.cuh.
#include "vec.cuh"

namespace tq {

namespace {
constexpr int VT = 256;  // threads
constexpr int VE = 8;    // elements per thread: two 16-byte quads of every operand in flight
}

int vec_blocks(long long n) { return ceil_div(n, (long long)VT * VE); }

// Element e of thread t in block b: quads at b*VT*VE + {0, VT*4} + 4t (coalesced 16-byte
// accesses).  n % 4 != 0 (odd-size stateless calls) takes the scalar path.
template <typename F4, typename F1>
__device__ __forceinline__ void vec_loop(long long n, F4 &&body4, F1 &&body1) {
    if ((n & 3) == 0) {
#pragma unroll
        for (int h = 0; h < VE / 4; h++) {
            const long long i = (long long)blockIdx.x * VT * VE + h * VT * 4 + 4 * threadIdx.x;
            if (i < n) body4(i);
        }
    } else {
#pragma unroll
        for (int e = 0; e < VE; e++) {
            const long long i = (long long)blockIdx.x * VT * VE + e * VT + threadIdx.x;
            if (i < n) body1(i);
        }
    }
}

// x += alpha p (alpha from launch_cg_alpha).  WITH_P = true: the new direction p = r + beta p
// and each CTA's ||p||^2 into pp_out for the next step's alpha (read after this kernel: no
// last-block pass).  WITH_P = false (the last CG step of an inner solve): no new direction;
// the final ||x||^2 per node goes to scal[S_NORM] (the divergence check of tq_run).
template <typename T, bool WITH_P>
__global__ void __launch_bounds__(VT) cg_update_px(T *__restrict__ x, T *__restrict__ p, const T *__restrict__ r,
                                                   long long n, double *scal, double *partial, int part_stride,
                                                   unsigned *counter, double *pp_out, const AxUpdate au) {
    pdl_wait();
    __shared__ double red[VT / 32 + 1];
    __shared__ bool last;
    const int node = blockIdx.y;
    const long long base = (long long)node * n;
    double *sc = scal + (long long)node * S_NSLOT;
    const double alpha = sc[S_ALPHA];
    const double beta = sc[S_BETA];
    if (au.ax) {  // A x += alpha A p over the node's sinogram rows (x += alpha p below)
        const long long ne = (long long)au.nang[node] * au.n_det, r0 = au.row0[node];
        T *axp = reinterpret_cast<T *>(au.ax);
        const T *sp_ = reinterpret_cast<const T *>(au.s);
        for (long long e = (long long)blockIdx.x * VT + threadIdx.x; e < ne; e += (long long)gridDim.x * VT) {
            const long long row = r0 + e / au.n_det, j = e % au.n_det;
            const long long ia = row * au.n_det + j;
            axp[ia] = (T)((double)axp[ia] + alpha * (double)sp_[row * au.sp + 1 + j]);
        }
    }
    x += base; p += base; r += base;
    double nrm = 0.0;
    vec_loop(n,
        [&](long long i) {
            Q4<T> xv = ld4(x + i), pv = ld4(p + i);
            Q4<T> rv;
            if (WITH_P) rv = ld4(r + i);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                xv.v[u] = (T)((double)xv.v[u] + alpha * (double)pv.v[u]);
                if (WITH_P) {
                    pv.v[u] = (T)((double)rv.v[u] + beta * (double)pv.v[u]);
                    nrm += (double)pv.v[u] * (double)pv.v[u];
                } else {
                    nrm += (double)xv.v[u] * (double)xv.v[u];
                }
            }
            st4(x + i, xv);
            if (WITH_P) st4(p + i, pv);
        },
        [&](long long i) {
            const T pv = p[i];
            const T xv = (T)((double)x[i] + alpha * (double)pv);
            x[i] = xv;
            if (WITH_P) {
                const T pn = (T)((double)r[i] + beta * (double)pv);
                p[i] = pn;
                nrm += (double)pn * (double)pn;
            } else {
                nrm += (double)xv * (double)xv;
            }
        });
    const double bs = block_sum<VT>(nrm, red);
    if (WITH_P) {  // read by the next step's cg_alpha (kernel order; no last-block pass)
        if (threadIdx.x == 0) pp_out[(long long)node * part_stride + blockIdx.x] = bs;
        return;
    }
    double *part = partial + (long long)node * part_stride;
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block_of_group(counter + node, gridDim.x, &last)) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += VT) s += __ldcg(part + b);
        s = block_sum<VT>(s, red);
        if (threadIdx.x == 0) sc[S_NORM] = s;
    }
}

template <typename T>
__global__ void __launch_bounds__(VT) norm2_kernel(const T *__restrict__ x, long long n, double *scal,
                                                   double *partial, int part_stride, unsigned *counter) {
    __shared__ double red[VT / 32 + 1];
    __shared__ bool last;
    const int node = blockIdx.y;
    x += (long long)node * n;
    double dot = 0.0;
    vec_loop(n,
        [&](long long i) {
            const Q4<T> xv = ld4(x + i);
#pragma unroll
            for (int u = 0; u < 4; u++) dot += (double)xv.v[u] * (double)xv.v[u];
        },
        [&](long long i) { dot += (double)x[i] * (double)x[i]; });
    const double bs = block_sum<VT>(dot, red);
    double *part = partial + (long long)node * part_stride;
    if (threadIdx.x == 0) part[blockIdx.x] = bs;
    if (last_block_of_group(counter + node, gridDim.x, &last)) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += VT) s += __ldcg(part + b);
        s = block_sum<VT>(s, red);
        if (threadIdx.x == 0) scal[(long long)node * S_NSLOT + S_NORM] = s;
    }
}

// stop test of tq_params.stop_tol: for vector v, out[2v] = ||cur_v - prev_v||^2 and
// out[2v+1] = ||cur_v||^2 (fixed-order fp64 sums), then prev_v = cur_v
template <typename T>
__global__ void __launch_bounds__(VT) rel_change_kernel(const void *const *cur_tab, T *__restrict__ prev,
                                                        long long n, double *out, double *partial,
                                                        int part_stride, unsigned *counter) {
    __shared__ double red[VT / 32 + 1];
    __shared__ bool last;
    const int v = blockIdx.y;
    const T *__restrict__ cur = (const T *)cur_tab[v];
    T *__restrict__ pv = prev + (long long)v * n;
    double dd = 0.0, xx = 0.0;
    vec_loop(n,
        [&](long long i) {
            const Q4<T> c = ld4(cur + i), p = ld4(pv + i);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const double d = (double)c.v[u] - (double)p.v[u];
                dd += d * d;
                xx += (double)c.v[u] * (double)c.v[u];
            }
            st4(pv + i, c);
        },
        [&](long long i) {
            const double c = (double)cur[i], d = c - (double)pv[i];
            dd += d * d;
            xx += c * c;
            pv[i] = cur[i];
        });
    const double bd = block_sum<VT>(dd, red);
    const double bx = block_sum<VT>(xx, red);
    double *part = partial + (long long)v * part_stride * 2;
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = bd; part[2 * blockIdx.x + 1] = bx; }
    if (last_block_of_group(counter + v, gridDim.x, &last)) {
        double sd = 0.0, sx = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += VT) { sd += __ldcg(part + 2 * b); sx += __ldcg(part + 2 * b + 1); }
        sd = block_sum<VT>(sd, red);
        sx = block_sum<VT>(sx, red);
        if (threadIdx.x == 0) { out[2 * v] = sd; out[2 * v + 1] = sx; }
    }
}

template <typename A, typename B>
__global__ void convert_kernel(const A *src, B *dst, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = (B)src[i];
}

__global__ void __launch_bounds__(VT) cg_alpha_kernel(double *scal, const double *cgs, int nfs_pa, const int *nang,
                                                      const double *cgp, int npp, const double *cnode, int part_stride) {
    pdl_wait();
    __shared__ double red[VT / 32 + 1];
    const int node = blockIdx.x;
    const double *fs = cgs + (long long)node * part_stride, *ps = cgp + (long long)node * part_stride;
    const int nfs = nfs_pa * nang[node];
    double s1 = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < nfs; i += VT) s1 += fs[i];
    for (int i = threadIdx.x; i < npp; i += VT) s2 += ps[i];
    s1 = block_sum<VT>(s1, red);
    s2 = block_sum<VT>(s2, red);
    if (threadIdx.x == 0) {
        double *sc = scal + (long long)node * S_NSLOT;
        const double pq = s1 + cnode[node] * (npp > 0 ? s2 : sc[S_PP]);
        sc[S_PQ] = pq;
        sc[S_ALPHA] = pq > 0.0 ? sc[S_RR] / pq : 0.0;
    }
}

template <typename T>
__global__ void resid_from_ax_kernel(const T *__restrict__ d, const T *__restrict__ ax, T *__restrict__ s, int n_rows,
                                     int n_det, int sp) {
    pdl_wait();
    const long long ne = (long long)n_rows * n_det;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (long long)gridDim.x * blockDim.x) {
        const long long row = e / n_det, j = e % n_det;
        s[row * sp + 1 + j] = d[e] - ax[e];
    }
}

void launch_resid_from_ax(int prec, const void *d, const void *ax, void *s, int n_rows, int n_det, int sp,
                          cudaStream_t st) {
    const long long ne = (long long)n_rows * n_det;
    if (ne == 0) return;
    const int blocks = (int)std::min<long long>(1184, (ne + 255) / 256);
    if (prec == 0) launch_pdl(resid_from_ax_kernel<float>, blocks, 256, 0, st, (const float *)d, (const float *)ax, (float *)s, n_rows, n_det, sp);
    else launch_pdl(resid_from_ax_kernel<double>, blocks, 256, 0, st, (const double *)d, (const double *)ax, (double *)s, n_rows, n_det, sp);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_cg_alpha(int L, double *scal, const double *cgs, int nfs_pa, const int *nang, const double *cgp,
                     int npp, const double *cnode, int part_stride, cudaStream_t st) {
    if (L == 0) return;
    launch_pdl(cg_alpha_kernel, L, VT, 0, st, scal, cgs, nfs_pa, nang, cgp, npp, cnode, part_stride);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_cg_update_px(int prec, void *x, void *p, const void *r, long long n, int L, double *scal,
                         double *partial, int part_stride, unsigned *counter, bool with_p, double *pp_out,
                         const AxUpdate &au, cudaStream_t st) {
    dim3 grid(vec_blocks(n), L);
    if (prec == 0) {
        if (with_p) launch_pdl(cg_update_px<float, true>, grid, VT, 0, st, (float *)x, (float *)p, (const float *)r, n, scal, partial, part_stride, counter, pp_out, au);
        else launch_pdl(cg_update_px<float, false>, grid, VT, 0, st, (float *)x, (float *)p, (const float *)r, n, scal, partial, part_stride, counter, pp_out, au);
    } else {
        if (with_p) launch_pdl(cg_update_px<double, true>, grid, VT, 0, st, (double *)x, (double *)p, (const double *)r, n, scal, partial, part_stride, counter, pp_out, au);
        else launch_pdl(cg_update_px<double, false>, grid, VT, 0, st, (double *)x, (double *)p, (const double *)r, n, scal, partial, part_stride, counter, pp_out, au);
    }
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

void launch_rel_change(int prec, const void *const *cur_tab, void *prev, long long n, int V, double *out,
                       double *partial, int part_stride, unsigned *counter, cudaStream_t st) {
    if (V == 0) return;
    dim3 grid(vec_blocks(n), V);
    if (prec == 0)
        rel_change_kernel<float><<<grid, VT, 0, st>>>(cur_tab, (float *)prev, n, out, partial, part_stride, counter);
    else
        rel_change_kernel<double><<<grid, VT, 0, st>>>(cur_tab, (double *)prev, n, out, partial, part_stride, counter);
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
