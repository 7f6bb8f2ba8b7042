// consensus.cu -- see consensus.cuh.
#include "consensus.cuh"

namespace tq {

namespace {
constexpr int CT = 256;

inline dim3 grid_of(long long n, int L) {
    return dim3((unsigned)std::max(1LL, std::min<long long>((n + CT * 4 - 1) / (CT * 4), 65535)), L);
}
// the graph-rule kernel covers 8 elements per thread (2 quads)
inline dim3 grid_dual(long long n, int L) {
    return dim3((unsigned)std::max(1LL, std::min<long long>((n + CT * 8 - 1) / (CT * 8), 65535)), L);
}

constexpr int MAXNB = TQ_MAX_DEGREE;  // neighbour pointers cached in shared memory (host-validated)

template <typename T>
__device__ __forceinline__ void graph_dual_elem(const T *const *nb, int deg, const T *own, T *al, T *bp,
                                                long long p, double rho, int update) {
    const double x = (double)own[p];
    double s = 0.0;
    for (int k = 0; k < deg; k++) s += (double)nb[k][p];
    T a = al[p];
    if (update) {
        a = (T)((double)a + rho * ((double)deg * x - s));
        al[p] = a;
    }
    bp[p] = (T)(-(double)a + rho * ((double)deg * x + s));
}

// one node per blockIdx.y; 4 elements per thread per step through 16-byte accesses
template <typename T>
__global__ void __launch_bounds__(CT) graph_dual(const T *const *own_ptr, const T *const *nbr_ptr,
                                                 const int *nbr_off, T *alpha,
                                                 T *bprime, long long n, double rho, int update) {
    pdl_wait();
    __shared__ const T *nb[MAXNB];
    const int i = blockIdx.y;
    const T *own = own_ptr[i];
    const int k0 = nbr_off[i], deg = nbr_off[i + 1] - k0;
    for (int k = threadIdx.x; k < deg; k += CT) nb[k] = nbr_ptr[k0 + k];
    __syncthreads();
    T *al = alpha + (long long)i * n;
    T *bp = bprime + (long long)i * n;
    if ((n & 3) == 0) {
        for (long long p = 4 * ((long long)blockIdx.x * CT + threadIdx.x); p < n; p += 4LL * gridDim.x * CT) {
            const Q4<T> xv = ld4(own + p);
            Q4<T> av = ld4(al + p), bv;
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            int k = 0;
            for (; k + 4 <= deg; k += 4) {  // four neighbour quads in flight (fixed summation order)
                Q4<T> y[4];
#pragma unroll
                for (int j = 0; j < 4; j++) y[j] = ld4(nb[k + j] + p);
#pragma unroll
                for (int j = 0; j < 4; j++)
#pragma unroll
                    for (int u = 0; u < 4; u++) s[u] += (double)y[j].v[u];
            }
            for (; k < deg; k++) {
                const Q4<T> y = ld4(nb[k] + p);
#pragma unroll
                for (int u = 0; u < 4; u++) s[u] += (double)y.v[u];
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const double x = (double)xv.v[u];
                if (update) av.v[u] = (T)((double)av.v[u] + rho * ((double)deg * x - s[u]));
                bv.v[u] = (T)(-(double)av.v[u] + rho * ((double)deg * x + s[u]));
            }
            if (update) st4(al + p, av);
            st4(bp + p, bv);
        }
    } else {
        for (long long p = (long long)blockIdx.x * CT + threadIdx.x; p < n; p += (long long)gridDim.x * CT)
            graph_dual_elem(nb, deg, own, al, bp, p, rho, update);
    }
}

template <typename T>
__global__ void __launch_bounds__(CT) paper_alg3(const T *u, const T *lam, T *const *xg,
                                                 const long long *lo, const long long *lens,
                                                 float *const *seg, long long n, double rho,
                                                 double eta2, int e2) {
    const int i = blockIdx.y;
    const long long base = lo[i], len = lens[i];
    T *x = xg[i];
    float *out = seg ? seg[i] : nullptr;
    for (long long q = (long long)blockIdx.x * CT + threadIdx.x; q < len; q += (long long)gridDim.x * CT) {
        const long long p = base + q;
        double xs = (double)x[p];
        const double uv = (double)u[(long long)i * n + p], lv = (double)lam[(long long)i * n + p];
        for (int it = 0; it < e2; it++) {
            const double delta = rho * (xs - uv - lv / rho);
            xs = xs - eta2 * delta;
        }
        if (out) out[q] = (float)xs;
        else x[p] = (T)xs;
    }
}

template <typename T>
__global__ void __launch_bounds__(CT) paper_dual(const T *u, T *lam, T *bprime, const T *const *xg,
                                                 long long n, double rho, int update) {
    const int i = blockIdx.y;
    const T *x = xg[i];
    for (long long p = (long long)blockIdx.x * CT + threadIdx.x; p < n; p += (long long)gridDim.x * CT) {
        const long long g = (long long)i * n + p;
        const double xv = (double)x[p];
        T l = lam[g];
        if (update) {
            l = (T)((double)l + rho * ((double)u[g] - xv));
            lam[g] = l;
        }
        bprime[g] = (T)(rho * xv - (double)l);
    }
}

template <typename T>
__global__ void __launch_bounds__(CT) consensus_partial(const T *u, const T *lam, double *csum, const int *slice_of,
                                                        const int *first, const int *cnt, long long n, double rho) {
    const int js = blockIdx.y;
    const int i0 = first[js], c = cnt[js];
    double *out = csum + (long long)slice_of[js] * n;
    for (long long p = (long long)blockIdx.x * CT + threadIdx.x; p < n; p += (long long)gridDim.x * CT) {
        double acc = 0.0;
        for (int q = 0; q < c; q++) {
            const long long g = (long long)(i0 + q) * n + p;
            acc += (double)u[g] + (double)lam[g] / rho;
        }
        out[p] = acc;
    }
}

template <typename T>
__global__ void __launch_bounds__(CT) consensus_segment(const double *csum, const int *node_slice, T *const *xg,
                                                        const long long *lo, const long long *lens,
                                                        float *const *seg, long long n, int M) {
    const int i = blockIdx.y;
    const long long base = lo[i], len = lens[i];
    const double *cs = csum + (long long)node_slice[i] * n;
    T *x = xg[i];
    float *out = seg ? seg[i] : nullptr;
    for (long long q = (long long)blockIdx.x * CT + threadIdx.x; q < len; q += (long long)gridDim.x * CT) {
        const double v = cs[base + q] / (double)M;
        if (out) out[q] = (float)v;
        else x[base + q] = (T)v;
    }
}

template <typename T>
__global__ void __launch_bounds__(CT) to_float(const T *const *src, float *const *dst, long long n) {
    const int i = blockIdx.y;
    const T *s = src[i];
    float *d = dst[i];
    for (long long p = (long long)blockIdx.x * CT + threadIdx.x; p < n; p += (long long)gridDim.x * CT)
        d[p] = (float)s[p];
}

}  // namespace

int launch_graph_dual(int prec, const void *const *own_ptr, const void *const *nbr_ptr, const int *nbr_off,
                      void *alpha, void *bprime, long long n, int L, double rho,
                      int update_alpha, cudaStream_t st) {
    if (L == 0) return 0;
    if (prec == 0)
        launch_pdl(graph_dual<float>, grid_dual(n, L), CT, 0, st, (const float *const *)own_ptr,
                   (const float *const *)nbr_ptr, nbr_off, (float *)alpha, (float *)bprime, n, rho, update_alpha);
    else
        graph_dual<double><<<grid_dual(n, L), CT, 0, st>>>((const double *const *)own_ptr, (const double *const *)nbr_ptr,
                                                         nbr_off, (double *)alpha, (double *)bprime, n,
                                                         rho, update_alpha);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

int launch_paper_alg3(int prec, const void *u, const void *lam, void *const *xg_tab,
                      const long long *lo, const long long *len, long long max_len,
                      float *const *seg_tab, long long n, int L, double rho, double eta2, int e2,
                      cudaStream_t st) {
    if (L == 0) return 0;
    if (prec == 0)
        paper_alg3<float><<<grid_of(max_len, L), CT, 0, st>>>((const float *)u, (const float *)lam,
                                                              (float *const *)xg_tab, lo, len, seg_tab,
                                                              n, rho, eta2, e2);
    else
        paper_alg3<double><<<grid_of(max_len, L), CT, 0, st>>>((const double *)u, (const double *)lam,
                                                               (double *const *)xg_tab, lo, len,
                                                               seg_tab, n, rho, eta2, e2);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

int launch_paper_dual(int prec, const void *u, void *lam, void *bprime, const void *const *xg_tab,
                      long long n, int L, double rho, int update_lam, cudaStream_t st) {
    if (L == 0) return 0;
    if (prec == 0)
        paper_dual<float><<<grid_of(n, L), CT, 0, st>>>((const float *)u, (float *)lam, (float *)bprime,
                                                        (const float *const *)xg_tab, n, rho, update_lam);
    else
        paper_dual<double><<<grid_of(n, L), CT, 0, st>>>((const double *)u, (double *)lam,
                                                         (double *)bprime, (const double *const *)xg_tab,
                                                         n, rho, update_lam);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

int launch_consensus_partial(int prec, const void *u, const void *lam, double *csum, const int *slice_of,
                             const int *first, const int *cnt, int n_local_slices, long long n, double rho,
                             cudaStream_t st) {
    if (n_local_slices == 0) return 0;
    if (prec == 0)
        consensus_partial<float><<<grid_of(n, n_local_slices), CT, 0, st>>>((const float *)u, (const float *)lam, csum,
                                                                            slice_of, first, cnt, n, rho);
    else
        consensus_partial<double><<<grid_of(n, n_local_slices), CT, 0, st>>>((const double *)u, (const double *)lam,
                                                                             csum, slice_of, first, cnt, n, rho);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

int launch_consensus_segment(int prec, const double *csum, const int *node_slice, void *const *xg_tab,
                             const long long *lo, const long long *len, long long max_len, float *const *seg_tab,
                             long long n, int L, int M, cudaStream_t st) {
    if (L == 0) return 0;
    if (prec == 0)
        consensus_segment<float><<<grid_of(max_len, L), CT, 0, st>>>(csum, node_slice, (float *const *)xg_tab, lo,
                                                                     len, seg_tab, n, M);
    else
        consensus_segment<double><<<grid_of(max_len, L), CT, 0, st>>>(csum, node_slice, (double *const *)xg_tab, lo,
                                                                      len, seg_tab, n, M);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

int launch_to_float(int prec, const void *const *src_tab, float *const *dst_tab, long long n, int L,
                    cudaStream_t st) {
    if (L == 0) return 0;
    if (prec == 0)
        to_float<float><<<grid_of(n, L), CT, 0, st>>>((const float *const *)src_tab, dst_tab, n);
    else
        to_float<double><<<grid_of(n, L), CT, 0, st>>>((const double *const *)src_tab, dst_tab, n);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace tq
