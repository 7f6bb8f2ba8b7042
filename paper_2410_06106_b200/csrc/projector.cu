// projector.cu -- see projector.cuh.
#include "projector.cuh"

namespace tq {

namespace {

constexpr int FP_THREADS = 128;   // consecutive bins of one (node, angle)
constexpr int BP_TX = 32, BP_TY = 8, BP_PX = 2;  // tile = (32*PX) x 8 pixels
constexpr int BP_THREADS = BP_TX * BP_TY;
constexpr int BP_MAXA = 128;      // angles staged per smem chunk

template <typename T>
__device__ __forceinline__ T floor_split(T x, int &i);
template <>
__device__ __forceinline__ float floor_split<float>(float x, int &i) { return floor_pos(x, i); }
template <>
__device__ __forceinline__ double floor_split<double>(double x, int &i) {
    double f = floor(x);
    i = (int)f;
    return f;
}

// Range of lines l in [0, N) where the ray's fractional index f0 + l df lies in
// (-1, N) (outside it both taps are off the grid).  Conservative by one line.
__device__ __forceinline__ void line_range(double f0, double df, int N, int &lo, int &hi) {
    if (fabs(df) < 1e-12) {
        if (f0 > -1.0 && f0 < (double)N) { lo = 0; hi = N; } else { lo = 0; hi = 0; }
        return;
    }
    double a = (-1.0 - f0) / df, b = ((double)N - f0) / df;
    double l0 = fmin(a, b), l1 = fmax(a, b);
    lo = (int)fmax(0.0, floor(l0) - 1.0);
    hi = (int)fmin((double)N, ceil(l1) + 2.0);
    if (hi < lo) hi = lo;
}

template <typename T, bool RESID>
__global__ void __launch_bounds__(FP_THREADS) fp_kernel(const FpArgs<T> a) {
    const RayRow rr = a.rows[blockIdx.y];
    const int j = blockIdx.x * FP_THREADS + threadIdx.x;
    if (j >= a.n_det) return;
    const int N = a.N;
    const T *__restrict__ img = a.img + (long long)rr.node * a.n;
    const double2 cs_sn = a.trig[rr.angle];
    const double cs = cs_sn.x, sn = cs_sn.y;
    const bool xm = a.xmaj[rr.angle] != 0;
    const double half = 0.5 * (double)(N - 1);
    const double t = (double)j - 0.5 * (double)(a.n_det - 1);
    // fractional index of the ray on line l: y-major -> column on row l,
    // x-major -> row on column l (R-1 ray-driven form)
    double f0, df, inv_m;
    if (!xm) { f0 = (t - half * sn) / cs + half; df = sn / cs; inv_m = 1.0 / fabs(cs); }
    else     { f0 = half - (t + half * cs) / sn; df = cs / sn; inv_m = 1.0 / fabs(sn); }
    int lo, hi;
    line_range(f0, df, N, lo, hi);
    const T dfT = (T)df;
    T acc0 = 0, acc1 = 0;
    for (int L0 = lo; L0 < hi; L0 += 32) {
        const double b = f0 + (double)L0 * df;
        const int bi = (int)floor(b) - 64;
        const T bf = (T)(b - (double)bi);          // in [64, 65)
        const int cnt = min(32, hi - L0);
        if (!xm) {
            const T *rowp = img + (long long)L0 * N;
#pragma unroll 4
            for (int l = 0; l < cnt; l++, rowp += N) {
                int i0;
                const T cl = bf + (T)l * dfT;
                const T fl = floor_split<T>(cl, i0);
                i0 += bi;
                const T f = cl - fl;
                const T v0 = ((unsigned)i0 < (unsigned)N) ? __ldg(rowp + i0) : (T)0;
                const T v1 = ((unsigned)(i0 + 1) < (unsigned)N) ? __ldg(rowp + i0 + 1) : (T)0;
                if (l & 1) acc1 += v0 + f * (v1 - v0); else acc0 += v0 + f * (v1 - v0);
            }
        } else {
            const T *colp = img + L0;
#pragma unroll 4
            for (int l = 0; l < cnt; l++, colp++) {
                int i0;
                const T cl = bf + (T)l * dfT;
                const T fl = floor_split<T>(cl, i0);
                i0 += bi;
                const T f = cl - fl;
                const T v0 = ((unsigned)i0 < (unsigned)N) ? __ldg(colp + (long long)i0 * N) : (T)0;
                const T v1 = ((unsigned)(i0 + 1) < (unsigned)N) ? __ldg(colp + (long long)(i0 + 1) * N) : (T)0;
                if (l & 1) acc1 += v0 + f * (v1 - v0); else acc0 += v0 + f * (v1 - v0);
            }
        }
    }
    T v = (acc0 + acc1) * (T)inv_m;
    const long long o = (long long)blockIdx.y * a.out_stride + a.out_off + j;
    if (RESID) v = a.d[(long long)blockIdx.y * a.n_det + j] - v;
    a.out[o] = v;
}

template <typename T>
struct AngleRec {
    T base_f, cs, sn, inv_m, inv_m2, w1c;  // w1c = inv_m - inv_m2
    int base_i, row;
};

template <typename T, int EPI>
__global__ void __launch_bounds__(BP_THREADS) bp_kernel(const BpArgs<T> a) {
    __shared__ AngleRec<T> tab[BP_MAXA];
    __shared__ double red[BP_THREADS / 32 + 1];
    __shared__ bool last_flag;
    const int node = blockIdx.y;
    const int N = a.N;
    const int tiles_x = (N + BP_TX * BP_PX - 1) / (BP_TX * BP_PX);
    const int tile_r = blockIdx.x / tiles_x, tile_c = blockIdx.x % tiles_x;
    const int r0 = tile_r * BP_TY, c0 = tile_c * BP_TX * BP_PX;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int r = r0 + ty;
    const double half = 0.5 * (double)(N - 1);
    // tile reference point (centre of the tile) for the tile-relative t (precision)
    const double cref = (double)c0 + 0.5 * (BP_TX * BP_PX) , rref = (double)r0;
    const int nang = a.node_nang[node], row0 = a.node_row0[node];
    T acc[BP_PX];
#pragma unroll
    for (int i = 0; i < BP_PX; i++) acc[i] = 0;
    const T dr = (T)(r - r0);
    for (int k0 = 0; k0 < nang; k0 += BP_MAXA) {
        const int kc = min(BP_MAXA, nang - k0);
        __syncthreads();
        for (int k = threadIdx.x; k < kc; k += BP_THREADS) {
            const int row = row0 + k0 + k;
            const int ang = a.rows[row].angle;
            const double2 t2 = a.trig[ang];
            const double m = a.xmaj[ang] ? fabs(t2.y) : fabs(t2.x);
            const double base = (cref - half) * t2.x + (half - rref) * t2.y + 0.5 * (double)(a.n_det - 1);
            const int bi = (int)floor(base) - 48;
            AngleRec<T> rec;
            rec.base_f = (T)(base - (double)bi);
            rec.cs = (T)t2.x;
            rec.sn = (T)t2.y;
            rec.inv_m = (T)(1.0 / m);
            rec.inv_m2 = (T)(1.0 / (m * m));
            rec.w1c = (T)(1.0 / m - 1.0 / (m * m));
            rec.base_i = bi;
            rec.row = row;
            tab[k] = rec;
        }
        __syncthreads();
        for (int k = 0; k < kc; k++) {
            const AngleRec<T> rec = tab[k];
            const T *__restrict__ srow = a.s + (long long)rec.row * a.s_stride + a.s_off;
            // t of this thread's first pixel relative to the tile reference
            const T tl0 = rec.base_f + ((T)tx - (T)(0.5 * (BP_TX * BP_PX))) * rec.cs - dr * rec.sn;
#pragma unroll
            for (int i = 0; i < BP_PX; i++) {
                const T tl = tl0 + (T)(BP_TX * i) * rec.cs;
                int ji;
                const T fl = floor_split<T>(tl, ji);
                const T u = tl - fl;
                const int j = rec.base_i + ji;
                const T w0 = max((T)0, rec.inv_m - u * rec.inv_m2);
                const T w1 = max((T)0, rec.w1c + u * rec.inv_m2);
                acc[i] += w0 * __ldg(srow + j) + w1 * __ldg(srow + j + 1);
            }
        }
    }
    // ---------------- epilogue
    const double c = (EPI == EPI_CGQ || EPI == EPI_RESID || EPI == EPI_GD) ? a.cnode[node] : 0.0;
    double dot = 0.0;
    const long long nb = (long long)node * a.n;
#pragma unroll
    for (int i = 0; i < BP_PX; i++) {
        const int col = c0 + tx + BP_TX * i;
        if (r >= N || col >= N) continue;
        const long long p = nb + (long long)r * N + col;
        const double g = (double)acc[i];
        if (EPI == EPI_PLAIN) {
            a.out[p] = acc[i];
        } else if (EPI == EPI_CGQ) {
            const double pv = (double)a.vin[p];
            const T q = (T)(g + c * pv);
            a.out[p] = q;
            dot += pv * (double)q;
        } else if (EPI == EPI_RESID) {
            const T rv = (T)(g + (double)a.bprime[p] - c * (double)a.vin[p]);
            a.out[p] = rv;
            a.out2[p] = rv;
            dot += (double)rv * (double)rv;
        } else {  // EPI_GD: x <- x - eta (c x - b' - A^T(d - A x))
            const double xv = (double)a.vin[p];
            a.out[p] = (T)(xv - a.eta[node] * (c * xv - (double)a.bprime[p] - g));
        }
    }
    if (EPI == EPI_CGQ || EPI == EPI_RESID) {
        const double bs = block_sum<BP_THREADS>(dot, red);
        double *part = a.partial + (long long)node * a.part_stride;
        if (threadIdx.x == 0) part[blockIdx.x] = bs;
        if (last_block_of_group(a.counter + node, gridDim.x, &last_flag)) {
            double s = 0.0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += BP_THREADS) s += part[b];
            s = block_sum<BP_THREADS>(s, red);
            if (threadIdx.x == 0) {
                double *sc = a.scal + (long long)node * S_NSLOT;
                if (EPI == EPI_CGQ) {
                    sc[S_PQ] = s;
                    sc[S_ALPHA] = s > 0.0 ? sc[S_RR] / s : 0.0;
                } else {
                    sc[S_RR] = s;
                }
            }
        }
    }
}

}  // namespace

int bp_tiles(int N) {
    const int tx = (N + BP_TX * BP_PX - 1) / (BP_TX * BP_PX);
    const int ty = (N + BP_TY - 1) / BP_TY;
    return tx * ty;
}

void launch_fp(int prec, bool resid, const void *args, int n_rows, int n_det, cudaStream_t st) {
    dim3 grid(ceil_div(n_det, FP_THREADS), n_rows);
    if (n_rows == 0) return;
    if (prec == 0) {
        const auto &A = *static_cast<const FpArgs<float> *>(args);
        if (resid) fp_kernel<float, true><<<grid, FP_THREADS, 0, st>>>(A);
        else fp_kernel<float, false><<<grid, FP_THREADS, 0, st>>>(A);
    } else {
        const auto &A = *static_cast<const FpArgs<double> *>(args);
        if (resid) fp_kernel<double, true><<<grid, FP_THREADS, 0, st>>>(A);
        else fp_kernel<double, false><<<grid, FP_THREADS, 0, st>>>(A);
    }
    TQ_CHECK_CUDA(cudaGetLastError());
}

template <typename T>
static void bp_dispatch(int epi, const BpArgs<T> &A, dim3 grid, cudaStream_t st) {
    switch (epi) {
        case EPI_PLAIN: bp_kernel<T, EPI_PLAIN><<<grid, BP_THREADS, 0, st>>>(A); break;
        case EPI_CGQ: bp_kernel<T, EPI_CGQ><<<grid, BP_THREADS, 0, st>>>(A); break;
        case EPI_RESID: bp_kernel<T, EPI_RESID><<<grid, BP_THREADS, 0, st>>>(A); break;
        default: bp_kernel<T, EPI_GD><<<grid, BP_THREADS, 0, st>>>(A); break;
    }
}

void launch_bp(int prec, int epi, const void *args, int L, int N, cudaStream_t st) {
    if (L == 0) return;
    dim3 grid(bp_tiles(N), L);
    if (prec == 0) bp_dispatch<float>(epi, *static_cast<const BpArgs<float> *>(args), grid, st);
    else bp_dispatch<double>(epi, *static_cast<const BpArgs<double> *>(args), grid, st);
    TQ_CHECK_CUDA(cudaGetLastError());
}

}  // namespace tq
