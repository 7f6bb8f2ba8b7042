// dct.cu -- JPEG-style DCT quantizer ("dADMM-J"), exact integer pipeline
// of DESIGN.md R-18.  One 8x8 block per 8-lane group; 32 blocks per 256-thread CTA.
#include <math.h>

#include "codecs.cuh"

namespace tq {

namespace {

constexpr int DT = 256;              // threads per CTA
constexpr int BLK_PER_CTA = DT / 8;  // 8x8 blocks per CTA

struct DctTables {
    int C[64];  // C[u*8+x] = round(2^14 alpha(u) cos((2x+1) u pi / 16))
    int Q[64];  // quality-scaled luminance table, natural order
};

// JPEG luminance quantisation table (ITU-T T.81 Annex K, Table K.1), natural order.
const int kLuma[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                       14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                       18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                       49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};

DctTables make_tables(int quality) {
    DctTables t;
    dct_host_tables(quality, t.C, t.Q);
    return t;
}

__device__ __forceinline__ int rs10(int v) { return (v + 512) >> 10; }
__device__ __forceinline__ long long rs(long long v, int k) { return (v + (1LL << (k - 1))) >> k; }

// per-payload min / max (exact in any order); written to the payload header.  A few
// CTAs per payload stream it with 16-byte loads (warp-shuffle block reduction); the last
// CTA of a payload combines the per-CTA partials with one warp.
__device__ __forceinline__ void warp_minmax(float &mn, float &mx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
}
__global__ void __launch_bounds__(DT) dct_minmax(const float *const *vin, long long nv, float *partial,
                                                 int part_stride, unsigned *counter,
                                                 uint8_t *const *pay, float *mm_work) {
    __shared__ float smn[DT / 32], smx[DT / 32];
    __shared__ bool last;
    const int b = blockIdx.y;
    const float *vb = vin[b];
    float mn = INFINITY, mx = -INFINITY;
    const long long stride = (long long)gridDim.x * DT;
    if ((nv & 3) == 0 && ((uintptr_t)vb & 15) == 0) {
        const float4 *v4 = reinterpret_cast<const float4 *>(vb);
        for (long long i = (long long)blockIdx.x * DT + threadIdx.x; i < nv / 4; i += stride) {
            const float4 x = __ldg(v4 + i);
            mn = fminf(fminf(mn, x.x), fminf(x.y, fminf(x.z, x.w)));
            mx = fmaxf(fmaxf(mx, x.x), fmaxf(x.y, fmaxf(x.z, x.w)));
        }
    } else {
        for (long long i = (long long)blockIdx.x * DT + threadIdx.x; i < nv; i += stride) {
            const float x = vb[i];
            mn = fminf(mn, x);
            mx = fmaxf(mx, x);
        }
    }
    warp_minmax(mn, mx);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { smn[warp] = mn; smx[warp] = mx; }
    __syncthreads();
    if (warp == 0) {
        mn = lane < DT / 32 ? smn[lane] : INFINITY;
        mx = lane < DT / 32 ? smx[lane] : -INFINITY;
        warp_minmax(mn, mx);
    }
    float *part = partial + (long long)b * part_stride;
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = mn; part[2 * blockIdx.x + 1] = mx; }
    if (last_block_of_group(counter + b, gridDim.x, &last) && warp == 0) {
        float a = INFINITY, c = -INFINITY;
        for (unsigned k = lane; k < gridDim.x; k += 32) { a = fminf(a, __ldcg(part + 2 * k)); c = fmaxf(c, __ldcg(part + 2 * k + 1)); }
        warp_minmax(a, c);
        if (lane == 0) {
            mm_work[2 * b] = a;
            mm_work[2 * b + 1] = c;
            float *hdr = reinterpret_cast<float *>(pay[b]);
            hdr[0] = a;
            hdr[1] = c;
        }
    }
}

__global__ void __launch_bounds__(DT) dct_enc(const float *const *vin, int rows, int cols,
                                              const float *mm, DctTables tab, uint8_t *const *pay,
                                              int16_t *coef_base) {
    __shared__ int Ts[BLK_PER_CTA][8][9];
    __shared__ int Cs[64], Qs[64];
    if (threadIdx.x < 64) { Cs[threadIdx.x] = tab.C[threadIdx.x]; Qs[threadIdx.x] = tab.Q[threadIdx.x]; }
    __syncthreads();
    const int b = blockIdx.y;
    const int g = threadIdx.x >> 3, lane8 = threadIdx.x & 7;
    const int nbc = cols / 8;
    const long long nblk = (long long)(rows / 8) * nbc;
    const long long blk = (long long)blockIdx.x * BLK_PER_CTA + g;
    const bool active = blk < nblk;
    const float mn = mm[2 * b], mx = mm[2 * b + 1];
    const int br = active ? (int)(blk / nbc) : 0, bc = active ? (int)(blk % nbc) : 0;
    if (active) {
        int B[8];
        const float *src = vin[b] + (long long)(8 * br + lane8) * cols + 8 * bc;
        const double den = (double)mx - (double)mn;
#pragma unroll
        for (int y = 0; y < 8; y++) {
            const double num = __dsub_rn((double)src[y], (double)mn);
            double p = rint(__ddiv_rn(__dmul_rn(num, 255.0), den));
            p = fmin(255.0, fmax(0.0, p));
            B[y] = (int)p - 128;
        }
        // row pass (lane8 = row x): T[x][w] = rs(sum_y B[x][y] C[w][y], 10)
#pragma unroll
        for (int w = 0; w < 8; w++) {
            int s = 0;
#pragma unroll
            for (int y = 0; y < 8; y++) s += B[y] * Cs[w * 8 + y];
            Ts[g][lane8][w] = rs10(s);
        }
    }
    __syncwarp();
    if (!active) return;
    int16_t *out = (coef_base ? coef_base + (long long)b * rows * cols : reinterpret_cast<int16_t *>(pay[b] + 8)) +
                   blk * 64;
    const int w = lane8;  // column pass: lane = column w
#pragma unroll
    for (int u = 0; u < 8; u++) {
        int Y = 0;
#pragma unroll
        for (int x = 0; x < 8; x++) Y += Cs[u * 8 + x] * Ts[g][x][w];
        int q = 0;
        if (mn != mx) {
            const int D = Qs[u * 8 + w] << 18;
            const int a = Y < 0 ? -Y : Y;
            q = (a + D / 2) / D;
            if (Y < 0) q = -q;
        }
        out[u * 8 + w] = (int16_t)q;
    }
}

template <typename T>
__global__ void __launch_bounds__(DT) dct_dec(const uint8_t *const *pay, int rows, int cols,
                                              DctTables tab, T *const *outp, const int16_t *coef_base) {
    __shared__ long long Ts[BLK_PER_CTA][8][9];
    __shared__ int Cs[64], Qs[64];
    if (threadIdx.x < 64) { Cs[threadIdx.x] = tab.C[threadIdx.x]; Qs[threadIdx.x] = tab.Q[threadIdx.x]; }
    __syncthreads();
    const int b = blockIdx.y;
    const int g = threadIdx.x >> 3, lane8 = threadIdx.x & 7;
    const int nbc = cols / 8;
    const long long nblk = (long long)(rows / 8) * nbc;
    const long long blk = (long long)blockIdx.x * BLK_PER_CTA + g;
    const bool active = blk < nblk;
    const float *hdr = reinterpret_cast<const float *>(pay[b]);
    const float mn = hdr[0], mx = hdr[1];
    if (active) {
        const int16_t *in = (coef_base ? coef_base + (long long)b * rows * cols
                                       : reinterpret_cast<const int16_t *>(pay[b] + 8)) +
                            blk * 64;
        const int w = lane8;  // pass 1, lane = column w: T'[x][w] = rs(sum_u C[u][x] G[u][w], 10)
        long long G[8];
#pragma unroll
        for (int u = 0; u < 8; u++) G[u] = (long long)in[u * 8 + w] * Qs[u * 8 + w];
#pragma unroll
        for (int x = 0; x < 8; x++) {
            long long s = 0;
#pragma unroll
            for (int u = 0; u < 8; u++) s += (long long)Cs[u * 8 + x] * G[u];
            Ts[g][x][w] = rs(s, 10);
        }
    }
    __syncwarp();
    if (!active) return;
    const int br = (int)(blk / nbc), bc = (int)(blk % nbc);
    const int x = lane8;  // pass 2, lane = row x: R[x][y] = sum_w T'[x][w] C[w][y]
    const float step = (float)(((double)mx - (double)mn) / 255.0);
    T *dst = outp[b] + (long long)(8 * br + x) * cols + 8 * bc;
#pragma unroll
    for (int y = 0; y < 8; y++) {
        long long R = 0;
#pragma unroll
        for (int w = 0; w < 8; w++) R += Ts[g][x][w] * (long long)Cs[w * 8 + y];
        long long smp = rs(R, 18) + 128;
        smp = smp < 0 ? 0 : (smp > 255 ? 255 : smp);
        const float val = (mn == mx) ? mn : __fadd_rn(mn, __fmul_rn((float)smp, step));
        dst[y] = (T)val;
    }
}

}  // namespace

void dct_host_tables(int quality, int *C, int *Q) {
    const int q = std::min(100, std::max(1, quality));
    const int s = q < 50 ? 5000 / q : 200 - 2 * q;  // IJG scaling
    for (int i = 0; i < 64; i++) Q[i] = std::min(255, std::max(1, (kLuma[i] * s + 50) / 100));
    for (int u = 0; u < 8; u++)
        for (int x = 0; x < 8; x++) {
            const double al = u == 0 ? sqrt(0.125) : 0.5;
            C[u * 8 + x] = (int)lround(16384.0 * al * cos((2 * x + 1) * u * M_PI / 16.0));
        }
}

long long dct_payload_bytes(long long nv) { return 8 + 2 * nv; }

void DctWork::alloc(int P_, long long nv) {
    P = P_;
    // CTAs per payload for the min / max pass: ~16 K elements each, at most 128
    part_stride = 2 * (int)std::max(1LL, std::min(128LL, (nv + 16383) / 16384));
    TQ_CHECK_CUDA(cudaMalloc(&minmax, sizeof(float) * 2 * std::max(1, P)));
    TQ_CHECK_CUDA(cudaMalloc(&partial, sizeof(float) * part_stride * std::max(1, P)));
    TQ_CHECK_CUDA(cudaMalloc(&counter, sizeof(unsigned) * std::max(1, P)));
    TQ_CHECK_CUDA(cudaMemset(counter, 0, sizeof(unsigned) * std::max(1, P)));
}

void DctWork::release() {
    if (minmax) cudaFree(minmax);
    if (partial) cudaFree(partial);
    if (counter) cudaFree(counter);
    *this = DctWork();
}

int dct_encode(const float *const *vin, int P, int rows, int cols, int quality, DctWork &ws,
               uint8_t *const *pay, cudaStream_t st, JpegWork *jw) {
    if (P == 0) return 0;
    TQ_REQUIRE(rows % 8 == 0 && cols % 8 == 0 && rows > 0, "dct: rows and cols must be multiples of 8");
    const long long nv = (long long)rows * cols;
    const int mblocks = ws.part_stride / 2;
    dct_minmax<<<dim3(mblocks, P), DT, 0, st>>>(vin, nv, ws.partial, ws.part_stride, ws.counter, pay,
                                                 ws.minmax);
    const DctTables tab = make_tables(quality);
    const long long nblk = nv / 64;
    dct_enc<<<dim3(ceil_div(nblk, BLK_PER_CTA), P), DT, 0, st>>>(vin, rows, cols, ws.minmax, tab, pay,
                                                                  jw ? jw->coef : nullptr);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 2 + (jw ? jpeg_encode(pay, *jw, st) : 0);
}

int dct_decode(const uint8_t *const *pay, int P, int rows, int cols, int quality, int prec,
               void *const *out, cudaStream_t st, JpegWork *jw) {
    if (P == 0) return 0;
    const int kj = jw ? jpeg_decode(const_cast<uint8_t *const *>(pay), *jw, st) : 0;
    TQ_REQUIRE(rows % 8 == 0 && cols % 8 == 0 && rows > 0, "dct: rows and cols must be multiples of 8");
    const DctTables tab = make_tables(quality);
    const long long nblk = (long long)rows * cols / 64;
    const dim3 grid(ceil_div(nblk, BLK_PER_CTA), P);
    const int16_t *cb = jw ? jw->coef : nullptr;
    if (prec == 0)
        dct_dec<float><<<grid, DT, 0, st>>>(pay, rows, cols, tab, (float *const *)out, cb);
    else
        dct_dec<double><<<grid, DT, 0, st>>>(pay, rows, cols, tab, (double *const *)out, cb);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1 + kj;
}

}  // namespace tq
