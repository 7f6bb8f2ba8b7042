// projector.cu -- see projector.cuh.
#include <cuda.h>

#include <cstdlib>

#include "projector.cuh"

namespace tq {

namespace {

// ------------------------------------------------------------------ shared helpers
constexpr int FP_HALO_A = (FP_HALO + 3) / 4 * 4;          // 16-byte aligned halo (40)
constexpr int FP_PITCH_Y = FP_TW + 2 * FP_HALO_A;        // 208: rows of the wide tile, float4 stores
constexpr int FP_PITCH_X = FP_TW + 2 * FP_HALO_A + 1;    // 209: odd, conflict-free transposed stores
static_assert(FP_PITCH_Y % 4 == 0, "row pitch must keep 16-byte alignment");

constexpr int BP_TS = 64;       // backprojector pixel tile side
constexpr int BP_THREADS = 256;
constexpr int BP_WB = 96;       // staged bins per angle: >= 63(|cos|+|sin|) + 4
constexpr int BP_MAXA = 32;     // angles per staged batch
// fp32 epilogues with two prefetched operands (x and b') stage 16 angles per batch, so the
// CTA stays within a quarter of the SM's shared memory (4 CTAs/SM, as the CG variant)
template <typename T, int EPI>
constexpr int bp_maxa() { return (sizeof(T) == 4 && (EPI == 2 || EPI == 3 || EPI == 4)) ? 16 : BP_MAXA; }

template <typename T>
__device__ __forceinline__ T floor_split(T x, int &i);
template <>
__device__ __forceinline__ double floor_split<double>(double x, int &i) {
    const double f = floor(x);
    i = (int)f;
    return f;
}

template <typename T>
__device__ __forceinline__ T sat(T x);
template <>
__device__ __forceinline__ double sat<double>(double x) { return fmin(fmax(x, 0.0), 1.0); }

// Ray geometry along the major axis (R-1/R-2, the ray-driven form of the
// oracle's or_project): on major-axis line l (row for y-major, column for x-major)
// the ray (theta, t) sits at fractional cross index  a0 + t*at + l*B.
struct LineGeo {
    double a0, at, B, inv_m;
};
__device__ __forceinline__ LineGeo line_geo(double cs, double sn, int xmajor, int N) {
    const double h = 0.5 * (double)(N - 1);
    LineGeo g;
    if (!xmajor) {  // column on row r: (t - y_r sin)/cos + h, y_r = h - r
        g.at = 1.0 / cs; g.a0 = h - h * sn / cs; g.B = sn / cs; g.inv_m = 1.0 / fabs(cs);
    } else {        // row on column c: h - (t - x_c cos)/sin, x_c = c - h
        g.at = -1.0 / sn; g.a0 = h - h * cs / sn; g.B = cs / sn; g.inv_m = 1.0 / fabs(sn);
    }
    return g;
}

// Shared-memory load at a 32-bit shared address + immediate byte offset.  The
// fp32 fast paths below index with the float bits of (x + 2^23) directly:
// addr = (bits << 2) + base - (0x4B000000 << 2), so one LEA forms the address of
// floor(x) and both taps use immediate offsets.
template <int OFF>
__device__ __forceinline__ float lds(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
    return v;
}
// shared base minus the magic bits (0x4B000000 << log2(entry bytes), mod 2^32), passed as a kernel argument,
// so ptxas cannot split the constant back out of the base register and re-add it
// before every load (it does that when it can see the constant).
__device__ __forceinline__ uint32_t magic_base(const void *smem_ptr, uint32_t magic) {
    return (uint32_t)__cvta_generic_to_shared(smem_ptr) - magic;
}

template <typename T>
struct V16;  // 16-byte vector of T
template <>
struct V16<float> {
    using type = float4;
    static constexpr int n = 4;
};
template <>
struct V16<double> {
    using type = double2;
    static constexpr int n = 2;
};

// ------------------------------------------------------------------ forward: tile pass
// slope 1/w of the Siddon band fraction (w = |cross drift per line|); 2^22 for axis rays
template <typename T>
__device__ __forceinline__ T siddon_iw(T B) {
    const T w = B < (T)0 ? -B : B;
    return w > (T)1e-9 ? (T)1 / w : (T)4194304;
}

template <typename T, int O, bool SID = false>  // O = 0: y-major angles (lines = rows), 1: x-major (lines = columns)
__global__ void __launch_bounds__(FP_THREADS) fp_tile_kernel(const FpArgs<T> a) {
    constexpr int PITCH = O == 0 ? FP_PITCH_Y : FP_PITCH_X;
    constexpr int H = FP_HALO_A;
    extern __shared__ __align__(16) unsigned char fp_smem[];
    T *tile = reinterpret_cast<T *>(fp_smem);  // [FP_TH][PITCH]
    __shared__ double s_kap[FP_MAXA], s_at[FP_MAXA];
    __shared__ T s_B[FP_MAXA];
    __shared__ int s_row[FP_MAXA], s_W[FP_MAXA], s_jlo[FP_MAXA], s_cofs[FP_MAXA + 1], s_wsum[2];
    static_assert(FP_MAXA == 64, "the chunk prefix below uses two warps");

    const int node = blockIdx.y;
    const int grp = 2 * node + O;
    const int a_begin = a.oofs[grp], a_end = a.oofs[grp + 1];
    if (a_begin == a_end) return;  // uniform over the block
    const int N = a.N;
    const int tile_id = blockIdx.x;
    const int ntiles = a.nt_line * a.nt_cross;
    const int lt = tile_id / a.nt_cross, ct = tile_id % a.nt_cross;
    const int L0 = lt * FP_TH, X0 = ct * FP_TW;
    const T *img = a.img + (long long)node * a.n;

    // ---- stage the tile: tile[l][k] = image at (line L0+l, cross X0-H+k); zero outside
    for (int i = threadIdx.x; i < FP_TH * (PITCH - FP_TW); i += FP_THREADS) {
        const int l = i / (PITCH - FP_TW), k = i % (PITCH - FP_TW);
        tile[l * PITCH + (k < H ? k : k + FP_TW)] = (T)0;
    }
    using VT = typename V16<T>::type;
    constexpr int VN = V16<T>::n;
    if (N % VN != 0 || ((uintptr_t)img & 15) != 0) {  // rows not 16-byte aligned (stateless calls only): scalar staging
        for (int i = threadIdx.x; i < FP_TH * FP_TW; i += FP_THREADS) {
            const int l = i / FP_TW, x = i % FP_TW;
            const int r = O == 0 ? L0 + l : X0 + x, c = O == 0 ? X0 + x : L0 + l;
            tile[l * PITCH + H + x] = (r < N && c < N && L0 + l < N && X0 + x < N) ? img[(long long)r * N + c] : (T)0;
        }
    } else if (O == 0) {  // rows of the image: 16-byte loads along the row, 16-byte stores
        constexpr int VPL = FP_TW / VN;
        for (int i = threadIdx.x; i < FP_TH * VPL; i += FP_THREADS) {
            const int l = i / VPL, q = i % VPL;
            const int r = L0 + l, c = X0 + q * VN;
            VT v;
            if (r < N && c < N) v = __ldg(reinterpret_cast<const VT *>(img + (long long)r * N + c));
            else memset(&v, 0, sizeof(v));
            *reinterpret_cast<VT *>(tile + l * PITCH + H + q * VN) = v;
        }
    } else {  // columns of the image: a warp reads 16-byte pieces of consecutive rows
        constexpr int VPR = FP_TH / VN;
        for (int i = threadIdx.x; i < FP_TW * VPR; i += FP_THREADS) {
            const int y = i / VPR, q = i % VPR;
            const int r = X0 + y, c = L0 + q * VN;
            VT v;
            if (r < N && c < N) v = __ldg(reinterpret_cast<const VT *>(img + (long long)r * N + c));
            else memset(&v, 0, sizeof(v));
            const T *e = reinterpret_cast<const T *>(&v);
#pragma unroll
            for (int u = 0; u < VN; u++) tile[(q * VN + u) * PITCH + H + y] = e[u];
        }
    }

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b0 = a_begin; b0 < a_end; b0 += FP_MAXA) {
        const int nb = min(FP_MAXA, a_end - b0);
        __syncthreads();  // tile staged / previous batch consumed
        // ---- static window of each angle (fp_setup): rays [jlo, jlo + W) cross the tile
        if (threadIdx.x < FP_MAXA) {
            const int k = threadIdx.x;
            int nch = 0;
            if (k < nb) {
                const int row = a.olist[b0 + k];
                const FpWin wv = a.wins[(long long)row * ntiles + tile_id];
                const FpRowGeo rg = a.rgeo[row];
                s_row[k] = row;
                s_jlo[k] = wv.jlo;
                s_W[k] = wv.W;
                s_kap[k] = wv.kap;
                s_at[k] = rg.at;
                s_B[k] = (T)rg.B;
                nch = (wv.W + 31) >> 5;
            }
            // exclusive prefix of the chunk counts over the (<= 64) angles: two warps
            int inc = nch;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_wsum[warp] = inc;
            s_cofs[k] = inc - nch;
        }
        __syncthreads();
        if (threadIdx.x >= 32 && threadIdx.x < FP_MAXA) s_cofs[threadIdx.x] += s_wsum[0];
        if (threadIdx.x == 0) s_cofs[FP_MAXA] = s_wsum[0] + s_wsum[1];
        __syncthreads();
        const int nitems = s_cofs[FP_MAXA];
        // ---- one warp item = 32 consecutive rays of one angle over the tile's TH lines
        for (int it = warp; it < nitems; it += FP_THREADS / 32) {
            int lo = 0, hi = FP_MAXA - 1;  // largest k with s_cofs[k] <= it (empty angles repeat offsets)
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_cofs[mid] <= it) lo = mid; else hi = mid - 1;
            }
            const int k = lo;
            const int W = s_W[k];
            const int w = (it - s_cofs[k]) * 32 + lane;
            const int wc = min(w, W - 1);
            const T kap = (T)(s_kap[k] + (double)wc * s_at[k]);
            const T B = s_B[k];
            const T iw = SID ? siddon_iw(B) : (T)1, hw = SID ? (T)0.5 - (T)0.5 * iw : (T)0;
            T acc0 = 0, acc1 = 0;
            if constexpr (sizeof(T) == 4) {
                const uint32_t sb = magic_base(tile, a.magic);
#pragma unroll
                for (int l = 0; l < FP_TH; l++) {
                    const float kf = fmaf((float)l, B, kap);
                    const float m = __fadd_rd(kf, 8388608.0f);     // 2^23 + floor(kf)
                    const uint32_t ad = (__float_as_uint(m) << 2) + sb;
                    const float v0 = lds<0>(ad + l * PITCH * 4), v1 = lds<4>(ad + l * PITCH * 4);
                    float f = kf - (m - 8388608.0f);
                    if (SID) f = __saturatef(fmaf(f, iw, hw));
                    acc0 += v0;
                    acc1 = fmaf(f, v1 - v0, acc1);
                }
            } else {
#pragma unroll
                for (int l = 0; l < FP_TH; l++) {
                    const T kf = fma((T)l, B, kap);
                    int i0;
                    const T fl = floor_split<T>(kf, i0);
                    T f = kf - fl;
                    if (SID) f = sat<T>(fma(f, iw, hw));
                    const T *p = tile + l * PITCH + i0;
                    const T v0 = p[0], v1 = p[1];
                    acc0 += v0;
                    acc1 = fma(f, v1 - v0, acc1);
                }
            }
            if (w < W) a.partial[((long long)s_row[k] * a.nt_line + lt) * 2 * fp_ps(a.n_det) + (ct & 1) * fp_ps(a.n_det) + s_jlo[k] + w] = acc0 + acc1;
        }
    }
}

// ------------------------------------------------------------------ forward: fp32 tile pass
// The fp32 production kernel.  Shared memory holds, for every cross index i of every
// tile line, the pair (e_i, d_i) with d_i = x_{i+1} - x_i and e_i = x_i - (i - ORG) d_i,
// so a bilinear sample at cross coordinate kf' = kf - ORG is  e_i + kf' d_i  with
// i = floor(kf):  x_i + (kf - i)(x_{i+1} - x_i).  Per sample: FFMA (position), FADD.RM
// (floor into the mantissa of 2^23 + ORG + kf'), LEA, LDS.64, FFMA + FADD (sample and
// accumulate) -- six instructions.  ORG = the middle of the padded row keeps |i - ORG|
// <= 104, so e_i loses no more than the plain lerp does.
// Rays of consecutive angles are packed into full 32-lane items.
constexpr int FP2_PITCH = FP_TW + 2 * FP_HALO_A;  // 208 pairs per line
constexpr int FP2_ORG = FP2_PITCH / 2;            // 104
constexpr float FP2_MAGIC = 8388608.0f + (float)FP2_ORG;

__device__ __forceinline__ float2 lds64(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

template <int O>
__global__ void __launch_bounds__(FP_THREADS, 4) fp_tile_f32(const FpArgs<float> a) {
    constexpr int H = FP_HALO_A;
    extern __shared__ __align__(16) unsigned char fp_smem[];
    float2 *pt = reinterpret_cast<float2 *>(fp_smem);  // [FP_TH][FP2_PITCH] (e, d)
    __shared__ double s_kap[FP_MAXA], s_at[FP_MAXA];
    __shared__ float s_B[FP_MAXA];
    __shared__ int s_row[FP_MAXA], s_jlo[FP_MAXA], s_pre[FP_MAXA + 1];

    const int node = blockIdx.y;
    const int grp = 2 * node + O;
    const int a_begin = a.oofs[grp], a_end = a.oofs[grp + 1];
    if (a_begin == a_end) return;  // uniform over the block
    const int N = a.N;
    const int tile_id = blockIdx.x;
    const int ntiles = a.nt_line * a.nt_cross;
    const int lt = tile_id / a.nt_cross, ct = tile_id % a.nt_cross;
    const int L0 = lt * FP_TH, X0 = ct * FP_TW;
    const float *img = a.img + (long long)node * a.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- stage the (e, d) pairs; x = 0 outside the image and outside [H, H + TW)
    for (int i = threadIdx.x; i < FP_TH * (FP2_PITCH - FP_TW - 1); i += FP_THREADS) {
        const int l = i / (FP2_PITCH - FP_TW - 1), k = i % (FP2_PITCH - FP_TW - 1);
        pt[l * FP2_PITCH + (k < H - 1 ? k : k + FP_TW + 1)] = make_float2(0.f, 0.f);
    }
    auto pair = [](float x, float xn, int i) {
        const float d = xn - x;
        return make_float2(fmaf(-(float)(i - FP2_ORG), d, x), d);
    };
    if ((N & 3) != 0 || ((uintptr_t)img & 15) != 0) {  // unaligned rows (stateless calls only): scalar loads
        for (int i = threadIdx.x; i < FP_TH * (FP_TW + 1); i += FP_THREADS) {
            const int l = i / (FP_TW + 1), k = i % (FP_TW + 1) - 1;  // k = -1 .. TW-1
            auto at = [&](int kk) -> float {
                if (kk < 0 || kk >= FP_TW) return 0.f;
                const int r = O == 0 ? L0 + l : X0 + kk, c = O == 0 ? X0 + kk : L0 + l;
                return (r < N && c < N) ? img[(long long)r * N + c] : 0.f;
            };
            pt[l * FP2_PITCH + H + k] = pair(at(k), at(k + 1), H + k);
        }
    } else if (O == 0) {  // a warp stages one row segment of 128: float4 per lane, neighbour by shuffle
        for (int l = warp; l < FP_TH; l += FP_THREADS / 32) {
            const int r = L0 + l, c = X0 + 4 * lane;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r < N && c < N) v = __ldg(reinterpret_cast<const float4 *>(img + (long long)r * N + c));
            float nx = __shfl_down_sync(0xffffffffu, v.x, 1);
            if (lane == 31) nx = 0.f;
            const int i0 = H + 4 * lane;
            float4 *dst = reinterpret_cast<float4 *>(pt + l * FP2_PITCH + i0);
            const float2 p0 = pair(v.x, v.y, i0), p1 = pair(v.y, v.z, i0 + 1), p2 = pair(v.z, v.w, i0 + 2),
                         p3 = pair(v.w, nx, i0 + 3);
            dst[0] = make_float4(p0.x, p0.y, p1.x, p1.y);
            dst[1] = make_float4(p2.x, p2.y, p3.x, p3.y);
            if (lane == 0) pt[l * FP2_PITCH + H - 1] = pair(0.f, v.x, H - 1);
        }
    } else {  // lines are image columns: lanes along rows (cross), float4 = 4 lines, neighbour by shuffle
        for (int job = warp; job < (FP_TW / 32) * (FP_TH / 4); job += FP_THREADS / 32) {
            const int yg = job % (FP_TW / 32), q = job / (FP_TW / 32);
            const int y = 32 * yg + lane, r = X0 + y, c = L0 + 4 * q;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r < N && c < N) v = __ldg(reinterpret_cast<const float4 *>(img + (long long)r * N + c));
            float4 nv;
            nv.x = __shfl_down_sync(0xffffffffu, v.x, 1);
            nv.y = __shfl_down_sync(0xffffffffu, v.y, 1);
            nv.z = __shfl_down_sync(0xffffffffu, v.z, 1);
            nv.w = __shfl_down_sync(0xffffffffu, v.w, 1);
            if (lane == 31) {
                nv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (y + 1 < FP_TW && r + 1 < N && c < N)
                    nv = __ldg(reinterpret_cast<const float4 *>(img + (long long)(r + 1) * N + c));
            }
            const int i = H + y;
            pt[(4 * q + 0) * FP2_PITCH + i] = pair(v.x, nv.x, i);
            pt[(4 * q + 1) * FP2_PITCH + i] = pair(v.y, nv.y, i);
            pt[(4 * q + 2) * FP2_PITCH + i] = pair(v.z, nv.z, i);
            pt[(4 * q + 3) * FP2_PITCH + i] = pair(v.w, nv.w, i);
            if (yg == 0 && lane == 0) {
                pt[(4 * q + 0) * FP2_PITCH + H - 1] = pair(0.f, v.x, H - 1);
                pt[(4 * q + 1) * FP2_PITCH + H - 1] = pair(0.f, v.y, H - 1);
                pt[(4 * q + 2) * FP2_PITCH + H - 1] = pair(0.f, v.z, H - 1);
                pt[(4 * q + 3) * FP2_PITCH + H - 1] = pair(0.f, v.w, H - 1);
            }
        }
    }

    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(pt) - a.magic;  // a.magic = 0x4B000000 << 3
    for (int b0 = a_begin; b0 < a_end; b0 += FP_MAXA) {
        const int nb = min(FP_MAXA, a_end - b0);
        __syncthreads();  // tile staged / previous batch consumed
        if (threadIdx.x < FP_MAXA) {
            const int k = threadIdx.x;
            int W = 0;
            if (k < nb) {
                const int row = a.olist[b0 + k];
                const FpWin wv = a.wins[(long long)row * ntiles + tile_id];
                const FpRowGeo rg = a.rgeo[row];
                s_row[k] = row;
                s_jlo[k] = wv.jlo;
                s_kap[k] = wv.kap - (double)FP2_ORG;
                s_at[k] = rg.at;
                s_B[k] = (float)rg.B;
                W = wv.W;
            }
            int inc = W;  // exclusive prefix of the window sizes over the (<= 64) angles
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            s_pre[k + 1] = inc;  // provisional (warp 1 adds warp 0's total below)
            if (k == 0) s_pre[0] = 0;
        }
        __syncthreads();
        if (threadIdx.x >= 32 && threadIdx.x < FP_MAXA) s_pre[threadIdx.x + 1] += s_pre[32];
        __syncthreads();
        const int R = s_pre[nb];
        // ---- one warp item = 32 consecutive rays of the batch (angles packed back to back)
        for (int g0 = warp * 32; g0 < R; g0 += FP_THREADS) {
            const int g = min(g0 + lane, R - 1);
            int lo = 0, hi = nb - 1;  // angle of the first lane, then step forward per lane
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_pre[mid] <= g0) lo = mid; else hi = mid - 1;
            }
            int k = lo;
            while (s_pre[k + 1] <= g) k++;
            const int w = g - s_pre[k];
            const float kap = (float)(s_kap[k] + (double)w * s_at[k]);
            const float B = s_B[k];
            float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
            for (int l = 0; l < FP_TH; l += 2) {
                const float kf0 = fmaf((float)l, B, kap), kf1 = fmaf((float)(l + 1), B, kap);
                const float m0 = __fadd_rd(kf0, FP2_MAGIC), m1 = __fadd_rd(kf1, FP2_MAGIC);
                const float2 q0 = lds64((__float_as_uint(m0) << 3) + sb + l * FP2_PITCH * 8);
                const float2 q1 = lds64((__float_as_uint(m1) << 3) + sb + (l + 1) * FP2_PITCH * 8);
                acc0 += fmaf(kf0, q0.y, q0.x);
                acc1 += fmaf(kf1, q1.y, q1.x);
            }
            if (g0 + lane < R)
                a.partial[((long long)s_row[k] * a.nt_line + lt) * 2 * fp_ps(a.n_det) + (ct & 1) * fp_ps(a.n_det) + s_jlo[k] + w] =
                    acc0 + acc1;
        }
    }
}

// ------------------------------------------------------------------ forward: persistent fp32
// Persistent, software-pipelined version of fp_tile_f32: each CTA walks the work units
// u = (orientation, node, tile) round-robin; while it computes unit u from the pair
// tile P, cp.async (LDGSTS) brings the raw pixels of its next unit into R and that
// unit's window records into a second table buffer, so the global-memory latency of
// staging is hidden behind the previous unit's ray walks.
constexpr int FPP_RAW = FP_TH * FP_TW;  // raw floats per unit (both orientations)

struct FpUnit {
    int O, node, tile, a_begin, a_end;
};
__device__ __forceinline__ FpUnit fp_unit(const FpArgs<float> &a, int u, int ntiles) {
    FpUnit U;
    const int per = a.L * ntiles;
    U.O = u / per;
    const int rem = u - U.O * per;
    U.node = rem / ntiles;
    U.tile = rem - U.node * ntiles;
    const int grp = 2 * U.node + U.O;
    U.a_begin = a.oofs[grp];
    U.a_end = a.oofs[grp + 1];
    return U;
}

// mbarrier / TMA helpers (sm_90+ PTX; sm_100a SASS: SYNCS / UTMALDG / UBLKCP)
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned phase) {
    unsigned ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, unsigned bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// rays per half-warp item: 16 lanes on one line span <= 16 consecutive pair slots
__device__ __forceinline__ int fp_half_rays(double at) {
    const int h = (int)(15.0 / fabs(at)) + 1;
    return h < 1 ? 1 : (h > 16 ? 16 : h);
}

// Persistent, TMA-pipelined forward tile pass.  Each CTA walks the work units
// u = (orientation, node, tile) round-robin; while it computes unit u from the pair
// tile P, one thread has already issued the TMA tensor load of unit u+grid's raw tile
// (y-major: a 32 x 128 box of the [L][N][N] images; x-major: a 128 x 32 box stored with
// the 128-byte swizzle, i.e. conflict-free column reads) and a bulk copy of its window
// records, both completing on one mbarrier.  Out-of-image pixels are zero-filled by TMA.
template <bool SID>  // SID: Siddon weights (R-26) over natural pairs (x_i, d_i)
__global__ void __launch_bounds__(FP_THREADS, 3) fp_persist_f32(const FpArgs<float> a, int nunits,
                                                                const __grid_constant__ CUtensorMap tm_rows,
                                                                const __grid_constant__ CUtensorMap tm_cols) {
    constexpr int H = FP_HALO_A;
    extern __shared__ __align__(16) unsigned char fp_smem_raw[];
    // raw first, 1024-byte aligned (TMA 128-byte swizzle)
    unsigned char *fp_smem = fp_smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(fp_smem_raw) & 1023u)) & 1023u);
    float *raw = reinterpret_cast<float *>(fp_smem);                          // [FPP_RAW]
    float2 *pt = reinterpret_cast<float2 *>(raw + FPP_RAW);                    // [TH][PITCH] (e, d)
    FpRec *rec = reinterpret_cast<FpRec *>(pt + FP_TH * FP2_PITCH);            // [2][FPP_MAXA]
    FpUnitTab *utb = reinterpret_cast<FpUnitTab *>(rec + 2 * FPP_MAXA);          // [2]
    __shared__ __align__(8) unsigned long long bar;
    __shared__ int s_hdr[2][8];  // per unit buffer: O, tile, a_begin, a_end, lt, ct (written by thread 0)
    const int ntiles = a.nt_line * a.nt_cross;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t raw_s = (uint32_t)__cvta_generic_to_shared(raw);
    const uint32_t rec_s = (uint32_t)__cvta_generic_to_shared(rec);
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);

    // halo pairs are (0, 0) for every unit
    for (int i = threadIdx.x; i < FP_TH * (FP2_PITCH - FP_TW - 1); i += FP_THREADS) {
        const int l = i / (FP2_PITCH - FP_TW - 1), k = i % (FP2_PITCH - FP_TW - 1);
        pt[l * FP2_PITCH + (k < H - 1 ? k : k + FP_TW + 1)] = make_float2(0.f, 0.f);
    }
    if (threadIdx.x == 0) {
        mbar_init(bar_s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // the images come from the previous kernel
    // thread 0: decodes unit u into s_hdr[rb] and issues the TMA of its raw tile + bulk
    // copies of its first window records and item plan (units without angles of their
    // orientation load only the tile and are skipped); every thread learns whether a load
    // is pending from u alone, so the integer divisions of the decode run in one thread
    auto issue = [&](int u, int rb) -> bool {
        if (u >= nunits) return false;
        if (threadIdx.x == 0) {
            const FpUnit U = fp_unit(a, u, ntiles);
            // unit tables are laid out over all L_all nodes: (O, node0 + node, tile)
            const long long ug = ((long long)U.O * a.L_all + a.node0 + U.node) * ntiles + U.tile;
            const int lt = U.tile / a.nt_cross, ct = U.tile % a.nt_cross;
            s_hdr[rb][0] = U.O; s_hdr[rb][1] = U.tile; s_hdr[rb][2] = U.a_begin; s_hdr[rb][3] = U.a_end;
            s_hdr[rb][4] = lt; s_hdr[rb][5] = ct;
            const int L0 = lt * FP_TH, X0 = ct * FP_TW;
            const int nb = min(FPP_MAXA, U.a_end - U.a_begin);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of raw before the async write
            mbar_expect_tx(bar_s, FPP_RAW * 4 + (nb > 0 ? nb * (unsigned)sizeof(FpRec) + (unsigned)sizeof(FpUnitTab) : 0u));
            if (U.O == 0) tma_load_3d(raw_s, &tm_rows, X0, L0, U.node, bar_s);
            else tma_load_3d(raw_s, &tm_cols, L0, X0, U.node, bar_s);
            if (nb > 0) {
                bulk_load(rec_s + (uint32_t)(rb * FPP_MAXA * sizeof(FpRec)), a.recs + (long long)U.tile * a.n_olist + U.a_begin,
                          nb * (unsigned)sizeof(FpRec), bar_s);
                bulk_load((uint32_t)__cvta_generic_to_shared(utb + rb), a.utab + ug, (unsigned)sizeof(FpUnitTab), bar_s);
            }
        }
        return true;
    };
    auto pair = [](float x, float xn, int i) {
        const float d = xn - x;
        return SID ? make_float2(x, d) : make_float2(fmaf(-(float)(i - FP2_ORG), d, x), d);
    };

    int rb = 0;
    unsigned phase = 0;
    bool pending = issue(blockIdx.x, rb);
    for (int u = blockIdx.x; u < nunits; u += gridDim.x, rb ^= 1) {
        if (pending) {
            mbar_wait(bar_s, phase);
            phase ^= 1;
        }
        __syncthreads();  // raw + rec[rb] of unit u landed; previous unit's P reads done; s_hdr[rb] set
        FpUnit U;
        U.O = s_hdr[rb][0]; U.tile = s_hdr[rb][1]; U.a_begin = s_hdr[rb][2]; U.a_end = s_hdr[rb][3];
        const bool active = U.a_begin != U.a_end;
        const int lt = s_hdr[rb][4], ct = s_hdr[rb][5];
        if (active) {  // ---- raw -> (e, d) pairs
            if (U.O == 0) {
                // lane-consecutive 8-byte reads and 16-byte stores (two pixels' pairs per store):
                // every access of a warp is one contiguous run, no bank conflicts
                for (int l = warp; l < FP_TH; l += FP_THREADS / 32) {
                    const float2 *rr = reinterpret_cast<const float2 *>(raw + l * FP_TW);
                    const float2 va = rr[lane], vb = rr[lane + 32];  // pixels 2 lane (+1), 64 + 2 lane (+1)
                    float na = __shfl_down_sync(0xffffffffu, va.x, 1);
                    float nb = __shfl_down_sync(0xffffffffu, vb.x, 1);
                    const float v64 = __shfl_sync(0xffffffffu, vb.x, 0);
                    if (lane == 31) { na = v64; nb = 0.f; }
                    const int ia = H + 2 * lane, ib = ia + 64;
                    const float2 p0 = pair(va.x, va.y, ia), p1 = pair(va.y, na, ia + 1);
                    const float2 p2 = pair(vb.x, vb.y, ib), p3 = pair(vb.y, nb, ib + 1);
                    *reinterpret_cast<float4 *>(pt + l * FP2_PITCH + ia) = make_float4(p0.x, p0.y, p1.x, p1.y);
                    *reinterpret_cast<float4 *>(pt + l * FP2_PITCH + ib) = make_float4(p2.x, p2.y, p3.x, p3.y);
                    if (lane == 0) pt[l * FP2_PITCH + H - 1] = pair(0.f, va.x, H - 1);
                }
            } else {
                for (int job = warp; job < (FP_TW / 32) * (FP_TH / 4); job += FP_THREADS / 32) {
                    const int yg = job % (FP_TW / 32), q = job / (FP_TW / 32);
                    const int y = 32 * yg + lane;
                    const float4 v = *reinterpret_cast<const float4 *>(raw + 4 * (8 * y + (q ^ (y & 7))));
                    float4 nv;
                    nv.x = __shfl_down_sync(0xffffffffu, v.x, 1);
                    nv.y = __shfl_down_sync(0xffffffffu, v.y, 1);
                    nv.z = __shfl_down_sync(0xffffffffu, v.z, 1);
                    nv.w = __shfl_down_sync(0xffffffffu, v.w, 1);
                    if (lane == 31) {
                        const int y1 = y + 1;
                        nv = y1 < FP_TW ? *reinterpret_cast<const float4 *>(raw + 4 * (8 * y1 + (q ^ (y1 & 7))))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    const int i = H + y;
                    pt[(4 * q + 0) * FP2_PITCH + i] = pair(v.x, nv.x, i);
                    pt[(4 * q + 1) * FP2_PITCH + i] = pair(v.y, nv.y, i);
                    pt[(4 * q + 2) * FP2_PITCH + i] = pair(v.z, nv.z, i);
                    pt[(4 * q + 3) * FP2_PITCH + i] = pair(v.w, nv.w, i);
                    if (yg == 0 && lane == 0) {
                        pt[(4 * q + 0) * FP2_PITCH + H - 1] = pair(0.f, v.x, H - 1);
                        pt[(4 * q + 1) * FP2_PITCH + H - 1] = pair(0.f, v.y, H - 1);
                        pt[(4 * q + 2) * FP2_PITCH + H - 1] = pair(0.f, v.z, H - 1);
                        pt[(4 * q + 3) * FP2_PITCH + H - 1] = pair(0.f, v.w, H - 1);
                    }
                }
            }
        }
        __syncthreads();  // P ready; raw free
        pending = issue(u + gridDim.x, rb ^ 1);
        if (!active) continue;
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(pt) - a.magic;
        for (int b0 = U.a_begin; b0 < U.a_end; b0 += FPP_MAXA) {
            const int nb = min(FPP_MAXA, U.a_end - b0);
            FpRec *R = rec + rb * FPP_MAXA;
            if (b0 != U.a_begin) {  // later batches (> 64 angles per orientation): plain loads
                __syncthreads();
                for (int k = threadIdx.x; k < nb; k += FP_THREADS) R[k] = a.recs[(long long)U.tile * a.n_olist + b0 + k];
                __syncthreads();
            }
            FpUnitTab &ut = utb[rb];
            if (b0 != U.a_begin) {  // later batches: plan computed here, over the unit's table
                if (threadIdx.x < FPP_MAXA) {
                    const int k = threadIdx.x;
                    const int nh = k < nb ? fp_half_rays(R[k].at) : 1;
                    int inc = k < nb ? (R[k].W + nh - 1) / nh : 0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, inc, o);
                        if (lane >= o) inc += y;
                    }
                    ut.hpre[k + 1] = inc;
                    ut.nh[k] = (unsigned char)nh;
                    if (k == 0) ut.hpre[0] = 0;
                }
                __syncthreads();
                for (int k = threadIdx.x; k < nb; k += FP_THREADS)
                    for (int it = ut.hpre[k]; it < ut.hpre[k + 1]; it++) ut.hk[it] = fp_hk_pack(k, ut.nh[k], it - ut.hpre[k]);
                __syncthreads();
            }
            const unsigned short *hk = ut.hk;
            const int Hn = ut.hpre[nb];
            const int hl = lane & 15;
            // one warp item = two half-warp items (each nh_k <= 16 rays of one angle)
            for (int h0 = 2 * warp; h0 < Hn; h0 += 2 * (FP_THREADS / 32)) {
                const int hraw = h0 + (lane >> 4);
                const int hi = min(hraw, Hn - 1);
                const unsigned pk = hk[hi];
                const int k = pk & 31, nh = (pk >> 5) & 31, rk = (int)(pk >> 10);
                const double2 ka = *reinterpret_cast<const double2 *>(&R[k].kap);  // (kap, at)
                const int4 bj = *reinterpret_cast<const int4 *>(&R[k].B);          // (B, jlo, W, row)
                const int W = bj.z;
                const int w0 = rk * nh + hl;
                const bool ok = hraw < Hn && hl < nh && w0 < W;
                const int w = min(min(w0, rk * nh + nh - 1), W - 1);  // idle lanes repeat a ray
                const float kap = (float)(ka.x + (double)w * ka.y);
                const float B = __int_as_float(bj.x);
                float acc0 = 0.f, acc1 = 0.f;
                if (!SID) {
                    // lines l, l + 1 as one packed pair: FFMA2 (positions), FADD2.RM (floors) and
                    // FADD2 (accumulate) -- the same IEEE operations as the scalar form, two per issue
                    const float2 B2 = make_float2(B, B), kap2 = make_float2(kap, kap);
                    const float2 mg2 = make_float2(FP2_MAGIC, FP2_MAGIC);
                    float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int l = 0; l < FP_TH; l += 2) {
                        const float2 kf = __ffma2_rn(make_float2((float)l, (float)(l + 1)), B2, kap2);
                        const float2 m = __fadd2_rd(kf, mg2);
                        const float2 q0 = lds64((__float_as_uint(m.x) << 3) + sb + l * FP2_PITCH * 8);
                        const float2 q1 = lds64((__float_as_uint(m.y) << 3) + sb + (l + 1) * FP2_PITCH * 8);
                        acc2 = __fadd2_rn(acc2, make_float2(fmaf(kf.x, q0.y, q0.x), fmaf(kf.y, q1.y, q1.x)));
                    }
                    acc0 = acc2.x;
                    acc1 = acc2.y;
                } else {  // pixel a + 1 gets g = sat((u - 1/2) / w + 1/2) of the band's length
                    const float iw = siddon_iw(B), hw = 0.5f - 0.5f * iw;
                    const float2 B2 = make_float2(B, B), kap2 = make_float2(kap, kap);
                    const float2 mg2 = make_float2(FP2_MAGIC, FP2_MAGIC), nmg2 = make_float2(-FP2_MAGIC, -FP2_MAGIC);
                    const float2 m1v = make_float2(-1.0f, -1.0f);
                    float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int l = 0; l < FP_TH; l += 2) {  // line pairs packed as in the Joseph loop
                        const float2 kf = __ffma2_rn(make_float2((float)l, (float)(l + 1)), B2, kap2);
                        const float2 m = __fadd2_rd(kf, mg2);
                        const float2 q0 = lds64((__float_as_uint(m.x) << 3) + sb + l * FP2_PITCH * 8);
                        const float2 q1 = lds64((__float_as_uint(m.y) << 3) + sb + (l + 1) * FP2_PITCH * 8);
                        const float2 u = __ffma2_rn(__fadd2_rn(m, nmg2), m1v, kf);  // kf - floor(kf)
                        const float g0 = __saturatef(fmaf(u.x, iw, hw)), g1 = __saturatef(fmaf(u.y, iw, hw));
                        acc2 = __fadd2_rn(acc2, make_float2(fmaf(g0, q0.y, q0.x), fmaf(g1, q1.y, q1.x)));
                    }
                    acc0 = acc2.x;
                    acc1 = acc2.y;
                }
                if (ok)
                    a.partial[((long long)bj.w * a.nt_line + lt) * 2 * fp_ps(a.n_det) + (ct & 1) * fp_ps(a.n_det) + bj.y + w] =
                        acc0 + acc1;
            }
            if (b0 + FPP_MAXA < U.a_end) __syncthreads();  // R / plan reuse by the next batch
        }
    }
    if (pending) mbar_wait(bar_s, phase);
}

// ------------------------------------------------------------------ forward: static windows
// For every (ray row, tile): the rays whose cross coordinate over the tile's real lines
// meets (X0 - 1, X0 + TW), padded by one ray below and two above, and the shared-memory
// cross coordinate of the first of them on the tile's first line.
__global__ void fp_setup_kernel(const RayRow *rows, const int *xmaj, const double2 *trig, int n_rows, int N,
                                int n_det, FpWin *wins, FpRowGeo *rgeo) {
    const int nt_line = (N + FP_TH - 1) / FP_TH, nt_cross = (N + FP_TW - 1) / FP_TW;
    const int ntiles = nt_line * nt_cross;
    const int row = blockIdx.y;
    const int ang = rows[row].angle;
    const int O = xmaj[ang];
    const double2 t2 = trig[ang];
    const LineGeo G = line_geo(t2.x, t2.y, O, N);
    const double c0 = 0.5 * (double)(n_det - 1);
    if (blockIdx.x == 0 && threadIdx.x == 0) rgeo[row] = FpRowGeo{G.at, G.B, G.a0};
    for (int tile = blockIdx.x * blockDim.x + threadIdx.x; tile < ntiles; tile += gridDim.x * blockDim.x) {
        const int lt = tile / nt_cross, ct = tile % nt_cross;
        const int L0 = lt * FP_TH, X0 = ct * FP_TW;
        const double l1 = (double)(min(L0 + FP_TH, N) - 1);
        const double bA = (double)L0 * G.B, bB = l1 * G.B;
        const double lo = (double)(X0 - 1) - fmax(bA, bB) - G.a0;   // t*at in (lo, hi)
        const double hi = (double)(X0 + FP_TW) - fmin(bA, bB) - G.a0;
        double tl = lo / G.at, th = hi / G.at;
        if (tl > th) { const double x = tl; tl = th; th = x; }
        const int jlo = max(0, (int)floor(tl + c0) - 1);
        const int jhi = min(n_det, (int)ceil(th + c0) + 2);
        FpWin w;
        w.jlo = jlo;
        w.W = max(0, jhi - jlo);
        w.kap = G.a0 + ((double)jlo - c0) * G.at + (double)L0 * G.B - (double)(X0 - FP_HALO_A);
        wins[(long long)row * ntiles + tile] = w;
    }
}

__global__ void fp_rec_kernel(const int *olist, int n_olist, int ntiles, const FpWin *wins,
                              const FpRowGeo *rgeo, FpRec *recs) {
    const int pos = blockIdx.y;
    const int row = olist[pos];
    for (int tile = blockIdx.x * blockDim.x + threadIdx.x; tile < ntiles; tile += gridDim.x * blockDim.x) {
        const FpWin w = wins[(long long)row * ntiles + tile];
        FpRec r;
        r.kap = w.kap - (double)FP2_ORG;
        r.at = rgeo[row].at;
        r.B = (float)rgeo[row].B;
        r.jlo = w.jlo;
        r.W = w.W;
        r.row = row;
        recs[(long long)tile * n_olist + pos] = r;
    }
}

__global__ void fp_unit_kernel(const int *oofs, const FpRec *recs, int n_olist, int ntiles, int L, FpUnitTab *utab) {
    __shared__ int pre[FPP_MAXA + 1];
    __shared__ unsigned char nhs[FPP_MAXA];
    const int u = blockIdx.x, per = L * ntiles;
    const int O = u / per, rem = u - O * per, node = rem / ntiles, tile = rem - node * ntiles;
    const int a0 = oofs[2 * node + O], a1 = oofs[2 * node + O + 1];
    const int nb = min(FPP_MAXA, a1 - a0);
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < FPP_MAXA; k++) {
            pre[k] = acc;
            int nh = 1;
            if (k < nb) {
                const FpRec r = recs[(long long)tile * n_olist + a0 + k];
                nh = fp_half_rays(r.at);
                acc += (r.W + nh - 1) / nh;
            }
            nhs[k] = (unsigned char)nh;
        }
        pre[FPP_MAXA] = acc;
    }
    __syncthreads();
    FpUnitTab *t = utab + u;
    for (int k = threadIdx.x; k <= FPP_MAXA; k += blockDim.x) t->hpre[k] = pre[k];
    for (int k = threadIdx.x; k < FPP_MAXA; k += blockDim.x) t->nh[k] = nhs[k];
    for (int it = threadIdx.x; it < FPP_HMAX; it += blockDim.x) {
        int lo = 0, hi = max(nb - 1, 0);  // angle of half-item it: largest k with pre[k] <= it
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= it) lo = mid; else hi = mid - 1;
        }
        t->hk[it] = fp_hk_pack(lo, nhs[lo], it - pre[lo]);
    }
}

// ------------------------------------------------------------------ forward: reduction
// s[row][j] = (1/m) * sum over line bands of the two parity slots; RESID: d - A x.
// RG groups of threads split the bands of 32 bins (one round of <= 16 independent loads
// per thread for nt_line <= 8 RG), then the group partials are added in a fixed order in
// shared memory (deterministic, no atomics).
constexpr int RJ = 32, RG = 4;  // bins per CTA, band groups
template <typename T>
__device__ __forceinline__ double fp_row_m(const FpRedArgs<T> &a, int row) {
    if (a.rowc) return a.rowc[row].z;
    const int ang = a.rows[row].angle;
    const double2 t2 = a.trig[ang];
    return a.xmaj[ang] ? fabs(t2.y) : fabs(t2.x);
}
// CG step: this CTA's sum of squared outputs into cgs (see FpRedArgs::cg); all threads call it
template <typename T, int NT>
__device__ __forceinline__ void fp_cg_partial(const FpRedArgs<T> &a, int row, double ss, double *red) {
    const double bs = block_sum<NT>(ss, red);
    if (threadIdx.x == 0) {
        const RayRow rr = a.rows[row];
        a.cgs[(long long)rr.node * a.part_stride + (long long)rr.k * gridDim.x + blockIdx.x] = bs;
    }
}

template <typename T, bool RESID>
__global__ void __launch_bounds__(RJ * RG) fp_reduce_kernel(const FpRedArgs<T> a) {
    __shared__ T part[RG][RJ];
    const int row = blockIdx.y + a.row_base;
    const double m_row = fp_row_m(a, row);  // issued first: its latency overlaps the slot loads
    const int jj = threadIdx.x % RJ, g = threadIdx.x / RJ;
    const int j = blockIdx.x * RJ + jj;
    const int nb = a.nt_line;
    const int per = (nb + RG - 1) / RG;
    const int l0 = g * per, l1 = min(nb, l0 + per);
    T acc = 0;
    if (j < a.n_det) {
        const int nd = fp_ps(a.n_det);  // slot row stride
        // 32-bit element offsets from the row's first slot (a row holds nt_line * 2 * stride
        // slots): one IMAD.WIDE per load instead of 64-bit multiplies
        const T *p = a.partial + (long long)row * nb * 2 * nd + j;
        int lt = l0;
        for (; lt + 8 <= l1; lt += 8) {  // 16 loads in flight
            T x[16];
            const T *q = p + 2 * lt * nd;
            asm("" : "+l"(q));  // keep q as a base register: one IMAD.WIDE per load below
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = __ldcg(q + u * nd);
            T s8[8];
#pragma unroll
            for (int u = 0; u < 8; u++) s8[u] = x[2 * u] + x[2 * u + 1];
            acc += ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
        }
        for (; lt < l1; lt++) acc += p[2 * lt * nd] + p[(2 * lt + 1) * nd];
    }
    part[g][jj] = acc;
    __syncthreads();
    double ss = 0.0;
    if (g == 0 && j < a.n_det) {
        T tot = part[0][jj];
#pragma unroll
        for (int q = 1; q < RG; q++) tot += part[q][jj];
        const double inv_m = 1.0 / m_row;
        T v = (T)((double)tot * inv_m);
        if (RESID) v = a.d[(long long)row * a.n_det + j] - v;
        a.out[(long long)row * a.out_stride + a.out_off + j] = v;
        ss = (double)v * (double)v;
    }
    if (!RESID && a.cg) {
        __shared__ double red[RJ * RG / 32 + 1];
        fp_cg_partial<T, RJ * RG>(a, row, ss, red);
    }
}

// fp32: four bins per thread (16-byte slot loads; the slot rows are padded to a multiple of
// four bins and the padding is never written, so it stays zero), RQ quads x RG band groups.
// With the row geometry (a.rgeo) a quad reads only the parity slots of the cross tiles its
// rays can cross in each band: the rays' cross coordinate over the band's lines, widened
// by a margin that covers the windows' padding (fp_setup_kernel), selects the cross tiles;
// the other slots are never written, i.e. zero, and are skipped (the sum is unchanged).
struct FpNeed {  // fp32 row geometry of one quad for fp_band_need
    float ca, cb, B, M;
    int N, nt_cross;
};
__device__ __forceinline__ unsigned fp_band_need(const FpNeed &n, int lt) {
    const int L0 = lt * FP_TH, L1 = min(L0 + FP_TH, n.N) - 1;
    const float bA = (float)L0 * n.B, bB = (float)L1 * n.B;
    const float cmin = n.ca + fminf(bA, bB) - n.M, cmax = n.cb + fmaxf(bA, bB) + n.M;
    const int lo = max(0, __float2int_rd(cmin * (1.0f / FP_TW)));
    const int hi = min(n.nt_cross - 1, __float2int_rd(cmax * (1.0f / FP_TW)));
    // bit 0: the even-parity slot, bit 1: the odd one
    return lo < hi ? 3u : (lo == hi ? 1u << (lo & 1) : 0u);
}
// 16-byte L2 load issued under a predicate (zeros otherwise): a run of these stays one
// batch of independent loads instead of a branch per load
__device__ __forceinline__ float4 ldcg_if(const float4 *p, unsigned c) {
    float4 v;
    asm(
        "{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n mov.b32 %2, 0;\n mov.b32 %3, 0;\n"
        " @q ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];\n}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "r"(c));
    return v;
}
constexpr int RQ = 32;
template <bool RESID>
__global__ void __launch_bounds__(RQ * RG) fp_reduce_f32(const FpRedArgs<float> a) {
    pdl_wait();
    __shared__ float4 part[RG][RQ];
    const int row = blockIdx.y + a.row_base;
    const double m_row = fp_row_m(a, row);  // issued first: its latency overlaps the slot loads
    const int q = threadIdx.x % RQ, g = threadIdx.x / RQ;
    const int j0 = 4 * (blockIdx.x * RQ + q);
    const int nb = a.nt_line, nd = fp_ps(a.n_det);
    const int per = (nb + RG - 1) / RG;
    const int l0 = g * per, l1 = min(nb, l0 + per);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j0 < a.n_det) {
        const float4 *p = reinterpret_cast<const float4 *>(a.partial + (long long)row * nb * 2 * nd + j0);
        const int nq = nd / 4;  // slot row stride in quads
        // cross coordinate range of the quad's rays before the line term (a.rgeo: see above);
        // fp32 is ample: |error| << the margin M of the windows' padding
        FpNeed nn{-1e30f, 1e30f, 0.f, 0.f, a.N, a.nt_cross};
        if (a.rgeo) {
            const FpRowGeo G = a.rgeo[row];
            const double c0 = 0.5 * (double)(a.n_det - 1);
            const double u0 = ((double)j0 - c0) * G.at, u1 = ((double)(j0 + 3) - c0) * G.at;
            nn.ca = (float)(G.a0 + fmin(u0, u1));
            nn.cb = (float)(G.a0 + fmax(u0, u1));
            nn.B = (float)G.B;
            nn.M = (float)(8.0 + 3.0 * fabs(G.at));
        }
        int lt = l0;
        constexpr int FB = 8;  // bands per batch: up to 16 quads in flight (the sums keep band order)
        for (; lt + FB <= l1; lt += FB) {
            unsigned nm[FB];
#pragma unroll
            for (int u = 0; u < FB; u++) nm[u] = a.rgeo ? fp_band_need(nn, lt + u) : 3u;
            float4 x[2 * FB];
#pragma unroll
            for (int u = 0; u < FB; u++) {
                x[2 * u] = ldcg_if(p + (2 * (lt + u)) * nq, nm[u] & 1u);
                x[2 * u + 1] = ldcg_if(p + (2 * (lt + u) + 1) * nq, nm[u] & 2u);
            }
#pragma unroll
            for (int u = 0; u < 2 * FB; u += 2) {
                acc.x += x[u].x + x[u + 1].x;
                acc.y += x[u].y + x[u + 1].y;
                acc.z += x[u].z + x[u + 1].z;
                acc.w += x[u].w + x[u + 1].w;
            }
        }
        for (; lt < l1; lt++) {
            const unsigned nm = a.rgeo ? fp_band_need(nn, lt) : 3u;
            const float4 x0 = ldcg_if(p + 2 * lt * nq, nm & 1u), x1 = ldcg_if(p + (2 * lt + 1) * nq, nm & 2u);
            acc.x += x0.x + x1.x;
            acc.y += x0.y + x1.y;
            acc.z += x0.z + x1.z;
            acc.w += x0.w + x1.w;
        }
    }
    part[g][q] = acc;
    __syncthreads();
    double ss = 0.0;
    if (g == 0 && j0 < a.n_det) {
        float4 tot = part[0][q];
#pragma unroll
        for (int r = 1; r < RG; r++) {
            tot.x += part[r][q].x;
            tot.y += part[r][q].y;
            tot.z += part[r][q].z;
            tot.w += part[r][q].w;
        }
        const double inv_m = 1.0 / m_row;
        const float tv[4] = {tot.x, tot.y, tot.z, tot.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int j = j0 + e;
            if (j >= a.n_det) break;
            float v = (float)((double)tv[e] * inv_m);
            if (RESID) v = a.d[(long long)row * a.n_det + j] - v;
            a.out[(long long)row * a.out_stride + a.out_off + j] = v;
            ss += (double)v * (double)v;
        }
    }
    if (!RESID && a.cg) {
        __shared__ double red[RQ * RG / 32 + 1];
        fp_cg_partial<float, RQ * RG>(a, row, ss, red);
    }
}

// ------------------------------------------------------------------ backprojector
template <typename T, int EPI>
__global__ void __launch_bounds__(BP_THREADS, sizeof(T) == 4 ? 4 : 1)
bp_tile_kernel(const BpArgs<T> a) {
    pdl_wait();
    constexpr int BP_MAXA = bp_maxa<T, EPI>();  // angles per staged batch of this variant
    extern __shared__ __align__(16) unsigned char bp_smem[];
    T *win = reinterpret_cast<T *>(bp_smem);  // [BP_MAXA][BP_WB], bins pre-scaled by 1/m (fp64)
    float2 *win2 = reinterpret_cast<float2 *>(bp_smem);  // fp32: [BP_MAXA][BP_WB] pairs (s'_j, s'_{j+1})
    // fp32: the epilogue operands of the tile, prefetched with cp.async at entry so their
    // latency overlaps the angle loop: ep[0] = vin (p or x), ep[1] = b' (RESID, GD) or r (CGR)
    float *ep = reinterpret_cast<float *>(bp_smem + (sizeof(T) == 4 ? sizeof(float2) : sizeof(T)) * BP_MAXA * BP_WB);
    // per-angle constants of the angle loop, packed so a thread reads them with three 16-byte loads
    struct __align__(16) AngC { double tau, csd, snd, pad; T cs, sn, a1, a0; };
    __shared__ AngC s_ang[BP_MAXA];
    __shared__ T s_im[BP_MAXA];
    __shared__ int s_jlo[BP_MAXA];
    __shared__ const T *s_src[BP_MAXA];
    __shared__ double red[BP_THREADS / 32 + 1];
    __shared__ bool last_flag;
    const int node = blockIdx.y;
    const int N = a.N;
    const int tpr = (N + BP_TS - 1) / BP_TS;
    const int r0 = (blockIdx.x / tpr) * BP_TS, c0 = (blockIdx.x % tpr) * BP_TS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lx = lane & 7, prow = 8 * warp + (lane >> 3);  // pixel (prow + 4 ky, 8 kx + lx)
    const double h = 0.5 * (double)(N - 1), t0 = -0.5 * (double)(a.n_det - 1);
    const int nang = a.node_nang[node], row0 = a.node_row0[node];
    constexpr int NEP = (EPI == EPI_CGQ) ? 1 : ((EPI == EPI_RESID || EPI == EPI_GD || EPI == EPI_CGR) ? 2 : 0);
    const bool pre = sizeof(T) == 4 && NEP > 0 && (N & 3) == 0;
    if (pre) {
        const long long nb0 = (long long)node * a.n;
        const uint32_t eps = (uint32_t)__cvta_generic_to_shared(ep);
        // thread t copies the 16-byte pieces (row t/16 + 16 i, columns 4 (t%16) .. +3) of each operand
        constexpr int RPI = BP_THREADS / (BP_TS / 4);  // rows per pass (16)
        const int tr = threadIdx.x / (BP_TS / 4), tc = 4 * (threadIdx.x % (BP_TS / 4));
        const bool col_ok = c0 + tc < N;
#pragma unroll
        for (int o = 0; o < NEP; o++) {
            const float *src = reinterpret_cast<const float *>(o == 0 ? (const void *)a.vin : (const void *)a.bprime) + nb0;
            const float *p0 = src + (long long)(r0 + tr) * N + c0 + tc;
            const uint32_t d0 = eps + 4u * (o * BP_TS * BP_TS + tr * BP_TS + tc);
#pragma unroll
            for (int i = 0; i < BP_TS / RPI; i++) {
                const bool ok = col_ok && r0 + tr + RPI * i < N;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d0 + 4u * RPI * BP_TS * i),
                             "l"(ok ? p0 + (long long)RPI * i * N : src), "r"(ok ? 16 : 0));
            }
        }
        asm volatile("cp.async.commit_group;");
    }
    T acc[2][8];
    float2 acc2[2][8];  // fp32: per pixel the (lower-tap, upper-tap) partial sums
#pragma unroll
    for (int ky = 0; ky < 2; ky++)
#pragma unroll
        for (int kx = 0; kx < 8; kx++) {
            acc[ky][kx] = 0;
            acc2[ky][kx] = make_float2(0.f, 0.f);
        }

    for (int k0 = 0; k0 < nang; k0 += BP_MAXA) {
        const int kc = min(BP_MAXA, nang - k0);
        __syncthreads();
        for (int k = threadIdx.x; k < kc; k += BP_THREADS) {
            double cs, sn, m, iw;
            if (a.rowc) {
                const double4 rc = a.rowc[row0 + k0 + k];
                cs = rc.x; sn = rc.y; m = rc.z; iw = rc.w;
            } else {
                const int ang = a.rows[row0 + k0 + k].angle;
                const double2 t2 = a.trig[ang];
                cs = t2.x; sn = t2.y;
                m = a.xmaj[ang] ? fabs(sn) : fabs(cs);
                const double w = a.xmaj[ang] ? fabs(cs / sn) : fabs(sn / cs);
                iw = w > 1e-9 ? 1.0 / w : 4194304.0;
            }
            const double tp0 = ((double)c0 - h) * cs + (h - (double)r0) * sn;  // t_p of pixel (r0, c0)
            const double ext = (double)(BP_TS - 1);
            const double tmin = tp0 + fmin(0.0, ext * cs) + fmin(0.0, -ext * sn);
            const int jlo = (int)floor(tmin - t0) - 1;  // one bin of margin below
            s_jlo[k] = jlo;
            s_src[k] = a.s + (long long)(row0 + k0 + k) * a.s_stride + a.s_off + jlo;
            AngC ac;
            ac.tau = tp0 - t0 - (double)jlo;  // tile-relative bin coordinate of pixel (r0, c0)
            ac.csd = cs;
            ac.snd = sn;
            ac.pad = 0.0;
            ac.cs = (T)cs;
            ac.sn = (T)sn;
            s_im[k] = (T)(1.0 / m);
            // tap weight sat(a0 - s a1) at bin distance s (times the 1/m pre-scale): Joseph
            // a1 = 1/m, a0 = 1; Siddon (R-26) a1 = 1/(m w), a0 = (1 + 1/w)/2, w = drift per line
            if (a.siddon) {
                ac.a1 = (T)(iw / m);
                ac.a0 = (T)(0.5 + 0.5 * iw);
            } else {
                ac.a1 = (T)(1.0 / m);
                ac.a0 = (T)1;
            }
            s_ang[k] = ac;
        }
        __syncthreads();
        // bins of the window: zero guards / pads stand in for j < 0 and j >= n_det (SPAD)
        if constexpr (sizeof(T) == 4) {
            // a warp per angle row: each bin loaded once, its right neighbour by shuffle
            static_assert(BP_WB == 96, "three bins per lane");
            for (int k = warp; k < kc; k += BP_THREADS / 32) {
                const T *src = s_src[k];
                const T im = s_im[k];
                const float v0 = __ldg(src + lane), v1 = __ldg(src + lane + 32), v2 = __ldg(src + lane + 64);
                const float v3 = lane == 0 ? __ldg(src + 96) : 0.f;
                const float n0 = __shfl_down_sync(0xffffffffu, v0, 1), n1 = __shfl_down_sync(0xffffffffu, v1, 1),
                            n2 = __shfl_down_sync(0xffffffffu, v2, 1);
                const float f1 = __shfl_sync(0xffffffffu, v1, 0), f2 = __shfl_sync(0xffffffffu, v2, 0),
                            f3 = __shfl_sync(0xffffffffu, v3, 0);
                float2 *row = win2 + k * BP_WB;
                row[lane] = make_float2(v0 * im, (lane == 31 ? f1 : n0) * im);
                row[lane + 32] = make_float2(v1 * im, (lane == 31 ? f2 : n1) * im);
                row[lane + 64] = make_float2(v2 * im, (lane == 31 ? f3 : n2) * im);
            }
        } else {
            for (int i = threadIdx.x; i < kc * BP_WB; i += BP_THREADS) {
                const int k = i / BP_WB, w = i - k * BP_WB;
                win[i] = __ldg(s_src[k] + w) * s_im[k];
            }
        }
        __syncthreads();
        for (int k = 0; k < kc; k++) {
            const AngC ac = s_ang[k];
            const T cs = ac.cs, sn = ac.sn, a1 = ac.a1, a0 = ac.a0, a0m = a0 - a1;
            const T tau_t = (T)(ac.tau + (double)lx * ac.csd - (double)prow * ac.snd);
            if constexpr (sizeof(T) == 4) {
                const uint32_t wb = magic_base(win2 + k * BP_WB, a.magic);  // magic = 0x4B000000 << 3
                // pixels kx, kx + 1 as one packed pair for the position, floor and fraction
                // (FFMA2 / FADD2.RM / FADD2 / FFMA2: the scalar form's IEEE operations, two per issue)
                const float2 cs2 = make_float2(cs, cs), mg2 = make_float2(8388608.0f, 8388608.0f);
                const float2 nmg2 = make_float2(-8388608.0f, -8388608.0f), m1 = make_float2(-1.0f, -1.0f);
#pragma unroll
                for (int ky = 0; ky < 2; ky++) {
                    const float tau_r = fmaf((float)(-4 * ky), sn, tau_t);
                    const float2 tr2 = make_float2(tau_r, tau_r);
#pragma unroll
                    for (int kx = 0; kx < 8; kx += 2) {
                        const float2 tau = __ffma2_rn(make_float2((float)(8 * kx), (float)(8 * kx + 8)), cs2, tr2);
                        const float2 m = __fadd2_rd(tau, mg2);   // 2^23 + floor(tau)
                        const float2 sv0 = lds64((__float_as_uint(m.x) << 3) + wb);
                        const float2 sv1 = lds64((__float_as_uint(m.y) << 3) + wb);
                        const float2 u = __ffma2_rn(__fadd2_rn(m, nmg2), m1, tau);  // tau - floor(tau)
                        // the two taps of a pixel accumulate into a packed (lower, upper) pair
                        acc2[ky][kx] = __ffma2_rn(make_float2(__saturatef(fmaf(-u.x, a1, a0)),
                                                              __saturatef(fmaf(u.x, a1, a0m))), sv0, acc2[ky][kx]);
                        acc2[ky][kx + 1] = __ffma2_rn(make_float2(__saturatef(fmaf(-u.y, a1, a0)),
                                                                  __saturatef(fmaf(u.y, a1, a0m))), sv1, acc2[ky][kx + 1]);
                    }
                }
            } else {
                const T *wk = win + k * BP_WB;
#pragma unroll
                for (int ky = 0; ky < 2; ky++) {
                    const T tau_r = fma((T)(-4 * ky), sn, tau_t);
#pragma unroll
                    for (int kx = 0; kx < 8; kx++) {
                        const T tau = fma((T)(8 * kx), cs, tau_r);
                        int i0;
                        const T fl = floor_split<T>(tau, i0);
                        const T u = tau - fl;
                        const T w0 = sat<T>(fma(-u, a1, a0));
                        const T w1 = sat<T>(fma(u, a1, a0m));
                        acc[ky][kx] = fma(w0, wk[i0], acc[ky][kx]);
                        acc[ky][kx] = fma(w1, wk[i0 + 1], acc[ky][kx]);
                    }
                }
            }
        }
    }
    if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int ky = 0; ky < 2; ky++)
#pragma unroll
            for (int kx = 0; kx < 8; kx++) acc[ky][kx] = acc2[ky][kx].x + acc2[ky][kx].y;
    }
    // ---------------- epilogue (fp64 in registers)
    if (pre) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
    }
    const double c = (EPI == EPI_CGQ || EPI == EPI_RESID || EPI == EPI_GD || EPI == EPI_CGR) ? a.cnode[node] : 0.0;
    const double alpha = EPI == EPI_CGR ? a.scal[(long long)node * S_NSLOT + S_ALPHA] : 0.0;  // launch_cg_alpha
    const float cf = (float)c;
    double dot = 0.0;
    float dotf = 0.f;
    const long long nb = (long long)node * a.n;
#pragma unroll
    for (int ky = 0; ky < 2; ky++)
#pragma unroll
        for (int kx = 0; kx < 8; kx++) {
            const int r = r0 + prow + 4 * ky, col = c0 + 8 * kx + lx;
            if (r >= N || col >= N) continue;
            const long long p = nb + (long long)r * N + col;
            const int sp = (prow + 4 * ky) * BP_TS + 8 * kx + lx;
            const double g = (double)acc[ky][kx];
            if (EPI == EPI_PLAIN) {
                a.out[p] = acc[ky][kx];
            } else if (EPI == EPI_CGQ) {
                if constexpr (sizeof(T) == 4) {  // fp32: one rounding (fmaf), per-thread fp32 partial of 16 products
                    const float pv = pre ? ep[sp] : (float)a.vin[p];
                    const float q = fmaf(cf, pv, acc[ky][kx]);
                    a.out[p] = q;
                    dotf = fmaf(pv, q, dotf);
                } else {
                    const double pv = (double)a.vin[p];
                    const T q = (T)(g + c * pv);
                    a.out[p] = q;
                    dot += pv * (double)q;
                }
            } else if (EPI == EPI_CGR) {  // q as in CGQ, then the CG residual update r -= alpha q
                T q;
                if constexpr (sizeof(T) == 4) {
                    const float pv = pre ? ep[sp] : (float)a.vin[p];
                    q = fmaf(cf, pv, acc[ky][kx]);
                } else {
                    q = (T)(g + c * (double)a.vin[p]);
                }
                const double rv = pre ? (double)ep[BP_TS * BP_TS + sp] : (double)a.bprime[p];
                const T rn = (T)(rv - alpha * (double)q);
                a.out[p] = rn;
                dot += (double)rn * (double)rn;
            } else if (EPI == EPI_RESID) {
                const double xv = pre ? (double)ep[sp] : (double)a.vin[p];
                const double bv = pre ? (double)ep[BP_TS * BP_TS + sp] : (double)a.bprime[p];
                const T rv = (T)(g + bv - c * xv);
                a.out[p] = rv;
                a.out2[p] = rv;
                dot += (double)rv * (double)rv;
            } else {  // EPI_GD: x <- x - eta (c x - b' - A^T(d - A x))
                const double xv = pre ? (double)ep[sp] : (double)a.vin[p];
                const double bv = pre ? (double)ep[BP_TS * BP_TS + sp] : (double)a.bprime[p];
                a.out[p] = (T)(xv - a.eta[node] * (c * xv - bv - g));
            }
        }
    if (EPI == EPI_CGQ || EPI == EPI_RESID || EPI == EPI_CGR) {
        const double bs = block_sum<BP_THREADS>(dot + (double)dotf, red);
        double *part = a.partial + (long long)node * a.part_stride;
        if (threadIdx.x == 0) part[blockIdx.x] = bs;
        if (last_block_of_group(a.counter + node, gridDim.x, &last_flag)) {
            double s = 0.0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += BP_THREADS) s += __ldcg(part + b);
            s = block_sum<BP_THREADS>(s, red);
            if (threadIdx.x == 0) {
                double *sc = a.scal + (long long)node * S_NSLOT;
                if (EPI == EPI_CGQ) {
                    sc[S_PQ] = s;
                    sc[S_ALPHA] = s > 0.0 ? sc[S_RR] / s : 0.0;
                } else if (EPI == EPI_CGR) {  // beta = rr_new / rr
                    const double rr = sc[S_RR];
                    sc[S_RRNEW] = s;
                    sc[S_BETA] = rr > 0.0 ? s / rr : 0.0;
                    sc[S_RR] = s;
                } else {  // RESID: r0 and p0 = r0
                    sc[S_RR] = s;
                    sc[S_PP] = s;
                }
            }
        }
    }
}

template <typename K>
void set_smem(K kernel, size_t dyn) {
    TQ_CHECK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
}

template <typename T>
size_t fp_smem(int o) { return sizeof(T) * FP_TH * (o == 0 ? FP_PITCH_Y : FP_PITCH_X); }
size_t fp2_smem() { return sizeof(float2) * FP_TH * FP2_PITCH; }
size_t fpp_smem() { return 1024 + sizeof(float2) * FP_TH * FP2_PITCH + sizeof(float) * FPP_RAW + sizeof(FpRec) * 2 * FPP_MAXA + 2 * sizeof(FpUnitTab); }
int g_fpp_grid = 0;  // persistent grid: SMs x resident CTAs (projector_setup)
int g_fpp_sms = 0, g_fpp_per = 0;
bool g_fpp_grid_set = false;  // TQ_FPP_GRID given: every launch uses it
template <typename T, int EPI>
size_t bp_smem() {
    constexpr int NEP = (EPI == EPI_CGQ) ? 1 : ((EPI == EPI_RESID || EPI == EPI_GD || EPI == EPI_CGR) ? 2 : 0);
    return sizeof(T) == 4 ? sizeof(float2) * bp_maxa<T, EPI>() * BP_WB + NEP * sizeof(float) * BP_TS * BP_TS
                          : sizeof(T) * BP_MAXA * BP_WB;
}

template <typename T>
void set_all_smem() {
    set_smem(fp_tile_kernel<T, 0>, fp_smem<T>(0));
    set_smem(fp_tile_kernel<T, 1>, fp_smem<T>(1));
    set_smem(fp_tile_kernel<T, 0, true>, fp_smem<T>(0));
    set_smem(fp_tile_kernel<T, 1, true>, fp_smem<T>(1));
    if (sizeof(T) == 4) {
        set_smem(fp_tile_f32<0>, fp2_smem());
        set_smem(fp_tile_f32<1>, fp2_smem());
        set_smem(fp_persist_f32<false>, fpp_smem());
        set_smem(fp_persist_f32<true>, fpp_smem());
        int dev = 0, sms = 0, per = 0;
        TQ_CHECK_CUDA(cudaGetDevice(&dev));
        TQ_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TQ_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fp_persist_f32<false>, FP_THREADS, fpp_smem()));
        g_fpp_grid = sms * std::max(1, per);
        g_fpp_sms = sms;
        g_fpp_per = std::max(1, per);
        if (const char *e = getenv("TQ_FPP_GRID"))  // A/B timing knob: persistent grid size
            if (atoi(e) > 0) { g_fpp_grid = atoi(e); g_fpp_grid_set = true; }
    }
    set_smem(bp_tile_kernel<T, EPI_PLAIN>, bp_smem<T, EPI_PLAIN>());
    set_smem(bp_tile_kernel<T, EPI_CGQ>, bp_smem<T, EPI_CGQ>());
    set_smem(bp_tile_kernel<T, EPI_RESID>, bp_smem<T, EPI_RESID>());
    set_smem(bp_tile_kernel<T, EPI_GD>, bp_smem<T, EPI_GD>());
    set_smem(bp_tile_kernel<T, EPI_CGR>, bp_smem<T, EPI_CGR>());
}

// TMA descriptors of the [L][N][N] fp32 images: a 128 x 32 (cols x rows) box for the
// y-major tiles and a 32 x 128 box with the 128-byte swizzle for the x-major tiles.
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        TQ_CHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) fail(TQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}
void make_image_maps(const float *img, int N, int L, CUtensorMap *rows, CUtensorMap *cols) {
    const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)L};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)N * N * 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint32_t box_r[3] = {FP_TW, FP_TH, 1}, box_c[3] = {FP_TH, FP_TW, 1};
    auto enc = encode_tiled();
    CUresult r1 = enc(rows, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)img, dims, strides, box_r, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(cols, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)img, dims, strides, box_c, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) fail(TQ_ECUDA, "cuTensorMapEncodeTiled failed");
}

template <typename T>
void fp_dispatch(const FpArgs<T> &A, int L, cudaStream_t st) {
    const dim3 grid(A.nt_line * A.nt_cross, L);
    const bool persist = sizeof(T) == 4 && A.N % 4 == 0 && A.recs && ((uintptr_t)A.img & 15) == 0;
    if (A.siddon && !persist) {  // Siddon (NEXT-3) outside the persistent fp32 kernel: the generic tile kernel
        FpArgs<T> S = A;
        S.magic = 0x4B000000u << 2;  // 4-byte entries
        fp_tile_kernel<T, 0, true><<<grid, FP_THREADS, fp_smem<T>(0), st>>>(S);
        fp_tile_kernel<T, 1, true><<<grid, FP_THREADS, fp_smem<T>(1), st>>>(S);
        return;
    }
    if constexpr (sizeof(T) == 4) {
        FpArgs<float> B = A;
        B.magic = 0x4B000000u << 3;  // 8-byte pairs (wraps mod 2^32)
        if (A.N % 4 == 0 && A.recs && ((uintptr_t)A.img & 15) == 0) {
            const int nunits = 2 * L * A.nt_line * A.nt_cross;
            CUtensorMap tr, tc;
            make_image_maps(A.img, A.N, L, &tr, &tc);
            // a node group's launch (L < L_all) shares the SMs with the other groups' concurrent
            // chains: SMs x ceil(2 x resident / groups) CTAs (A.L_all / L groups; measured best at
            // 2, 4 and 8 groups on C4_G1, DESIGN.md 6.1 "node groups")
            int grid = g_fpp_grid;
            if (L < A.L_all && g_fpp_per > 0 && !g_fpp_grid_set) {
                const int groups = std::max(1, (A.L_all + L - 1) / L);
                grid = g_fpp_sms * std::max(1, (2 * g_fpp_per + groups - 1) / groups);
            }
            grid = std::min(nunits, grid);
            if (A.siddon) launch_pdl(fp_persist_f32<true>, grid, FP_THREADS, fpp_smem(), st, B, nunits, tr, tc);
            else launch_pdl(fp_persist_f32<false>, grid, FP_THREADS, fpp_smem(), st, B, nunits, tr, tc);
        } else {
            fp_tile_f32<0><<<grid, FP_THREADS, fp2_smem(), st>>>(B);
            fp_tile_f32<1><<<grid, FP_THREADS, fp2_smem(), st>>>(B);
        }
    } else {
        fp_tile_kernel<T, 0><<<grid, FP_THREADS, fp_smem<T>(0), st>>>(A);
        fp_tile_kernel<T, 1><<<grid, FP_THREADS, fp_smem<T>(1), st>>>(A);
    }
}

template <typename T>
void bp_dispatch(int epi, const BpArgs<T> &A0, dim3 grid, cudaStream_t st) {
    BpArgs<T> A = A0;
    A.magic = 0x4B000000u << 3;  // fp32 pair windows (wraps mod 2^32)
    switch (epi) {
        case EPI_PLAIN: launch_pdl(bp_tile_kernel<T, EPI_PLAIN>, grid, BP_THREADS, bp_smem<T, EPI_PLAIN>(), st, A); break;
        case EPI_CGQ: launch_pdl(bp_tile_kernel<T, EPI_CGQ>, grid, BP_THREADS, bp_smem<T, EPI_CGQ>(), st, A); break;
        case EPI_RESID: launch_pdl(bp_tile_kernel<T, EPI_RESID>, grid, BP_THREADS, bp_smem<T, EPI_RESID>(), st, A); break;
        case EPI_CGR: launch_pdl(bp_tile_kernel<T, EPI_CGR>, grid, BP_THREADS, bp_smem<T, EPI_CGR>(), st, A); break;
        default: launch_pdl(bp_tile_kernel<T, EPI_GD>, grid, BP_THREADS, bp_smem<T, EPI_GD>(), st, A); break;
    }
}

}  // namespace

// Dynamic shared-memory limits of the projector kernels on the current device; called
// outside stream capture (Inner::init) because cudaFuncSetAttribute is not capturable.
void projector_setup() {
    set_all_smem<float>();
    set_all_smem<double>();
}

int fp_ntiles(int N) { return ceil_div(N, FP_TH) * ceil_div(N, FP_TW); }

int bp_tiles(int N) {
    const int t = ceil_div(N, BP_TS);
    return t * t;
}

void launch_fp(int prec, const void *args, int L, cudaStream_t st) {
    if (L == 0) return;
    if (prec == 0) fp_dispatch<float>(*static_cast<const FpArgs<float> *>(args), L, st);
    else fp_dispatch<double>(*static_cast<const FpArgs<double> *>(args), L, st);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_fp_setup(const RayRow *rows, const int *xmaj, const double2 *trig, int n_rows, int N, int n_det,
                     FpWin *wins, FpRowGeo *rgeo, const int *olist, int n_olist, FpRec *recs, const int *oofs, int L,
                     FpUnitTab *utab, cudaStream_t st) {
    if (n_rows == 0) return;
    const int ntiles = fp_ntiles(N);
    fp_setup_kernel<<<dim3(ceil_div(ntiles, 128), n_rows), 128, 0, st>>>(rows, xmaj, trig, n_rows, N, n_det, wins, rgeo);
    TQ_CHECK_CUDA(cudaGetLastError());
    if (n_olist) {
        fp_rec_kernel<<<dim3(ceil_div(ntiles, 128), n_olist), 128, 0, st>>>(olist, n_olist, ntiles, wins, rgeo, recs);
        TQ_CHECK_CUDA(cudaGetLastError());
        fp_unit_kernel<<<2 * L * ntiles, 64, 0, st>>>(oofs, recs, n_olist, ntiles, L, utab);
        TQ_CHECK_CUDA(cudaGetLastError());
    }
}

int fp_reduce_blocks(int prec, int n_det) { return prec == 0 ? ceil_div(n_det, 4 * RQ) : ceil_div(n_det, RJ); }

void launch_fp_reduce(int prec, bool resid, const void *args, int n_rows, int n_det, cudaStream_t st) {
    if (n_rows == 0) return;
    const dim3 grid(ceil_div(n_det, RJ), n_rows);
    if (prec == 0) {
        const auto &A = *static_cast<const FpRedArgs<float> *>(args);
        const dim3 gq(ceil_div(n_det, 4 * RQ), n_rows);
        if (resid) launch_pdl(fp_reduce_f32<true>, gq, RQ * RG, 0, st, A);
        else launch_pdl(fp_reduce_f32<false>, gq, RQ * RG, 0, st, A);
    } else {
        const auto &A = *static_cast<const FpRedArgs<double> *>(args);
        if (resid) fp_reduce_kernel<double, true><<<grid, RJ * RG, 0, st>>>(A);
        else fp_reduce_kernel<double, false><<<grid, RJ * RG, 0, st>>>(A);
    }
    TQ_CHECK_CUDA(cudaGetLastError());
}

__global__ void bp_rowc_kernel(const RayRow *rows, const double2 *trig, const int *xmaj, int n_rows,
                               double4 *rowc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    const int ang = rows[r].angle;
    const double cs = trig[ang].x, sn = trig[ang].y;
    const double m = xmaj[ang] ? fabs(sn) : fabs(cs);
    const double w = xmaj[ang] ? fabs(cs / sn) : fabs(sn / cs);
    rowc[r] = make_double4(cs, sn, m, w > 1e-9 ? 1.0 / w : 4194304.0);
}

void launch_bp_rowc(const RayRow *rows, const double2 *trig, const int *xmaj, int n_rows, double4 *rowc,
                    cudaStream_t st) {
    if (n_rows == 0) return;
    bp_rowc_kernel<<<ceil_div(n_rows, 128), 128, 0, st>>>(rows, trig, xmaj, n_rows, rowc);
    TQ_CHECK_CUDA(cudaGetLastError());
}

void launch_bp(int prec, int epi, const void *args, int L, int N, cudaStream_t st) {
    if (L == 0) return;
    const dim3 grid(bp_tiles(N), L);
    if (prec == 0) bp_dispatch<float>(epi, *static_cast<const BpArgs<float> *>(args), grid, st);
    else bp_dispatch<double>(epi, *static_cast<const BpArgs<double> *>(args), grid, st);
    TQ_CHECK_CUDA(cudaGetLastError());
}

}  // namespace tq
