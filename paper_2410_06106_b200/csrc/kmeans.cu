// kmeans.cu -- K-means quantizer (Alg. 5), exact rules DESIGN.md R-16.
//
// Sort-based exact Lloyd.  Each payload's values are mapped to order-preserving
// 32-bit keys and sorted by an LSD radix sort (4 passes of 8-bit digits: per-tile
// digit histograms, per-payload offset scan, stable tile sort + scatter).  On the
// sorted keys:
//   * the quantile init c_k = v_(floor((2k+1) n / 2K)) is a direct read (exact order
//     statistic);
//   * a Lloyd step needs, for each threshold b_k, C_k = #{v <= b_k} and
//     S_k = sum_{v <= b_k} fix(v): C_k is an upper bound in the sorted keys (binary
//     search over the tile heads in shared memory, then one warp counts inside one
//     2048-key tile), S_k = (exclusive prefix of the tile sums) + the in-tile part.
//     Cluster k = (b_{k-1}, b_k], i.e. label(v) = #{k : v > b_k}, ties to the lower
//     cluster -- the same decision the oracle takes per element.
// fix(v) = round(v 2^F) as int64 with F chosen from max|v| and n so no sum overflows:
// cluster sums are exact integers, hence independent of summation order.
// All Lloyd iterations of a payload run in one CTA; the cost of an iteration no
// longer depends on n.  The final assignment packs labels into bit-planes.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "codecs.cuh"

namespace tq {

namespace {

constexpr int KT = 256;               // threads of the per-tile kernels
constexpr int KI = 8;                 // keys per thread
constexpr int KTILE = KT * KI;        // keys per tile
constexpr int LT = 1024;              // threads of the Lloyd kernel
constexpr int MAX_TILES = 8192;       // per payload (n <= 16.7 M)

__device__ __forceinline__ uint32_t f2key(float f) {
    if (f == 0.0f) f = 0.0f;  // -0 and +0 are the same value for every comparison
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// label(v) = #{k < K-1 : v > thr[k]} for non-decreasing thr (ties go to the lower cluster)
__device__ __forceinline__ int kmeans_label(float v, const float *thr, int K) {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v > thr[mid]) lo = mid + 1; else hi = mid;
    }
    return lo;
}

struct KmPtr {
    uint32_t *keysA, *keysB, *hist, *base;
    long long *tsum;
    float *cen, *thr;
    int *fexp;
    int K, T;
    long long nv;
};

KmPtr ptrs(const KmeansWork &w) {
    return KmPtr{w.keysA, w.keysB, w.hist, w.base, w.tsum, w.cen, w.thr, w.fexp, w.K, w.T, w.nv};
}

__device__ __forceinline__ void load_tile(const uint32_t *keys, long long off, uint32_t (&k)[KI]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(keys + off + threadIdx.x * KI);
    const uint4 a = p[0], b = p[1];
    k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w;
    k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
}

// warp-aggregated shared histogram of one digit of the thread's keys
__device__ __forceinline__ void tile_hist(const uint32_t (&k)[KI], int shift, uint32_t *sh) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < KI; r++) {
        const uint32_t d = (k[r] >> shift) & 255u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (lane == __ffs(peers) - 1) atomicAdd(&sh[d], (uint32_t)__popc(peers));
    }
}

__device__ __forceinline__ void flush_hist(uint32_t *sh, uint32_t *g) {
    __syncthreads();
    g[threadIdx.x] = sh[threadIdx.x];  // KT == 256 digits
}

// keys of the raw payload (padding keys sort last) + digit-0 histogram
__global__ void __launch_bounds__(KT) km_keys(const float *const *vin, KmPtr w) {
    __shared__ uint32_t sh[256];
    const int b = blockIdx.y, t = blockIdx.x;
    sh[threadIdx.x] = 0u;
    __syncthreads();
    const float *v = vin[b];
    const long long i0 = (long long)t * KTILE + threadIdx.x * KI;
    uint32_t k[KI];
#pragma unroll
    for (int r = 0; r < KI; r++) k[r] = (i0 + r < w.nv) ? f2key(v[i0 + r]) : 0xffffffffu;
    uint4 *o = reinterpret_cast<uint4 *>(w.keysA + (long long)b * w.T * KTILE + i0);
    o[0] = make_uint4(k[0], k[1], k[2], k[3]);
    o[1] = make_uint4(k[4], k[5], k[6], k[7]);
    tile_hist(k, 0, sh);
    flush_hist(sh, w.hist + ((long long)b * w.T + t) * 256);
}

__global__ void __launch_bounds__(KT) km_hist(const uint32_t *keys, KmPtr w, int shift) {
    __shared__ uint32_t sh[256];
    const int b = blockIdx.y, t = blockIdx.x;
    sh[threadIdx.x] = 0u;
    __syncthreads();
    uint32_t k[KI];
    load_tile(keys, ((long long)b * w.T + t) * KTILE, k);
    tile_hist(k, shift, sh);
    flush_hist(sh, w.hist + ((long long)b * w.T + t) * 256);
}

// per payload: hist[t][d] <- sum_{t' < t} hist[t'][d]; base[d] <- sum_{d' < d} total[d']
__global__ void __launch_bounds__(256) km_scan(KmPtr w) {
    using Scan = cub::BlockScan<uint32_t, 256>;
    __shared__ typename Scan::TempStorage tmp;
    const int b = blockIdx.x, d = threadIdx.x;
    uint32_t *h = w.hist + (long long)b * w.T * 256 + d;
    uint32_t run = 0;
    int t = 0;
    for (; t + 4 <= w.T; t += 4) {
        const uint32_t c0 = h[(t + 0) * 256], c1 = h[(t + 1) * 256], c2 = h[(t + 2) * 256], c3 = h[(t + 3) * 256];
        h[(t + 0) * 256] = run; run += c0;
        h[(t + 1) * 256] = run; run += c1;
        h[(t + 2) * 256] = run; run += c2;
        h[(t + 3) * 256] = run; run += c3;
    }
    for (; t < w.T; t++) {
        const uint32_t c = h[t * 256];
        h[t * 256] = run;
        run += c;
    }
    uint32_t excl;
    Scan(tmp).ExclusiveSum(run, excl);
    w.base[(long long)b * 256 + d] = excl;
}

// stable sort of the tile by the digit, then scatter to base[d] + tile offset + rank
__global__ void __launch_bounds__(KT) km_scatter(const uint32_t *kin, uint32_t *kout, KmPtr w, int shift) {
    using Sort = cub::BlockRadixSort<uint32_t, KT, KI>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ uint32_t dstart[256], goff[256], lastd[KT];
    const int b = blockIdx.y, t = blockIdx.x;
    const long long pb = (long long)b * w.T * KTILE;
    uint32_t k[KI];
    load_tile(kin, pb + (long long)t * KTILE, k);
    goff[threadIdx.x] = w.base[(long long)b * 256 + threadIdx.x] +
                        w.hist[((long long)b * w.T + t) * 256 + threadIdx.x];
    Sort(tmp).Sort(k, shift, shift + 8);  // blocked arrangement, stable
    lastd[threadIdx.x] = (k[KI - 1] >> shift) & 255u;
    __syncthreads();
    uint32_t prev = threadIdx.x ? lastd[threadIdx.x - 1] : 0xffffffffu;
#pragma unroll
    for (int r = 0; r < KI; r++) {
        const uint32_t d = (k[r] >> shift) & 255u;
        if (d != prev) dstart[d] = threadIdx.x * KI + r;
        prev = d;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KI; r++) {
        const uint32_t d = (k[r] >> shift) & 255u;
        kout[pb + goff[d] + (threadIdx.x * KI + r - dstart[d])] = k[r];
    }
}

// fixed-point exponent F: |sum of nv values * 2^F| < 2^62
__device__ __forceinline__ int fixed_exp(const uint32_t *sorted, long long nv) {
    const double mx = fmax(fabs((double)key2f(sorted[0])), fabs((double)key2f(sorted[nv - 1])));
    if (!(mx > 0.0)) return 0;
    const int E = ilogb(mx) + 1;
    int lg = 0;
    while ((1LL << lg) < nv) lg++;
    return 62 - E - lg;
}

// per-tile sums of fix(v) over the sorted keys
__global__ void __launch_bounds__(KT) km_tsum(KmPtr w) {
    using Red = cub::BlockReduce<long long, KT>;
    __shared__ typename Red::TempStorage tmp;
    const int b = blockIdx.y, t = blockIdx.x;
    const uint32_t *sorted = w.keysA + (long long)b * w.T * KTILE;
    const int F = fixed_exp(sorted, w.nv);
    const double scale = ldexp(1.0, F);
    uint32_t k[KI];
    load_tile(sorted, (long long)t * KTILE, k);
    long long s = 0;
    const long long i0 = (long long)t * KTILE + threadIdx.x * KI;
#pragma unroll
    for (int r = 0; r < KI; r++)
        if (i0 + r < w.nv) s += __double2ll_rn((double)key2f(k[r]) * scale);
    const long long tot = Red(tmp).Sum(s);
    if (threadIdx.x == 0) {
        w.tsum[(long long)b * w.T + t] = tot;
        if (t == 0) w.fexp[b] = F;
    }
}

// one CTA per payload: quantile init, then `iters` exact Lloyd steps on the sorted keys
__global__ void __launch_bounds__(LT) km_lloyd(KmPtr w, int iters) {
    using Scan = cub::BlockScan<long long, LT>;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ __align__(16) unsigned char lsm[];
    long long *tpre = reinterpret_cast<long long *>(lsm);         // [T + 1]
    uint32_t *thead = reinterpret_cast<uint32_t *>(tpre + w.T + 1);  // [T]
    __shared__ float cen[256], thr[256];
    __shared__ long long Cs[256], Ss[256];
    const int b = blockIdx.x, K = w.K, T = w.T;
    const long long nv = w.nv;
    const uint32_t *sorted = w.keysA + (long long)b * T * KTILE;
    const long long *ts = w.tsum + (long long)b * T;
    const int F = w.fexp[b];
    const double scale = ldexp(1.0, F);
    // exclusive prefix of the tile sums (chunked block scan) and the tile head keys
    long long carry = 0;
    for (int c0 = 0; c0 < T; c0 += LT) {
        const int t = c0 + threadIdx.x;
        const long long x = t < T ? ts[t] : 0;
        long long ex, agg;
        Scan(tmp).ExclusiveSum(x, ex, agg);
        if (t < T) {
            tpre[t] = carry + ex;
            thead[t] = sorted[(long long)t * KTILE];
        }
        carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) tpre[T] = carry;
    // quantile init: c_k = v_(floor((2k+1) nv / 2K))
    for (int k = threadIdx.x; k < K; k += LT) {
        const long long idx = ((long long)(2 * k + 1) * nv) / (2LL * K);
        cen[k] = key2f(sorted[idx]);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = 0; it < iters; it++) {
        for (int k = threadIdx.x; k + 1 < K; k += LT) thr[k] = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
        __syncthreads();
        for (int k = warp; k + 1 < K; k += LT / 32) {
            const uint32_t kb = f2key(thr[k]);
            int lo = 0, hi = T - 1, tt = -1;  // last tile whose head key <= kb
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                if (thead[mid] <= kb) { tt = mid; lo = mid + 1; } else hi = mid - 1;
            }
            long long C = 0, S = 0;
            if (tt >= 0) {
                const long long off = (long long)tt * KTILE;
                int cnt = 0;
                long long s = 0;
                const uint4 *p = reinterpret_cast<const uint4 *>(sorted + off);
#pragma unroll 4
                for (int q = lane; q < KTILE / 4; q += 32) {
                    const uint4 v4 = p[q];
                    const uint32_t e[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const long long i = off + 4 * q + u;
                        if (e[u] <= kb && i < nv) {
                            cnt++;
                            s += __double2ll_rn((double)key2f(e[u]) * scale);
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                    s += __shfl_xor_sync(0xffffffffu, s, o);
                }
                C = off + cnt;
                S = tpre[tt] + s;
            }
            if (lane == 0) { Cs[k] = C; Ss[k] = S; }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < K; k += LT) {
            const long long c1 = k + 1 < K ? Cs[k] : nv, c0 = k ? Cs[k - 1] : 0;
            const long long s1 = k + 1 < K ? Ss[k] : tpre[T], s0 = k ? Ss[k - 1] : 0;
            if (c1 > c0) cen[k] = (float)(((double)(s1 - s0) / scale) / (double)(c1 - c0));
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < K; k += LT) {
        w.cen[(long long)b * K + k] = cen[k];
        if (k + 1 < K) w.thr[(long long)b * K + k] = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
    }
}

__global__ void __launch_bounds__(KT) km_final(const float *const *vin, KmPtr w, int B,
                                               uint8_t *const *pay, int32_t *const *labels_tab) {
    __shared__ float thr_s[256];
    const int b = blockIdx.y;
    const int K = w.K;
    for (int k = threadIdx.x; k + 1 < K; k += KT) thr_s[k] = w.thr[(long long)b * K + k];
    float *cen_out = reinterpret_cast<float *>(pay[b]);
    uint32_t *planes = reinterpret_cast<uint32_t *>(pay[b] + 4 * (long long)K);
    int32_t *labels = labels_tab ? labels_tab[b] : nullptr;
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < K; k += KT) cen_out[k] = w.cen[(long long)b * K + k];
    __syncthreads();
    const float *vb = vin[b];
    const long long G = (w.nv + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long warp0 = ((long long)blockIdx.x * KT + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * KT) >> 5;
    for (long long g = warp0; g < G; g += nwarps) {
        const long long i = g * 32 + lane;
        int l = 0;
        if (i < w.nv) {
            l = kmeans_label(vb[i], thr_s, K);
            if (labels) labels[i] = l;
        }
        for (int bit = 0; bit < B; bit++) {
            const unsigned word = __ballot_sync(0xffffffffu, (l >> bit) & 1);
            if (lane == 0) planes[g * B + bit] = word;
        }
    }
}

template <typename T>
__global__ void km_decode(const uint8_t *const *pay, long long nv, int K, int B, T *const *outp) {
    const int b = blockIdx.y;
    const float *c = reinterpret_cast<const float *>(pay[b]);
    const uint32_t *pl = reinterpret_cast<const uint32_t *>(pay[b] + 4 * (long long)K);
    T *out = outp[b];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv;
         i += (long long)gridDim.x * blockDim.x) {
        const long long g = i >> 5;
        const int lane = (int)(i & 31);
        int l = 0;
        for (int bit = 0; bit < B; bit++) l |= (int)((__ldg(pl + g * B + bit) >> lane) & 1u) << bit;
        out[i] = (T)c[l];
    }
}

size_t lloyd_smem(int T) { return sizeof(long long) * (T + 1) + sizeof(uint32_t) * T; }

}  // namespace

int kmeans_bits(int K) {
    int B = 0;
    while ((1 << B) < K) B++;
    return B;
}

long long kmeans_payload_bytes(int K, long long nv) {
    return 4LL * K + 4LL * ((nv + 31) / 32) * kmeans_bits(K);
}

void KmeansWork::alloc(int P_, int K_, long long nv_) {
    P = P_; K = K_; nv = nv_; B = kmeans_bits(K_);
    TQ_REQUIRE(K >= 1 && K <= 256, "kmeans: k must be in [1, 256]");
    TQ_REQUIRE(nv >= 1 && nv <= (long long)MAX_TILES * KTILE, "kmeans: payload length must be in [1, 16777216]");
    T = (int)((nv + KTILE - 1) / KTILE);
    const size_t nk = (size_t)P * T * KTILE;
    TQ_CHECK_CUDA(cudaMalloc(&keysA, sizeof(uint32_t) * nk));
    TQ_CHECK_CUDA(cudaMalloc(&keysB, sizeof(uint32_t) * nk));
    TQ_CHECK_CUDA(cudaMalloc(&hist, sizeof(uint32_t) * (size_t)P * T * 256));
    TQ_CHECK_CUDA(cudaMalloc(&base, sizeof(uint32_t) * (size_t)P * 256));
    TQ_CHECK_CUDA(cudaMalloc(&tsum, sizeof(long long) * (size_t)P * T));
    TQ_CHECK_CUDA(cudaMalloc(&cen, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&thr, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&fexp, sizeof(int) * P));
    TQ_CHECK_CUDA(cudaFuncSetAttribute(km_lloyd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lloyd_smem(T)));
}

void KmeansWork::release() {
    for (void *p : {(void *)keysA, (void *)keysB, (void *)hist, (void *)base, (void *)tsum, (void *)cen,
                    (void *)thr, (void *)fexp})
        if (p) cudaFree(p);
    *this = KmeansWork();
}

int kmeans_encode(const float *const *v, KmeansWork &ws, int lloyd, uint8_t *const *pay,
                  int32_t *const *labels, cudaStream_t st) {
    const KmPtr w = ptrs(ws);
    const int P = ws.P;
    if (P == 0) return 0;
    const dim3 tiles(ws.T, P);
    km_keys<<<tiles, KT, 0, st>>>(v, w);
    int k = 1;
    uint32_t *src = ws.keysA, *dst = ws.keysB;
    for (int pass = 0; pass < 4; pass++) {
        if (pass) { km_hist<<<tiles, KT, 0, st>>>(src, w, 8 * pass); k++; }
        km_scan<<<P, 256, 0, st>>>(w);
        km_scatter<<<tiles, KT, 0, st>>>(src, dst, w, 8 * pass);
        k += 2;
        std::swap(src, dst);
    }
    // four passes: A -> B -> A -> B -> A, sorted keys in keysA
    km_tsum<<<tiles, KT, 0, st>>>(w);
    km_lloyd<<<P, LT, lloyd_smem(ws.T), st>>>(w, lloyd);
    long long want = std::max(1LL, (148LL * 8 + P - 1) / P);
    long long need = (ws.nv + KT * 4 - 1) / (KT * 4);
    const dim3 grid((unsigned)std::max(1LL, std::min(want, need)), P);
    km_final<<<grid, KT, 0, st>>>(v, w, ws.B, pay, labels);
    TQ_CHECK_CUDA(cudaGetLastError());
    return k + 3;
}

int kmeans_decode(const uint8_t *const *pay, int P, long long nv, int K, int prec,
                  void *const *out, cudaStream_t st) {
    if (P == 0) return 0;
    const int B = kmeans_bits(K);
    const dim3 grid((unsigned)std::min<long long>(1024, (nv + 255) / 256), P);
    if (prec == 0)
        km_decode<float><<<grid, 256, 0, st>>>(pay, nv, K, B, (float *const *)out);
    else
        km_decode<double><<<grid, 256, 0, st>>>(pay, nv, K, B, (double *const *)out);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace tq
