// kmeans.cu -- K-means quantizer (Alg. 5), exact rules DESIGN.md R-16.
#include "codecs.cuh"

namespace tq {

namespace {

constexpr int KT = 256;
constexpr int SMEM_HIST_MAX_ROWS = 64;  // np*256 u32 histogram rows kept in shared memory

__device__ __forceinline__ uint32_t f2key(float f) {
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
    float *cen, *thr;
    uint32_t *prefix, *rank, *plist, *hist;
    int *np, *fexp;
    unsigned long long *acc_sum, *acc_cnt;
    unsigned *counter;
    int K, NT;
    long long nv;
};

KmPtr ptrs(const KmeansWork &w) {
    return KmPtr{w.cen, w.thr, w.prefix, w.rank, w.plist, w.hist, w.np, w.fexp, w.acc_sum,
                 w.acc_cnt, w.counter, w.K, w.K + 2, w.nv};
}

// targets: t = 0 -> rank 0 (min), t = 1..K -> floor((2k+1) nv / 2K), t = K+1 -> nv-1 (max)
__global__ void km_init(KmPtr w) {
    const int b = blockIdx.x;
    const int NT = w.NT;
    for (int t = threadIdx.x; t < NT; t += blockDim.x) {
        unsigned long long r;
        if (t == 0) r = 0;
        else if (t == NT - 1) r = (unsigned long long)(w.nv - 1);
        else r = ((unsigned long long)(2 * (t - 1) + 1) * (unsigned long long)w.nv) /
                 (unsigned long long)(2 * w.K);
        w.rank[(long long)b * NT + t] = (uint32_t)r;
        w.prefix[(long long)b * NT + t] = 0u;
    }
    if (threadIdx.x == 0) {
        w.np[b] = 1;
        w.plist[(long long)b * NT] = 0u;
    }
}

template <bool SMEM>
__global__ void __launch_bounds__(KT) km_hist(const float *const *vin, KmPtr w, int shift) {
    extern __shared__ uint32_t sh[];
    const int b = blockIdx.y;
    const int np = w.np[b];
    const uint32_t *plist = w.plist + (long long)b * w.NT;
    uint32_t *gh = w.hist + (long long)b * w.NT * 256;
    if (SMEM) {
        for (int i = threadIdx.x; i < np * 256; i += KT) sh[i] = 0u;
        __syncthreads();
    }
    const float *vb = vin[b];
    for (long long i = (long long)blockIdx.x * KT + threadIdx.x; i < w.nv; i += (long long)gridDim.x * KT) {
        const uint32_t k = f2key(vb[i]);
        const uint32_t pf = (uint32_t)((unsigned long long)k >> (shift + 8));
        int lo = 0, hi = np;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (plist[mid] < pf) lo = mid + 1; else hi = mid;
        }
        if (lo < np && plist[lo] == pf) {
            const int d = (k >> shift) & 255;
            if (SMEM) atomicAdd(&sh[lo * 256 + d], 1u);
            else atomicAdd(&gh[lo * 256 + d], 1u);
        }
    }
    if (SMEM) {
        __syncthreads();
        for (int i = threadIdx.x; i < np * 256; i += KT)
            if (sh[i]) atomicAdd(&gh[i], sh[i]);
    }
}

__global__ void __launch_bounds__(KT) km_select(KmPtr w, int shift) {
    const int b = blockIdx.x;
    const int NT = w.NT;
    __shared__ int np_s;
    if (threadIdx.x == 0) np_s = w.np[b];
    __syncthreads();
    const int np = np_s;
    uint32_t *plist = w.plist + (long long)b * NT;
    uint32_t *prefix = w.prefix + (long long)b * NT;
    uint32_t *rank = w.rank + (long long)b * NT;
    uint32_t *hist = w.hist + (long long)b * NT * 256;
    for (int t = threadIdx.x; t < NT; t += KT) {
        const uint32_t pf = prefix[t];
        int lo = 0, hi = np;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (plist[mid] < pf) lo = mid + 1; else hi = mid;
        }
        const uint32_t *H = hist + (long long)lo * 256;
        uint32_t r = rank[t], cum = 0;
        int d = 255;
        for (int q = 0; q < 256; q++) {
            const uint32_t c = H[q];
            if (r < cum + c) { d = q; break; }
            cum += c;
        }
        rank[t] = r - cum;
        prefix[t] = (shift == 24) ? (uint32_t)d : ((pf << 8) | (uint32_t)d);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * 256; i += KT) hist[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = 0;
        for (int t = 0; t < NT; t++)
            if (t == 0 || prefix[t] != prefix[t - 1]) plist[m++] = prefix[t];
        w.np[b] = m;
        if (shift == 0) {
            // order statistics found: centres, and the fixed-point exponent F such that
            // |sum of nv values * 2^F| < 2^62 (deterministic integer cluster sums)
            const int K = w.K;
            float *cen = w.cen + (long long)b * K;
            for (int k = 0; k < K; k++) cen[k] = key2f(prefix[1 + k]);
            const double mx = fmax(fabs((double)key2f(prefix[0])), fabs((double)key2f(prefix[NT - 1])));
            int F = 0;
            if (mx > 0.0) {
                const int E = ilogb(mx) + 1;
                int lg = 0;
                while ((1LL << lg) < w.nv) lg++;
                F = 62 - E - lg;
            }
            w.fexp[b] = F;
            float *thr = w.thr + (long long)b * K;
            for (int k = 0; k + 1 < K; k++) thr[k] = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
        }
    }
}

__global__ void __launch_bounds__(KT) km_lloyd(const float *const *vin, KmPtr w) {
    extern __shared__ unsigned long long shl[];  // sum[K] then cnt[K]
    __shared__ float thr_s[256];
    __shared__ bool last;
    const int b = blockIdx.y;
    const int K = w.K;
    unsigned long long *s_sum = shl, *s_cnt = shl + K;
    for (int k = threadIdx.x; k < K; k += KT) {
        s_sum[k] = 0ull;
        s_cnt[k] = 0ull;
        if (k + 1 < K) thr_s[k] = w.thr[(long long)b * K + k];
    }
    __syncthreads();
    const double scale = ldexp(1.0, w.fexp[b]);
    const float *vb = vin[b];
    for (long long i0 = ((long long)blockIdx.x * KT + threadIdx.x) * 4; i0 < w.nv;
         i0 += (long long)gridDim.x * KT * 4) {
        int cur = -1;
        long long csum = 0;
        unsigned long long ccnt = 0;
        for (int e = 0; e < 4; e++) {
            const long long i = i0 + e;
            if (i >= w.nv) break;
            const float x = vb[i];
            const int l = kmeans_label(x, thr_s, K);
            const long long fx = __double2ll_rn((double)x * scale);
            if (l != cur) {
                if (cur >= 0) {
                    atomicAdd(&s_sum[cur], (unsigned long long)csum);
                    atomicAdd(&s_cnt[cur], ccnt);
                }
                cur = l; csum = 0; ccnt = 0;
            }
            csum += fx;
            ccnt += 1;
        }
        if (cur >= 0) {
            atomicAdd(&s_sum[cur], (unsigned long long)csum);
            atomicAdd(&s_cnt[cur], ccnt);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += KT) {
        if (s_cnt[k]) {
            atomicAdd(&w.acc_sum[(long long)b * K + k], s_sum[k]);
            atomicAdd(&w.acc_cnt[(long long)b * K + k], s_cnt[k]);
        }
    }
    if (last_block_of_group(w.counter + b, gridDim.x, &last)) {
        float *cen = w.cen + (long long)b * K;
        for (int k = threadIdx.x; k < K; k += KT) {
            const unsigned long long c = w.acc_cnt[(long long)b * K + k];
            const long long s = (long long)w.acc_sum[(long long)b * K + k];
            if (c) cen[k] = (float)(((double)s / scale) / (double)c);
            w.acc_cnt[(long long)b * K + k] = 0ull;
            w.acc_sum[(long long)b * K + k] = 0ull;
        }
        __syncthreads();
        float *thr = w.thr + (long long)b * K;
        for (int k = threadIdx.x; k + 1 < K; k += KT)
            thr[k] = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
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

int grid_for(long long nv, int P) {
    // enough blocks to fill 148 SMs a few times over all payloads
    long long want = std::max(1LL, (148LL * 8 + P - 1) / P);
    long long need = (nv + KT * 4 - 1) / (KT * 4);
    return (int)std::max(1LL, std::min(want, need));
}

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
    const int NT = K + 2;
    TQ_REQUIRE(K >= 1 && K <= 256, "kmeans: k must be in [1, 256]");
    TQ_CHECK_CUDA(cudaFuncSetAttribute(km_hist<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_HIST_MAX_ROWS * 256 * 4));
    TQ_CHECK_CUDA(cudaMalloc(&cen, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&thr, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&prefix, sizeof(uint32_t) * P * NT));
    TQ_CHECK_CUDA(cudaMalloc(&rank, sizeof(uint32_t) * P * NT));
    TQ_CHECK_CUDA(cudaMalloc(&plist, sizeof(uint32_t) * P * NT));
    TQ_CHECK_CUDA(cudaMalloc(&np, sizeof(int) * P));
    TQ_CHECK_CUDA(cudaMalloc(&hist, sizeof(uint32_t) * P * NT * 256));
    TQ_CHECK_CUDA(cudaMemset(hist, 0, sizeof(uint32_t) * P * NT * 256));
    TQ_CHECK_CUDA(cudaMalloc(&fexp, sizeof(int) * P));
    TQ_CHECK_CUDA(cudaMalloc(&acc_sum, sizeof(unsigned long long) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&acc_cnt, sizeof(unsigned long long) * P * K));
    TQ_CHECK_CUDA(cudaMemset(acc_sum, 0, sizeof(unsigned long long) * P * K));
    TQ_CHECK_CUDA(cudaMemset(acc_cnt, 0, sizeof(unsigned long long) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&counter, sizeof(unsigned) * P));
    TQ_CHECK_CUDA(cudaMemset(counter, 0, sizeof(unsigned) * P));
}

void KmeansWork::release() {
    for (void *p : {(void *)cen, (void *)thr, (void *)prefix, (void *)rank, (void *)plist, (void *)np,
                    (void *)hist, (void *)fexp, (void *)acc_sum, (void *)acc_cnt, (void *)counter})
        if (p) cudaFree(p);
    *this = KmeansWork();
}

int kmeans_encode(const float *const *v, KmeansWork &ws, int lloyd, uint8_t *const *pay,
                  int32_t *const *labels, cudaStream_t st) {
    const KmPtr w = ptrs(ws);
    const int P = ws.P;
    if (P == 0) return 0;
    TQ_REQUIRE(ws.nv >= 1 && ws.nv < (1LL << 31), "kmeans: payload length must be in [1, 2^31)");
    km_init<<<P, 64, 0, st>>>(w);
    const dim3 grid(grid_for(ws.nv, P), P);
    const bool smem = w.NT <= SMEM_HIST_MAX_ROWS;
    const size_t hsm = smem ? (size_t)w.NT * 256 * 4 : 0;  // opt-in set in KmeansWork::alloc
    for (int shift = 24; shift >= 0; shift -= 8) {
        if (smem) km_hist<true><<<grid, KT, hsm, st>>>(v, w, shift);
        else km_hist<false><<<grid, KT, 0, st>>>(v, w, shift);
        km_select<<<P, KT, 0, st>>>(w, shift);
    }
    const size_t lsm = sizeof(unsigned long long) * 2 * ws.K;
    for (int it = 0; it < lloyd; it++) km_lloyd<<<grid, KT, lsm, st>>>(v, w);
    km_final<<<grid, KT, 0, st>>>(v, w, ws.B, pay, labels);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1 + 8 + lloyd + 1;
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
