// kmeans.cu -- K-means quantizer (Alg. 5), exact rules DESIGN.md R-16.
//
// Sort-based exact Lloyd.  Each payload's values are mapped to order-preserving 32-bit
// keys and ordered by an LSD radix sort on the key bytes 1..3 (3 passes of 8-bit digits:
// per-tile digit histograms stored tile-major, one exclusive scan per payload over
// (digit, tile) = the global output offsets, stable ballot-multisplit tile ranking +
// scatter).  The keys end up ordered by their top 24 bits -- a "group" = one sign, exponent
// and top 15 mantissa bits, i.e. values within 2^-15 relative -- with the low byte unordered
// inside a group; the fourth pass is not needed because every query below resolves the one
// group it touches.  On the group-sorted keys:
//   * the quantile init c_k = v_(floor((2k+1) n / 2K)) is an exact order statistic: the
//     rank falls in the group of the key at that position; the keys of smaller groups are
//     counted and the group's low bytes histogrammed by one warp;
//   * a Lloyd step needs, for each threshold b_k, C_k = #{v <= b_k} and
//     S_k = sum_{v <= b_k} fix(v): the super-chunk heads (shared memory) bound the keys of
//     b_k's group to a few super-chunks, which one warp reads, counting and summing the keys
//     <= b_k; everything before them is below b_k (exclusive prefix of fix at their start).
//     Cluster k = (b_{k-1}, b_k], i.e. label(v) = #{k : v > b_k}, ties to the lower
//     cluster -- the same decision the oracle takes per element.
// fix(v) = round(v 2^F) as int64 with F chosen from max|v| and n so no sum overflows:
// cluster sums are exact integers, hence independent of summation order.
// All Lloyd iterations of a payload run in one thread-block cluster (8 CTAs exchanging
// (C_k, S_k) through distributed shared memory); the cost of an iteration does not
// depend on n.  The final assignment (bucket table) packs labels into bit-planes.
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "codecs.cuh"

namespace tq {

namespace {

constexpr int KT = 256;               // threads of the per-tile kernels
constexpr int KI = 16;                // keys per thread
constexpr int KTILE = KT * KI;        // keys per tile
constexpr int MAX_TILES = 4096;       // per payload (n <= 16.7 M)
constexpr int KCH = 128;              // keys per prefix-sum chunk
constexpr int CPT = KTILE / KCH;      // chunks per tile (32)
constexpr int LSC_MAX = 8192;         // super-chunks resident in the Lloyd kernel's shared memory (32 * 32 * 8)
static_assert(CPT == 32, "one warp lane per chunk head");

__device__ __forceinline__ uint32_t f2key(float f) {
    if (f == 0.0f) f = 0.0f;  // -0 and +0 are the same value for every comparison
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

struct KmPtr {
    uint32_t *keysA, *keysB, *hist, *dtot;
    long long *csum, *cpre;
    float *cen, *thr;
    int *fexp;
    int K, T;
    long long nv;
    int *lut;
    float *lutmap;
    uint32_t *heads;
};

KmPtr ptrs(const KmeansWork &w) {
    return KmPtr{w.keysA, w.keysB, w.hist, w.dtot, w.csum, w.cpre, w.cen, w.thr, w.fexp, w.K, w.T, w.nv,
                 w.lut, w.lutmap, w.heads};
}

// final-assignment bucket map (see km_final): 1024 buckets over [min, max] of the payload
constexpr int LUT_NB = 1024;
__device__ __forceinline__ int km_bucket(float v, float lo, float scale) {
    float t = __fmul_rn(__fsub_rn(v, lo), scale);
    t = fminf(fmaxf(t, 0.0f), (float)(LUT_NB - 1));
    return (int)t;
}

__device__ __forceinline__ void load_tile(const uint32_t *keys, long long off, uint32_t (&k)[KI]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(keys + off + threadIdx.x * KI);
#pragma unroll
    for (int q = 0; q < KI / 4; q++) {
        const uint4 a = p[q];
        k[4 * q] = a.x; k[4 * q + 1] = a.y; k[4 * q + 2] = a.z; k[4 * q + 3] = a.w;
    }
}

// Warp multisplit by ballots: peers = lanes of the warp whose digit equals mine
// (8 ballots, no match/atomics).  Keys of a tile are warp-striped: warp w, round r,
// lane l holds key w*256 + r*32 + l, so (w, r, l) is the tile's index order.
// Per bit: one predicate from the digit (R2P), one VOTE, and the lane keeps either the
// ballot or its complement (a predicated LOP3); the eight words meet in four 3-input ANDs.
__device__ __forceinline__ unsigned digit_ballot(uint32_t d, uint32_t bit) {
    unsigned bal;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
        "@!p not.b32 %0, %0;\n\t}"
        : "=r"(bal) : "r"(d), "r"(bit));
    return bal;
}
__device__ __forceinline__ unsigned and3(unsigned a, unsigned b, unsigned c) {
    unsigned r;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ unsigned digit_peers(uint32_t d) {
    // the eight (possibly complemented) ballots combined by three-input ANDs (4 LOP3)
    const unsigned b0 = digit_ballot(d, 1u), b1 = digit_ballot(d, 2u), b2 = digit_ballot(d, 4u),
                   b3 = digit_ballot(d, 8u), b4 = digit_ballot(d, 16u), b5 = digit_ballot(d, 32u),
                   b6 = digit_ballot(d, 64u), b7 = digit_ballot(d, 128u);
    return and3(and3(and3(b0, b1, b2), b3, b4), and3(b5, b6, b7), 0xffffffffu);
}

__device__ __forceinline__ void load_striped(const uint32_t *keys, long long off, uint32_t (&k)[KI]) {
    const uint32_t *p = keys + off + (threadIdx.x >> 5) * 32 * KI + (threadIdx.x & 31);
#pragma unroll
    for (int r = 0; r < KI; r++) k[r] = p[r * 32];
}

// tile histogram: per-warp private digit counters updated with shared-memory atomics
// (integer counts: the result does not depend on the order of the updates), then the
// column sums into sh[256]
__device__ __forceinline__ void tile_hist(const uint32_t (&k)[KI], int shift, uint32_t *wc /* [8][256] */,
                                          uint32_t *sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *c = wc + warp * 256;
    for (int i = lane; i < 256; i += 32) c[i] = 0u;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < KI; r++) atomicAdd(&c[(k[r] >> shift) & 255u], 1u);
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < KT / 32; w++) tot += wc[w * 256 + threadIdx.x];
    sh[threadIdx.x] = tot;
}

// tile-major [P][T][256] (coalesced rows); km_scan turns each digit column into the
// global output offsets of (digit, tile)
__device__ __forceinline__ void flush_hist(const uint32_t *sh, uint32_t *hp, int T, int t) {
    __syncthreads();
    hp[(long long)t * 256 + threadIdx.x] = sh[threadIdx.x];  // KT == 256 digits
}

// keys of the raw payload (padding keys sort last) + the histogram of the first sorted digit
// (bits 8..15: the low byte is never sorted, see kmeans_encode)
__global__ void __launch_bounds__(KT) km_keys(const float *const *vin, KmPtr w) {
    pdl_wait();
    __shared__ uint32_t sh[256], wc[KT / 32 * 256];
    const int b = blockIdx.y, t = blockIdx.x;
    const float *v = vin[b];
    const long long i0 = (long long)t * KTILE + (threadIdx.x >> 5) * 32 * KI + (threadIdx.x & 31);
    uint32_t k[KI];
#pragma unroll
    for (int r = 0; r < KI; r++) k[r] = (i0 + r * 32 < w.nv) ? f2key(v[i0 + r * 32]) : 0xffffffffu;
    uint32_t *o = w.keysB + (long long)b * w.T * KTILE + i0;
#pragma unroll
    for (int r = 0; r < KI; r++) o[r * 32] = k[r];
    tile_hist(k, 8, wc, sh);
    flush_hist(sh, w.hist + (long long)b * 256 * w.T, w.T, t);
}

__global__ void __launch_bounds__(KT) km_hist(const uint32_t *keys, KmPtr w, int shift) {
    pdl_wait();
    __shared__ uint32_t sh[256], wc[KT / 32 * 256];
    const int b = blockIdx.y, t = blockIdx.x;
    uint32_t k[KI];
    load_tile(keys, ((long long)b * w.T + t) * KTILE, k);  // order does not matter for counting
    tile_hist(k, shift, wc, sh);
    flush_hist(sh, w.hist + (long long)b * 256 * w.T, w.T, t);
}

// exclusive scan down each digit column of a payload's tile-major counts, in place; the
// column total goes to dtot[payload][digit].  One CTA per (payload, 32 digits): lane =
// digit (rows of 32 digits are 128-byte coalesced), warp w owns a contiguous range of
// tiles; warp totals are combined in a fixed order.
constexpr int SCW = 8;  // warps per CTA
__global__ void __launch_bounds__(SCW * 32) km_scan(KmPtr w) {
    pdl_wait();
    __shared__ uint32_t tot[SCW][32];
    const int b = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = blockIdx.x * 32 + lane;
    const int T = w.T, per = (T + SCW - 1) / SCW;
    const int t0 = warp * per, t1 = min(T, t0 + per);
    uint32_t *h = w.hist + (long long)b * T * 256 + d;
    uint32_t sum = 0;
    for (int t = t0; t < t1; t++) sum += h[(long long)t * 256];
    tot[warp][lane] = sum;
    __syncthreads();
    uint32_t run = 0, all = 0;
#pragma unroll
    for (int q = 0; q < SCW; q++) {
        if (q < warp) run += tot[q][lane];
        all += tot[q][lane];
    }
    for (int t = t0; t < t1; t++) {
        const uint32_t c = h[(long long)t * 256];
        h[(long long)t * 256] = run;
        run += c;
    }
    if (warp == 0) w.dtot[(long long)b * 256 + d] = all;
}

// stable scatter of one tile by the digit: rank = (keys of the digit in earlier warps)
// + (in earlier rounds of my warp) + (in lower lanes of my round); destination =
// offset(digit, tile) + rank.  STABLE = false (the first LSD pass, whose input order is
// arbitrary anyway): the in-warp rank is a shared-memory atomic on the warp's digit counter
// instead of the ballot multisplit.  The order of equal keys inside a 24-bit group is never
// observed (every Lloyd quantity is a count or an integer sum over whole groups, R-16), so
// the results stay bitwise deterministic.
template <bool STABLE>
__global__ void __launch_bounds__(KT, 3) km_scatter(const uint32_t *kin, uint32_t *kout, KmPtr w, int shift) {
    pdl_wait();
    using Scan = cub::BlockScan<uint32_t, KT>;
    __shared__ typename Scan::TempStorage stmp;
    __shared__ uint32_t wc[KT / 32 * 256], goff[256], sk[KTILE];
    const int b = blockIdx.y, t = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long pb = (long long)b * w.T * KTILE;
    uint32_t k[KI], rank[KI];
    load_striped(kin, pb + (long long)t * KTILE, k);
    uint32_t base;
    Scan(stmp).ExclusiveSum(w.dtot[(long long)b * 256 + threadIdx.x], base);
    goff[threadIdx.x] = base + w.hist[((long long)b * w.T + t) * 256 + threadIdx.x];
    uint32_t *c = wc + warp * 256;
    for (int i = lane; i < 256; i += 32) c[i] = 0u;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    if (STABLE) {
#pragma unroll
        for (int r = 0; r < KI; r++) {
            const uint32_t d = (k[r] >> shift) & 255u;
            const unsigned peers = digit_peers(d);
            const uint32_t before = c[d];
            const uint32_t lower = (uint32_t)__popc(peers & lt);  // 0 for the lowest peer
            rank[r] = before + lower;
            __syncwarp();
            if (lower == 0u) c[d] = before + (uint32_t)__popc(peers);
            __syncwarp();
        }
    } else {
#pragma unroll
        for (int r = 0; r < KI; r++) rank[r] = atomicAdd(&c[(k[r] >> shift) & 255u], 1u);
    }
    __syncthreads();
    uint32_t run = 0;  // exclusive prefix over warps, per digit (thread = digit), in place
#pragma unroll
    for (int q = 0; q < KT / 32; q++) {
        const uint32_t x = wc[q * 256 + threadIdx.x];
        wc[q * 256 + threadIdx.x] = run;
        run += x;
    }
    uint32_t ts;  // first tile-local position of the digit
    Scan(stmp).ExclusiveSum(run, ts);
    // fold the tile start into the per-warp bases and out of the global offset, so each
    // key below needs one shared-memory lookup per phase
#pragma unroll
    for (int q = 0; q < KT / 32; q++) wc[q * 256 + threadIdx.x] += ts;
    goff[threadIdx.x] -= ts;  // destination of tile position i (digit d) = goff[d] + i (mod 2^32)
    __syncthreads();
    // tile-local sort through shared memory, then runs of equal digits leave coalesced
#pragma unroll
    for (int r = 0; r < KI; r++) {
        const uint32_t d = (k[r] >> shift) & 255u;
        sk[c[d] + rank[r]] = k[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KI; r++) {
        const int i = r * KT + threadIdx.x;
        const uint32_t key = sk[i];
        const uint32_t d = (key >> shift) & 255u;
        kout[pb + (uint32_t)(goff[d] + (uint32_t)i)] = key;
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

// chunk (128 keys) sums of fix(v) over the sorted keys: csum[chunk] = exclusive prefix of
// the chunk sums within its tile, cpre[tile] = the tile's total
__global__ void __launch_bounds__(KT) km_csum(KmPtr w, int sh) {
    pdl_wait();
    __shared__ long long ch[CPT];
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
#pragma unroll
    for (int o = 1; o < KCH / KI; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);  // KCH/KI lanes per chunk
    if ((threadIdx.x & (KCH / KI - 1)) == 0) {
        ch[threadIdx.x / (KCH / KI)] = s;
        // first key of every Lloyd super-chunk (2^sh chunks), contiguous for km_lloyd
        const long long chunk = (long long)t * CPT + threadIdx.x / (KCH / KI);
        if ((chunk & ((1LL << sh) - 1)) == 0) w.heads[(long long)b * LSC_MAX + (chunk >> sh)] = k[0];
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const long long x = ch[threadIdx.x];
        long long inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (threadIdx.x >= o) inc += y;
        }
        w.csum[(long long)b * w.T * CPT + (long long)t * CPT + threadIdx.x] = inc - x;
        if (threadIdx.x == 31) w.cpre[(long long)b * w.T + t] = inc;
    }
    if (t == 0 && threadIdx.x == 0) w.fexp[b] = F;
}

// All Lloyd iterations of one payload in one thread-block cluster of LCL CTAs (one per
// SM).  Every CTA holds the super-chunk heads of the sorted keys (S = KCH << sh keys
// each, sh chosen so at most LSC_MAX of them) and the exclusive prefix of fix(v) at their
// starts in shared memory; CTA r answers the thresholds k = r (mod LCL), one warp each: a
// warp-parallel search over the heads plus ONE global read of one super-chunk (S / 32
// keys per lane), counted and summed by the warp.  Each (C_k, S_k) is stored into every
// CTA's shared memory (DSMEM, double-buffered by iteration parity), one cluster barrier
// per iteration, and every CTA recomputes the centres from the same integers (identical
// results).  Rank 0 writes the centres, thresholds and the final-assignment table.
// last index i of h[0..NS) with p(h[i]) (p monotone: true, then false), -1 if none: a
// warp-parallel search over strides 256, 8, 1 (NS <= 8192)
template <typename Pred>
__device__ __forceinline__ int warp_last(const uint32_t *h, int NS, Pred &&p) {
    const int lane = threadIdx.x & 31;
    const int i1 = lane * 256;
    const unsigned m1 = __ballot_sync(0xffffffffu, i1 < NS && p(h[i1]));
    if (!m1) return -1;
    const int b1 = (31 - __clz(m1)) * 256;
    const int i2 = b1 + lane * 8;
    const unsigned m2 = __ballot_sync(0xffffffffu, i2 < NS && p(h[i2]));
    const int b2 = b1 + (31 - __clz(m2)) * 8;
    const int i3 = b2 + lane;
    const unsigned m3 = __ballot_sync(0xffffffffu, lane < 8 && i3 < NS && p(h[i3]));
    return b2 + (31 - __clz(m3));
}

constexpr int LCL = 8;    // CTAs per payload (portable cluster size)
constexpr int LQ = 16;    // keys per lane in flight in the group scans
constexpr int LCT = 256;  // threads per CTA: LCL * 8 warps >= 64 thresholds
__global__ void __cluster_dims__(LCL, 1, 1) __launch_bounds__(LCT) km_lloyd(KmPtr w, int iters, int sh) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    using Scan = cub::BlockScan<long long, LCT>;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ __align__(16) unsigned char lsm[];
    pdl_wait();  // the sorted keys, chunk sums and heads come from the previous kernels
    const int T = w.T;
    const int S = KCH << sh;
    const int NS = (int)(((long long)T * KTILE) >> (7 + sh));       // super-chunks (KCH == 2^7)
    long long *tpre = reinterpret_cast<long long *>(lsm);            // [T + 1] tile prefix of fix sums
    long long *spre = tpre + T + 1;                                   // [NS] prefix at super-chunk starts
    uint32_t *shead = reinterpret_cast<uint32_t *>(spre + NS);        // [NS] first key of each super-chunk
    __shared__ float cen[256], thr[256];
    // (C_k, S_k) of the step, double-buffered: each threshold's owner warp writes its pair into
    // every CTA of the cluster with st.async, which also counts its 16 bytes on that CTA's
    // mbarrier xbar[buf] -- a step's exchange completes on the receiver's barrier, without a
    // cluster-wide barrier (and its release fence) per Lloyd step
    __shared__ __align__(16) longlong2 CS[2][256];
    __shared__ __align__(8) unsigned long long xbar[2];
    __shared__ long long total_s;
    __shared__ uint32_t lhist[LCT / 32 * 256];  // per-warp low-byte histograms (quantile init)
    const int rank = (int)cluster.block_rank();
    const int b = blockIdx.x / LCL, K = w.K;
    const long long nv = w.nv, nch = (long long)T * CPT;
    const uint32_t *sorted = w.keysA + (long long)b * T * KTILE;
    const long long *cp = w.csum + (long long)b * nch;  // in-tile exclusive chunk prefix
    const long long *ts = w.cpre + (long long)b * T;    // tile totals
    const double scale = ldexp(1.0, w.fexp[b]);
    {  // exclusive prefix over the (<= 4096) tile totals: 16 per thread
        constexpr int TPT = MAX_TILES / LCT;
        long long x[TPT], run = 0;
#pragma unroll
        for (int u = 0; u < TPT; u++) {
            const int t = TPT * threadIdx.x + u;
            x[u] = t < T ? ts[t] : 0;
            run += x[u];
        }
        long long ex, carry;
        Scan(tmp).ExclusiveSum(run, ex, carry);
#pragma unroll
        for (int u = 0; u < TPT; u++) {
            const int t = TPT * threadIdx.x + u;
            if (t < T) tpre[t] = ex;
            ex += x[u];
        }
        if (threadIdx.x == 0) total_s = carry;
    }
    __syncthreads();
    // super-chunk heads and prefixes: 8 global loads of a thread in flight per round
    constexpr int SPT = 8;
    for (int c0 = 0; c0 < NS; c0 += SPT * LCT) {
        uint32_t hv[SPT];
        long long pv[SPT];
#pragma unroll
        for (int u = 0; u < SPT; u++) {
            const int c = c0 + threadIdx.x + u * LCT;
            const long long k0 = (long long)c * S;
            hv[u] = c < NS ? w.heads[(long long)b * LSC_MAX + c] : 0u;
            pv[u] = c < NS ? cp[k0 / KCH] : 0;
        }
#pragma unroll
        for (int u = 0; u < SPT; u++) {
            const int c = c0 + threadIdx.x + u * LCT;
            if (c < NS) {
                shead[c] = hv[u];
                spre[c] = tpre[(int)(((long long)c * S) / KTILE)] + pv[u];
            }
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t xbar_s = (uint32_t)__cvta_generic_to_shared(&xbar[0]);
    const uint32_t cs_s = (uint32_t)__cvta_generic_to_shared(&CS[0][0]);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(xbar_s));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(xbar_s + 8u));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();  // every CTA of the cluster started (DSMEM targets and barriers exist) and staged
    // The keys are ordered by group (top 24 bits), unordered inside a group.  Keys of the
    // super-chunks [c_lo, c_hi] cover group g entirely: c_hi = the last super-chunk whose head
    // is in a group <= g, c_lo = the last one whose head is in a group < g (0 if none); every
    // key before c_lo's start is in a smaller group, every key after c_hi's end in a larger one.
    auto group_range = [&](uint32_t g, long long &beg, long long &end) -> bool {
        const int c_hi = warp_last(shead, NS, [&](uint32_t h) { return (h >> 8) <= g; });
        if (c_hi < 0) return false;  // every key is in a larger group
        const int c_lo = max(0, warp_last(shead, NS, [&](uint32_t h) { return (h >> 8) < g; }));
        beg = (long long)c_lo * S;
        end = min(nv, (long long)(c_hi + 1) * S);
        return true;
    };
    // quantile init: c_k = v_(floor((2k+1) nv / 2K)), the exact order statistic: rank r falls in
    // the group of the key at position r; keys of smaller groups are counted and the low bytes of
    // the group's keys histogrammed (one warp per k), then the byte holding the rank; c_k goes to
    // every CTA's shared memory
    uint32_t *wh = lhist + warp * 256;
    for (int k = rank + LCL * warp; k < K; k += LCL * (LCT / 32)) {
        const long long r = ((long long)(2 * k + 1) * nv) / (2LL * K);
        const uint32_t g = sorted[r] >> 8;
        long long beg = 0, end = 0;
        group_range(g, beg, end);  // non-empty: position r is in group g
        for (int d = lane; d < 256; d += 32) wh[d] = 0u;
        __syncwarp();
        int below = 0;
        for (long long i0 = beg + lane; i0 < end; i0 += 32 * LQ) {
            uint32_t e[LQ];
#pragma unroll
            for (int u = 0; u < LQ; u++) e[u] = i0 + 32 * u < end ? __ldg(sorted + i0 + 32 * u) : 0xffffffffu;
#pragma unroll
            for (int u = 0; u < LQ; u++) {
                if (i0 + 32 * u >= end) continue;
                if ((e[u] >> 8) < g) below++;
                else if ((e[u] >> 8) == g) atomicAdd(&wh[e[u] & 255u], 1u);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
        __syncwarp();
        const uint32_t rr = (uint32_t)(r - beg - below);  // rank inside the group
        uint32_t c8[8], s8 = 0;
#pragma unroll
        for (int u = 0; u < 8; u++) { c8[u] = wh[lane * 8 + u]; s8 += c8[u]; }
        uint32_t inc = s8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const unsigned own = __ballot_sync(0xffffffffu, rr >= inc - s8 && rr < inc);
        const int L = __ffs(own) - 1;
        uint32_t dsel = 0;
        if (lane == L) {
            uint32_t e = inc - s8;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                if (rr < e + c8[u]) { dsel = lane * 8 + u; break; }
                e += c8[u];
            }
        }
        dsel = __shfl_sync(0xffffffffu, dsel, L);
        if (lane < LCL) *cluster.map_shared_rank(&cen[k], lane) = key2f((g << 8) | dsel);
        __syncwarp();
    }
    cluster.sync();  // the initial centres delivered everywhere
    for (int it = 0; it < iters; it++) {
        const int buf = it & 1;
        if (threadIdx.x == 0)  // this step's pairs: one per threshold
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(xbar_s + 8u * buf), "r"(16u * (unsigned)(K - 1)) : "memory");
        for (int k = threadIdx.x; k + 1 < K; k += LCT) thr[k] = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
        __syncthreads();
        const int kk = rank + LCL * warp;  // this warp's threshold (at most one: K <= 256 < LCL * 8 * 4)
        for (int k0 = kk; k0 + 1 < K; k0 += LCL * (LCT / 32)) {
            const uint32_t kb = f2key(thr[k0]);
            long long beg = 0, end = 0;
            const bool any = group_range(kb >> 8, beg, end);  // keys before beg < kb < keys after end
            int cnt = 0;
            long long sm = 0;
            if (any) {  // rounds of LQ loads per lane in flight (one L2 round trip per 32 LQ keys)
                for (long long i0 = beg + lane; i0 < end; i0 += 32 * LQ) {
                    uint32_t e[LQ];
#pragma unroll
                    for (int u = 0; u < LQ; u++) e[u] = i0 + 32 * u < end ? __ldg(sorted + i0 + 32 * u) : 0u;
#pragma unroll
                    for (int u = 0; u < LQ; u++)
                        if (i0 + 32 * u < end && e[u] <= kb) { cnt++; sm += __double2ll_rn((double)key2f(e[u]) * scale); }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                sm += __shfl_xor_sync(0xffffffffu, sm, o);
            }
            const int c = any ? (int)(beg / S) : -1;
            const long long cv = c >= 0 ? beg + cnt : 0;
            const long long sv = c >= 0 ? spre[c] + sm : 0;
            if (lane < LCL) {  // lane r stores into CTA r's shared memory and counts on its barrier
                uint32_t dst, bar;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(cs_s + 16u * (unsigned)(buf * 256 + k0)), "r"(lane));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(xbar_s + 8u * buf), "r"(lane));
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.s64 [%0], {%1, %2}, [%3];"
                             ::"r"(dst), "l"(cv), "l"(sv), "r"(bar) : "memory");
            }
        }
        {  // every pair of this step has landed in this CTA's CS[buf] (its (it / 2)-th phase)
            const unsigned par = (unsigned)(it >> 1) & 1u;
            unsigned ok = 0;
            do {
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                             " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(xbar_s + 8u * buf), "r"(par) : "memory");
            } while (!ok);
        }
        for (int k = threadIdx.x; k < K; k += LCT) {
            const long long c1 = k + 1 < K ? CS[buf][k].x : nv, c0 = k ? CS[buf][k - 1].x : 0;
            const long long s1 = k + 1 < K ? CS[buf][k].y : total_s, s0 = k ? CS[buf][k - 1].y : 0;
            if (c1 > c0) cen[k] = (float)(((double)(s1 - s0) / scale) / (double)(c1 - c0));
        }
        __syncthreads();
    }
    if (rank != 0) {
        cluster.sync();  // keep this CTA's shared memory alive until every remote store landed
        return;
    }
    // final thresholds and the final assignment's bucket table: cnt[q] = #{k : bucket(thr_k) < q}
    const float lo = key2f(sorted[0]), span = __fsub_rn(key2f(sorted[nv - 1]), lo);
    const float bscale = (span > 0.0f && span < INFINITY) ? (float)LUT_NB / span : 0.0f;
    __shared__ int bk[256];
    for (int k = threadIdx.x; k < K; k += LCT) {
        w.cen[(long long)b * K + k] = cen[k];
        if (k + 1 < K) {
            const float t = (float)(((double)cen[k] + (double)cen[k + 1]) * 0.5);
            w.thr[(long long)b * K + k] = t;
            bk[k] = km_bucket(t, lo, bscale);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q <= LUT_NB; q += LCT) {
        int l0 = 0, h0 = K - 1;
        while (l0 < h0) {
            const int mid = (l0 + h0) >> 1;
            if (bk[mid] < q) l0 = mid + 1; else h0 = mid;
        }
        w.lut[(long long)b * (LUT_NB + 1) + q] = l0;
    }
    if (threadIdx.x == 0) { w.lutmap[2 * b] = lo; w.lutmap[2 * b + 1] = bscale; }
    cluster.sync();
}

// final assignment: label(v) = #{k : v > thr[k]}.  A 1024-bucket table over the payload's
// [min, max] (the first and last sorted keys) maps v to the thresholds that share its
// bucket: with bucket() monotone (one rounded subtraction and one rounded product), every
// threshold in an earlier bucket is < v and every one in a later bucket is > v, so
// label = cnt[b] + #{k in bucket b : v > thr_k} -- exact, usually zero or one comparison.
// Lane `bit` stores bit-plane `bit` of its warp's 32-element group; U groups per warp
// per step (loads in flight).
template <int B, typename TO>
__global__ void __launch_bounds__(KT) km_final(const float *const *vin, KmPtr w, uint8_t *const *pay,
                                               int32_t *const *labels_tab, TO *const *dec_out) {
    pdl_wait();
    __shared__ float thr_s[256], cen_s[256];
    __shared__ int cnt_s[LUT_NB + 1];
    const int b = blockIdx.y;
    const int K = w.K;
    const float lo = w.lutmap[2 * b], scale = w.lutmap[2 * b + 1];
    for (int k = threadIdx.x; k < 256; k += KT) thr_s[k] = (k + 1 < K) ? w.thr[(long long)b * K + k] : INFINITY;
    for (int q = threadIdx.x; q <= LUT_NB; q += KT) cnt_s[q] = w.lut[(long long)b * (LUT_NB + 1) + q];
    float *cen_out = reinterpret_cast<float *>(pay[b]);
    uint32_t *planes = reinterpret_cast<uint32_t *>(pay[b] + 4 * (long long)K);
    int32_t *labels = labels_tab ? labels_tab[b] : nullptr;
    TO *dec = dec_out ? dec_out[b] : nullptr;  // fused decode of this (local) payload
    for (int k = threadIdx.x; k < K; k += KT) {
        cen_s[k] = w.cen[(long long)b * K + k];
        if (blockIdx.x == 0) cen_out[k] = cen_s[k];
    }
    __syncthreads();
    const float *vb = vin[b];
    const long long nv = w.nv;
    const long long G = (nv + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long warp0 = ((long long)blockIdx.x * KT + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * KT) >> 5;
    constexpr int U = 8;
    for (long long g0 = warp0 * U; g0 < G; g0 += nwarps * U) {  // warp-uniform
        float v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long i = (g0 + u) * 32 + lane;
            v[u] = i < nv ? __ldg(vb + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int q = km_bucket(v[u], lo, scale);
            int l = cnt_s[q];
            const int e = cnt_s[q + 1];
#pragma unroll 1
            for (int k = l; k < e; k++) l += v[u] > thr_s[k] ? 1 : 0;  // usually 0 or 1 trips
            const long long i = (g0 + u) * 32 + lane;
            if (labels && i < nv) labels[i] = l;
            if (dec && i < nv) dec[i] = (TO)cen_s[l];
            // the B ballot words are warp-uniform: lane 0 stores them (no per-lane select)
            uint32_t word[B > 0 ? B : 1];
#pragma unroll
            for (int bit = 0; bit < B; bit++) {  // predicate from the label bit + VOTE (no SHF/ISETP)
                asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
                    "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
                    : "=r"(word[bit]) : "r"(l), "r"(1u << bit));
            }
            if (lane == 0 && g0 + u < G) {
#pragma unroll
                for (int bit = 0; bit < B; bit++) planes[(g0 + u) * B + bit] = word[bit];
            }
        }
    }
}

template <int B, typename T>
__global__ void __launch_bounds__(256) km_decode(const uint8_t *const *pay, long long nv, int K, T *const *outp) {
    __shared__ float c[256];
    const int b = blockIdx.y;
    for (int k = threadIdx.x; k < K; k += 256) c[k] = reinterpret_cast<const float *>(pay[b])[k];
    __syncthreads();
    const uint32_t *pl = reinterpret_cast<const uint32_t *>(pay[b] + 4 * (long long)K);
    T *out = outp[b];
    const int lane = threadIdx.x & 31;
    const long long G = (nv + 31) / 32;
    const long long warp0 = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * 256) >> 5;
    constexpr int U = 4;  // groups per warp per step, plane loads in flight
    for (long long g0 = warp0 * U; g0 < G; g0 += nwarps * U) {
        uint32_t word[U];
#pragma unroll
        for (int u = 0; u < U; u++) word[u] = (lane < B && g0 + u < G) ? __ldg(pl + (g0 + u) * B + lane) : 0u;
#pragma unroll
        for (int u = 0; u < U; u++) {
            int l = 0;
#pragma unroll
            for (int bit = 0; bit < B; bit++) l |= (int)((__shfl_sync(0xffffffffu, word[u], bit) >> lane) & 1u) << bit;
            const long long i = (g0 + u) * 32 + lane;
            if (i < nv) out[i] = (T)c[l];
        }
    }
}

template <typename F>
void with_bits(int B, F &&f) {
    switch (B) {
        case 0: f(std::integral_constant<int, 0>()); break;
        case 1: f(std::integral_constant<int, 1>()); break;
        case 2: f(std::integral_constant<int, 2>()); break;
        case 3: f(std::integral_constant<int, 3>()); break;
        case 4: f(std::integral_constant<int, 4>()); break;
        case 5: f(std::integral_constant<int, 5>()); break;
        case 6: f(std::integral_constant<int, 6>()); break;
        case 7: f(std::integral_constant<int, 7>()); break;
        default: f(std::integral_constant<int, 8>()); break;
    }
}

int lloyd_shift(int T) {
    int sh = 0;
    while ((((long long)T * KTILE) >> (7 + sh)) > LSC_MAX) sh++;
    return sh;
}
size_t lloyd_smem(int T) {
    const long long ns = ((long long)T * KTILE) >> (7 + lloyd_shift(T));
    return sizeof(long long) * (T + 1 + ns) + sizeof(uint32_t) * ns;
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
    TQ_REQUIRE(K >= 1 && K <= 256, "kmeans: k must be in [1, 256]");
    TQ_REQUIRE(nv >= 1 && nv <= (long long)MAX_TILES * KTILE, "kmeans: payload length must be in [1, 16777216]");
    T = (int)((nv + KTILE - 1) / KTILE);
    const size_t nk = (size_t)P * T * KTILE;
    TQ_CHECK_CUDA(cudaMalloc(&keysA, sizeof(uint32_t) * nk));
    TQ_CHECK_CUDA(cudaMalloc(&keysB, sizeof(uint32_t) * nk));
    TQ_CHECK_CUDA(cudaMalloc(&hist, sizeof(uint32_t) * (size_t)P * T * 256));
    TQ_CHECK_CUDA(cudaMalloc(&dtot, sizeof(uint32_t) * (size_t)P * 256));
    TQ_CHECK_CUDA(cudaMalloc(&csum, sizeof(long long) * (size_t)P * T * CPT));
    TQ_CHECK_CUDA(cudaMalloc(&cpre, sizeof(long long) * (size_t)P * T * CPT));
    TQ_CHECK_CUDA(cudaMalloc(&cen, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&thr, sizeof(float) * P * K));
    TQ_CHECK_CUDA(cudaMalloc(&fexp, sizeof(int) * P));
    TQ_CHECK_CUDA(cudaMalloc(&lut, sizeof(int) * P * (LUT_NB + 1)));
    TQ_CHECK_CUDA(cudaMalloc(&lutmap, sizeof(float) * 2 * P));
    TQ_CHECK_CUDA(cudaMalloc(&heads, sizeof(uint32_t) * P * LSC_MAX));
    TQ_CHECK_CUDA(cudaFuncSetAttribute(km_lloyd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lloyd_smem(T)));
}

void KmeansWork::release() {
    for (void *p : {(void *)keysA, (void *)keysB, (void *)hist, (void *)dtot, (void *)csum, (void *)cpre, (void *)cen,
                    (void *)thr, (void *)fexp, (void *)lut, (void *)lutmap, (void *)heads})
        if (p) cudaFree(p);
    *this = KmeansWork();
}

int kmeans_encode(const float *const *v, KmeansWork &ws, int lloyd, uint8_t *const *pay,
                  int32_t *const *labels, cudaStream_t st, void *const *dec_out, int prec) {
    const KmPtr w = ptrs(ws);
    const int P = ws.P;
    if (P == 0) return 0;
    const dim3 tiles(ws.T, P);
    // LSD passes on the key bytes 1, 2, 3 only: the keys end up ordered by their top 24 bits
    // ("groups": same sign, exponent and top 15 mantissa bits), the low byte unordered inside a
    // group -- km_lloyd resolves the groups it needs (one pass of 4 saved)
    launch_pdl(km_keys, tiles, KT, 0, st, v, w);
    int k = 1;
    uint32_t *src = ws.keysB, *dst = ws.keysA;
    for (int pass = 1; pass < 4; pass++) {
        if (pass > 1) { launch_pdl(km_hist, tiles, KT, 0, st, (const uint32_t *)src, w, 8 * pass); k++; }
        launch_pdl(km_scan, dim3(256 / 32, P), SCW * 32, 0, st, w);
        if (pass == 1) launch_pdl(km_scatter<false>, tiles, KT, 0, st, (const uint32_t *)src, dst, w, 8 * pass);
        else launch_pdl(km_scatter<true>, tiles, KT, 0, st, (const uint32_t *)src, dst, w, 8 * pass);
        k += 2;
        std::swap(src, dst);
    }
    // three passes: B -> A -> B -> A, group-sorted keys in keysA
    launch_pdl(km_csum, tiles, KT, 0, st, w, lloyd_shift(ws.T));
    launch_pdl(km_lloyd, LCL * P, LCT, lloyd_smem(ws.T), st, w, lloyd, lloyd_shift(ws.T));
    long long want = std::max(1LL, (148LL * 8 + P - 1) / P);
    long long need = (ws.nv + KT * 16 - 1) / (KT * 16);
    const dim3 grid((unsigned)std::max(1LL, std::min(want, need)), P);
    with_bits(ws.B, [&](auto Bc) {
        constexpr int BB = decltype(Bc)::value;
        if (prec == 1) launch_pdl(km_final<BB, double>, grid, KT, 0, st, v, w, pay, labels, (double *const *)dec_out);
        else launch_pdl(km_final<BB, float>, grid, KT, 0, st, v, w, pay, labels, (float *const *)dec_out);
    });
    TQ_CHECK_CUDA(cudaGetLastError());
    return k + 3;
}

int kmeans_decode(const uint8_t *const *pay, int P, long long nv, int K, int prec,
                  void *const *out, cudaStream_t st) {
    if (P == 0) return 0;
    const int B = kmeans_bits(K);
    const dim3 grid((unsigned)std::max(1LL, std::min<long long>(1184 / P + 1, (nv + 255) / 256)), P);
    with_bits(B, [&](auto Bc) {
        constexpr int BB = decltype(Bc)::value;
        if (prec == 0) km_decode<BB, float><<<grid, 256, 0, st>>>(pay, nv, K, (float *const *)out);
        else km_decode<BB, double><<<grid, 256, 0, st>>>(pay, nv, K, (double *const *)out);
    });
    TQ_CHECK_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace tq
