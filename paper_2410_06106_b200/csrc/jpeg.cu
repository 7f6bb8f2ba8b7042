// jpeg.cu -- baseline JPEG Huffman entropy coding of the DCT quantizer's coefficients
// (the lossless stage of "standard JPEG"; ITU-T T.81
// Annex C code generation, Annex F.1.2 / F.2.2 coding, Annex K.3 luminance tables,
// RSTm restart markers every R blocks; R-25).
//
// GPU design: one thread per restart interval.  Intervals are independent by
// construction (the DC predictor resets and the stream is byte-aligned at every RSTm),
// so encoding is two passes of the same sequential coder -- count the interval's
// bytes, exclusive scan per payload, write at the scanned offset -- and decoding is a
// marker scan (one CTA per payload) followed by one thread per interval.  Every
// operation is integer: the stream is bit-identical to the oracle's.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "codecs.cuh"

namespace tq {

namespace {

// ITU-T T.81 Table K.3 (DC luminance) and Table K.5 (AC luminance): BITS (codes per
// length 1..16) and HUFFVAL.
const uint8_t kDcBits[16] = {0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0};
const uint8_t kDcVal[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
const uint8_t kAcBits[16] = {0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 0x7d};
const uint8_t kAcVal[162] = {
    0x01, 0x02, 0x03, 0x00, 0x04, 0x11, 0x05, 0x12, 0x21, 0x31, 0x41, 0x06, 0x13, 0x51, 0x61, 0x07, 0x22, 0x71,
    0x14, 0x32, 0x81, 0x91, 0xa1, 0x08, 0x23, 0x42, 0xb1, 0xc1, 0x15, 0x52, 0xd1, 0xf0, 0x24, 0x33, 0x62, 0x72,
    0x82, 0x09, 0x0a, 0x16, 0x17, 0x18, 0x19, 0x1a, 0x25, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x34, 0x35, 0x36, 0x37,
    0x38, 0x39, 0x3a, 0x43, 0x44, 0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59,
    0x5a, 0x63, 0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a, 0x83,
    0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0x9a, 0xa2, 0xa3,
    0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3,
    0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe1, 0xe2,
    0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8, 0xe9, 0xea, 0xf1, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa};

// Everything a coder thread looks up, built once on the host and passed by value
// (copied to shared memory by each CTA).
struct JpegTabs {
    uint32_t ac_pk[256], dc_pk[16];  // encoder: (code << 8) | length by symbol
    uint8_t zz[64];                  // zig-zag position -> natural index
    uint8_t izz[64];                 // natural index -> zig-zag position
    uint16_t dc_co[16], ac_co[256];  // code by symbol
    uint8_t dc_si[16], ac_si[256];   // code length by symbol (0 = no code)
    int32_t dc_max[18], dc_min[17], dc_ptr[17];  // canonical decode per code length
    int32_t ac_max[18], ac_min[17], ac_ptr[17];
    uint8_t dc_val[16], ac_val[176];
    uint16_t dc_lut[512], ac_lut[512];  // first 9 bits -> (length << 8) | symbol, 0: longer code
};

// Annex C for one table: code lengths in order of BITS, canonical code values
// (increment within a length, shift left between lengths), then per length the first
// and last code and the index of the first symbol.
void build_table(const uint8_t *bits, const uint8_t *val, uint16_t *co, uint8_t *si, int32_t *mx, int32_t *mn,
                 int32_t *ptr) {
    int code = 0, k = 0;
    for (int l = 1; l <= 16; l++) {
        const int cnt = bits[l - 1];
        if (cnt == 0) {
            mx[l] = -1; mn[l] = 0; ptr[l] = k;
        } else {
            mn[l] = code; ptr[l] = k;
            for (int i = 0; i < cnt; i++, k++, code++) {
                co[val[k]] = (uint16_t)code;
                si[val[k]] = (uint8_t)l;
            }
            mx[l] = code - 1;
        }
        code <<= 1;
    }
    mx[17] = 0x7fffffff;  // sentinel: any 17-bit prefix ends the search (malformed)
}

const JpegTabs &tabs() {
    static JpegTabs t;
    static bool done = false;
    if (!done) {
        memset(&t, 0, sizeof t);
        build_table(kDcBits, kDcVal, t.dc_co, t.dc_si, t.dc_max, t.dc_min, t.dc_ptr);
        build_table(kAcBits, kAcVal, t.ac_co, t.ac_si, t.ac_max, t.ac_min, t.ac_ptr);
        memcpy(t.dc_val, kDcVal, 12);
        memcpy(t.ac_val, kAcVal, 162);
        // decode lookahead: every code of <= 9 bits fills the entries it prefixes
        auto fill = [](const uint16_t *co, const uint8_t *si, int nsym, uint16_t *lut) {
            for (int sym = 0; sym < nsym; sym++) {
                const int L = si[sym];
                if (L == 0 || L > 9) continue;
                const int base = co[sym] << (9 - L);
                for (int x = 0; x < (1 << (9 - L)); x++) lut[base + x] = (uint16_t)((L << 8) | sym);
            }
        };
        fill(t.dc_co, t.dc_si, 16, t.dc_lut);
        fill(t.ac_co, t.ac_si, 256, t.ac_lut);
        for (int sym = 0; sym < 256; sym++) t.ac_pk[sym] = ((uint32_t)t.ac_co[sym] << 8) | t.ac_si[sym];
        for (int sym = 0; sym < 16; sym++) t.dc_pk[sym] = ((uint32_t)t.dc_co[sym] << 8) | t.dc_si[sym];
        // zig-zag (T.81 Figure A.6): anti-diagonals d = row + col, even d walked with the
        // row decreasing, odd d with the row increasing
        int k = 0;
        for (int d = 0; d < 15; d++) {
            const int lo = d < 8 ? 0 : d - 7, hi = d < 8 ? d : 7;
            for (int i = 0; i <= hi - lo; i++) {
                const int row = (d & 1) ? lo + i : hi - i;
                t.zz[k++] = (uint8_t)(row * 8 + (d - row));
            }
        }
        for (int i = 0; i < 64; i++) t.izz[t.zz[i]] = (uint8_t)i;
        done = true;
    }
    return t;
}

constexpr int JT = 32;   // decoder threads (intervals) per CTA: one warp, so few intervals still spread over the SMs
constexpr int JW = 8;    // warps (intervals) per CTA of the long-interval coder
constexpr int RW = 128;  // words of a long-interval coder warp's bit ring (4096 bits)
constexpr int JENC = offsetof(JpegTabs, dc_co);  // bytes of the tables the encoder reads (packed codes, zig-zag)

__device__ __forceinline__ int category(int v) { return 32 - __clz(v < 0 ? -v : v); }
__device__ __forceinline__ unsigned low_bits(int v, int s) { return (unsigned)(v < 0 ? v - 1 : v) & ((1u << s) - 1u); }

__device__ __forceinline__ const int16_t *coef_of(uint8_t *const *pay, const int16_t *coef_base, int b,
                                                  long long nv) {
    return coef_base ? coef_base + (long long)b * nv : reinterpret_cast<const int16_t *>(pay[b] + 8);
}

// scratch slot of one interval: the raw size of its blocks; an interval whose stuffed
// stream (marker included) is longer makes the payload fall back to raw coefficients
__host__ __device__ __forceinline__ long long jpeg_slot(int R) { return 128LL * R + 16; }

// L <= 27 bits of `code`, MSB first, at stream bit p of a ring of RW big-endian words;
// disjoint bit ranges from different lanes may share a word, hence the OR atomics
__device__ __forceinline__ void ring_put(uint32_t *ring, long long p, unsigned code, int L) {
    const int w = (int)(p >> 5) & (RW - 1), o = (int)(p & 31);
    const unsigned long long v = (unsigned long long)code << (64 - o - L);
    atomicOr(ring + w, (uint32_t)(v >> 32));
    if ((uint32_t)v) atomicOr(ring + ((w + 1) & (RW - 1)), (uint32_t)v);
}

// Both coders leave in the interval's scratch slot its stream BEFORE byte stuffing
// (ulen bytes, fill bits included) and record len = the stuffed length (one 0x00 after
// every 0xFF, T.81 F.1.2.3) plus the RSTm marker; jpeg_place stuffs while copying.

// Long restart intervals (R > JBK blocks): one warp per interval, the 64 zig-zag
// positions of a block on the 32 lanes (k = lane and lane + 32).  A lane's symbol for a
// non-zero AC coefficient depends only on the distance to the previous non-zero one (the
// ballot mask of the block), a warp prefix sum over zig-zag order gives each code's bit
// offset, the codes are OR-ed into a bit ring in shared memory, and complete bytes are
// flushed to the slot as the ring fills.
__global__ void __launch_bounds__(JW * 32) jpeg_code_ring(const __grid_constant__ JpegTabs tab,
                                                          const int16_t *coef_base, uint8_t *const *pay,
                                                          long long nv, int R, int nint, long long *len,
                                                          long long *ulen, long long *csum, uint8_t *scratch,
                                                          unsigned *status) {
    __shared__ __align__(16) uint32_t tb[JENC / 4];
    __shared__ uint32_t ringS[JW][RW];
    for (int i = threadIdx.x; i < JENC / 4; i += JW * 32) tb[i] = reinterpret_cast<const uint32_t *>(&tab)[i];
    const JpegTabs &T = *reinterpret_cast<const JpegTabs *>(tb);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *ring = ringS[wid];
    for (int i = lane; i < RW; i += 32) ring[i] = 0;
    __syncthreads();
    const int b = blockIdx.y;
    const int k = blockIdx.x * JW + wid;
    if (k >= nint) return;
    const long long nblk = nv / 64;
    const long long b0 = (long long)k * R, b1 = min(nblk, b0 + R);
    const int16_t *coef = coef_of(pay, coef_base, b, nv);
    const long long slot = jpeg_slot(R);
    uint8_t *out = scratch + ((long long)b * nint + k) * slot;
    const int zz0 = T.zz[lane], zz1 = T.zz[lane + 32];
    const uint32_t zrl = T.ac_pk[0xF0], eob = T.ac_pk[0x00];
    long long pos = 0, fbyte = 0, nff = 0;  // bits coded, bytes flushed, 0xFF bytes among them
    bool bad = false;
    int pred = 0;
    // bytes [fbyte, nb) of the ring to the slot; the flushed words are cleared
    auto flush = [&](long long nb) {
        for (long long i0 = fbyte; i0 < nb; i0 += 32) {
            const long long i = i0 + lane;
            const bool in = i < nb;
            const unsigned byte = in ? (ring[(i >> 2) & (RW - 1)] >> (24 - 8 * (int)(i & 3))) & 0xffu : 0u;
            nff += __popc(__ballot_sync(~0u, in && byte == 0xffu));
            if (in && i < slot) out[i] = (uint8_t)byte;
        }
        __syncwarp();
        for (long long w = fbyte >> 2; w < (nb >> 2); w += 32)
            if (w + lane < (nb >> 2)) ring[(w + lane) & (RW - 1)] = 0;
        fbyte = nb;
        __syncwarp();
    };
    for (long long bl = b0; bl < b1; bl++) {
        const int16_t *cb = coef + bl * 64;
        const int v0 = __ldg(cb + zz0), v1 = __ldg(cb + zz1);
        const unsigned long long m = (unsigned long long)(__ballot_sync(~0u, v0 != 0) & ~1u) |
                                     ((unsigned long long)__ballot_sync(~0u, v1 != 0) << 32);
        const int dc = __shfl_sync(~0u, v0, 0);
        const int diff = dc - pred;
        pred = dc;
        // this lane's two items: code bits (value bits appended) and ZRL count
        unsigned c[2] = {0u, 0u};
        int L[2] = {0, 0}, lz[2] = {0, 0}, nz[2] = {0, 0};
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int kk = lane + 32 * h;
            const int v = h ? v1 : v0;
            if (kk == 0) {
                const int s = category(diff);
                if (s > 11) { bad = true; continue; }
                const uint32_t e = T.dc_pk[s];
                c[h] = ((e >> 8) << s) | low_bits(diff, s);
                lz[h] = (int)(e & 0xffu) + s;
            } else if (v != 0) {
                const unsigned long long below = m & ((1ull << kk) - 1ull);
                const int prev = below ? 63 - __clzll((long long)below) : 0;
                const int run = kk - prev - 1;
                const int sz = category(v);
                if (sz > 10) { bad = true; continue; }
                const uint32_t e = T.ac_pk[((run & 15) << 4) | sz];
                nz[h] = run >> 4;
                c[h] = ((e >> 8) << sz) | low_bits(v, sz);
                lz[h] = (int)(e & 0xffu) + sz;
            }
            L[h] = nz[h] * (int)(zrl & 0xffu) + lz[h];
        }
        // exclusive prefix over zig-zag order: positions 0..31, then 32..63
        int s0 = L[0], s1 = L[1];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t0 = __shfl_up_sync(~0u, s0, d), t1 = __shfl_up_sync(~0u, s1, d);
            if (lane >= d) { s0 += t0; s1 += t1; }
        }
        const int T0 = __shfl_sync(~0u, s0, 31), T1 = __shfl_sync(~0u, s1, 31);
        const long long p0 = pos + s0 - L[0], p1 = pos + T0 + s1 - L[1];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            if (!L[h]) continue;
            long long p = h ? p1 : p0;
            for (int z = 0; z < nz[h]; z++, p += zrl & 0xffu) ring_put(ring, p, zrl >> 8, zrl & 0xffu);
            ring_put(ring, p, c[h], lz[h]);
        }
        pos += T0 + T1;
        if (!(m >> 63)) {  // EOB unless the last coefficient is non-zero
            if (lane == 0) ring_put(ring, pos, eob >> 8, eob & 0xffu);
            pos += eob & 0xffu;
        }
        __syncwarp();
        if (pos - 8 * fbyte > 32 * RW / 2) flush(pos >> 3);  // <= 2055 bits pending, + <= 1700 per block
    }
    if (pos & 7) {  // fill bits: ones up to the byte boundary
        const int f = 8 - (int)(pos & 7);
        if (lane == 0) ring_put(ring, pos, (1u << f) - 1u, f);
        pos += f;
        __syncwarp();
    }
    flush(pos >> 3);
    if (__any_sync(~0u, bad) && lane == 0) atomicOr(status + 2 * b + 1, 1u);
    if (lane == 0) {
        const long long n = (pos >> 3) + nff + (k + 1 < nint ? 2 : 0);
        if (n > slot) atomicOr(status + 2 * b + 1, 16u);  // slot overflow: raw fallback (not an error)
        len[(long long)b * nint + k] = n;
        ulen[(long long)b * nint + k] = pos >> 3;
        atomicAdd(reinterpret_cast<unsigned long long *>(csum + (long long)b * gridDim.x + blockIdx.x),
                  (unsigned long long)n);
    }
}

constexpr int JB = 256;        // threads per CTA of the block coder
constexpr int JSUB = 4;        // threads per 8x8 block: zig-zag positions [16 sub, 16 sub + 16)
constexpr int JBK = JB / JSUB; // blocks per CTA; restart intervals up to JBK blocks use this coder

// L <= 27 bits of `code` at bit p of a linear big-endian word buffer of `cap` bits;
// bits past the end are dropped (the interval then overflows its slot anyway)
__device__ __forceinline__ void buf_put(uint32_t *buf, int p, int cap, unsigned code, int L) {
    if (p + L > cap) return;
    const int w = p >> 5, o = p & 31;
    const unsigned long long v = (unsigned long long)code << (64 - o - L);
    atomicOr(buf + w, (uint32_t)(v >> 32));
    if ((uint32_t)v) atomicOr(buf + w + 1, (uint32_t)v);
}

// The symbols of the non-zero AC positions `own` of one block, in stream order, with
// the DC difference first when `dc` (F.1.2.1) and the EOB last when `eob` (F.1.2.2: AC
// run/size with ZRL; `prev` = the last non-zero position before the first of `own`, 0 if
// none).  Returns the bit count.  EMIT == false collects the codes in `acc` (valid when
// the count is <= 64); EMIT == true ORs them into `buf` at bit p.
template <bool EMIT>
__device__ __forceinline__ int code_items(const JpegTabs &T, const int16_t *zb, unsigned long long own, int prev,
                                          bool dc, bool eob, int diff, unsigned long long &acc, uint32_t *buf, int p,
                                          int cap, bool &bad) {
    int n = 0;
    auto put = [&](unsigned code, int L) {
        if (EMIT) buf_put(buf, p + n, cap, code, L);
        else if (n + L <= 64) acc = (acc << L) | code;
        n += L;
    };
    if (dc) {
        const int s = category(diff);
        if (s > 11) bad = true;
        else put((T.dc_pk[s] >> 8 << s) | low_bits(diff, s), (int)(T.dc_pk[s] & 0xffu) + s);
    }
    while (own) {
        const int k = __ffsll((long long)own) - 1;
        own &= own - 1;
        int run = k - prev - 1;
        prev = k;
        for (; run > 15; run -= 16) put(T.ac_pk[0xF0] >> 8, (int)(T.ac_pk[0xF0] & 0xffu));
        const int v = zb[k];
        const int sz = category(v);
        if (sz > 10) { bad = true; continue; }
        const uint32_t e = T.ac_pk[(run << 4) | sz];
        put(((e >> 8) << sz) | low_bits(v, sz), (int)(e & 0xffu) + sz);
    }
    if (eob) put(T.ac_pk[0x00] >> 8, (int)(T.ac_pk[0x00] & 0xffu));
    return n;
}

// position of the r-th (0-based) set bit of m, 64 when r >= popc(m)
__device__ __forceinline__ int nth_set_bit(unsigned long long m, int r) {
    if (r >= __popcll(m)) return 64;
    int pos = 0;
#pragma unroll
    for (int s = 32; s; s >>= 1) {
        const int c = __popcll((m >> pos) & ((1ull << s) - 1ull));
        if (c <= r) { r -= c; pos += s; }
    }
    return pos;
}

// Restart intervals of R <= JBK blocks: JSUB threads per 8x8 block, the CTA holding
// JBK / R whole intervals.  A block's symbols depend only on its non-zero mask (a run is
// the distance to the previous non-zero coefficient) and the previous block's DC, so the
// block's non-zero AC coefficients are split into JSUB runs of equal count, consecutive
// in zig-zag order (DC with the first, EOB with the last), each coded by one thread into
// a 64-bit register.  One CTA scan over the threads, in stream order, gives every thread
// its bit offset inside its interval, and the codes are OR-ed into the interval's region
// of a shared-memory bit buffer (a thread with more than 64 bits walks its coefficients
// again and ORs them one code at a time).  The interval's words then go to its scratch
// slot with the 0xFF count.
__global__ void __launch_bounds__(JB, 8) jpeg_code_blocks(const __grid_constant__ JpegTabs tab,
                                                          const int16_t *coef_base, uint8_t *const *pay, long long nv,
                                                          int R, int nint, long long *len, long long *ulen,
                                                          long long *csum, uint8_t *scratch, unsigned *status) {
    using Scan = cub::BlockScan<int, JB>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ __align__(16) uint32_t tb[JENC / 4];
    __shared__ __align__(16) int16_t zblk[JBK * 64];  // blocks in zig-zag order
    __shared__ int sx[JB], ibytes[JBK], iff[JBK], csum_s;
    extern __shared__ uint4 ubuf4[];  // ipc slots of the interval streams
    uint32_t *ubuf = reinterpret_cast<uint32_t *>(ubuf4);
    const int ipc = JBK / R;
    const int slot = (int)jpeg_slot(R), slotw = slot / 4;
    for (int i = threadIdx.x; i < JENC / 4; i += JB) tb[i] = reinterpret_cast<const uint32_t *>(&tab)[i];
    for (int i = threadIdx.x; i < ipc * slot / 16; i += JB) ubuf4[i] = make_uint4(0, 0, 0, 0);
    const JpegTabs &T = *reinterpret_cast<const JpegTabs *>(tb);
    const int b = blockIdx.y;
    const int t = threadIdx.x, bi = t / JSUB, sub = t % JSUB;
    const long long nblk = nv / 64;
    const int kf = blockIdx.x * ipc;  // first interval of the CTA
    const int j = bi / R;             // this block's interval in the CTA
    const long long bl = (long long)kf * R + bi;
    const bool act = j < ipc && kf + j < nint && bl < nblk;
    int16_t *zb = zblk + bi * 64;
    if (t == 0) csum_s = 0;
    if (t < JBK) { ibytes[t] = 0; iff[t] = 0; }
    __syncthreads();  // tables in place before the zig-zag scatter reads T.izz
    if (act) {  // this thread's 16 coefficients (two rows) to their zig-zag positions
        const uint4 *src = reinterpret_cast<const uint4 *>(coef_of(pay, coef_base, b, nv) + bl * 64) + 2 * sub;
        const uint4 v0 = __ldg(src), v1 = __ldg(src + 1);
        const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        const uint8_t *iz = T.izz + 16 * sub;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            zb[iz[2 * i]] = (int16_t)(w[i] & 0xffffu);
            zb[iz[2 * i + 1]] = (int16_t)(w[i] >> 16);
        }
    }
    __syncthreads();
    unsigned m16 = 0;
    if (act) {
        const uint32_t *zw = reinterpret_cast<const uint32_t *>(zb) + 8 * sub;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t x = zw[i];
            m16 |= (unsigned)((x & 0xffffu) != 0) << (2 * i) | (unsigned)((x >> 16) != 0) << (2 * i + 1);
        }
    }
    if (sub == 0) m16 &= ~1u;  // DC is not part of the AC mask
    unsigned long long m = 0;
#pragma unroll
    for (int s2 = 0; s2 < JSUB; s2++) m |= (unsigned long long)__shfl_sync(~0u, m16, s2, JSUB) << (16 * s2);
    // this thread's share: non-zero coefficients [nz sub / JSUB, nz (sub + 1) / JSUB)
    const int nz = __popcll(m);
    const int ka = nth_set_bit(m, nz * sub / JSUB), kb = nth_set_bit(m, nz * (sub + 1) / JSUB);
    const unsigned long long own = ka == 64 ? 0ull : (m >> ka << ka) & (kb == 64 ? ~0ull : (1ull << kb) - 1ull);
    const unsigned long long below = ka == 64 ? m : m & ((1ull << ka) - 1ull);
    const int prev = below ? 63 - __clzll((long long)below) : 0;
    const bool eob = sub == JSUB - 1 && !(m >> 63);
    const int diff = (sub == 0 && act) ? zb[0] - (bi % R ? (int)zb[-64] : 0) : 0;
    bool bad = false;
    unsigned long long acc = 0;
    const int nb = act ? code_items<false>(T, zb, own, prev, sub == 0, eob, diff, acc, nullptr, 0, 0, bad) : 0;
    int ex;
    Scan(tmp).ExclusiveSum(nb, ex);
    sx[t] = ex;
    __syncthreads();
    const int t0 = j * R * JSUB;  // first thread of the interval
    const int nth = act ? JSUB * (int)min((long long)R, nblk - (long long)(kf + j) * R) : 0;  // the last may be short
    const bool lastt = act && t == t0 + nth - 1;
    const int p = ex - (act ? sx[t0] : 0), bits = p + nb;
    uint32_t *ib = ubuf + j * slotw;
    const int cap = 8 * slot;
    if (act && nb) {
        if (nb > 64) {
            code_items<true>(T, zb, own, prev, sub == 0, eob, diff, acc, ib, p, cap, bad);
        } else if (p + nb <= cap) {  // the <= 64 collected bits in one 96-bit window
            const int w = p >> 5;
            const unsigned __int128 win = (unsigned __int128)acc << (96 - (p & 31) - nb);
            const uint32_t w1 = (uint32_t)(win >> 32), w2 = (uint32_t)win;
            atomicOr(ib + w, (uint32_t)(win >> 64));
            if (w1) atomicOr(ib + w + 1, w1);
            if (w2) atomicOr(ib + w + 2, w2);
        }
    }
    if (lastt) {
        ibytes[j] = (bits + 7) / 8;
        if ((bits & 7) && bits < cap) buf_put(ib, bits, cap, (1u << (8 - (bits & 7))) - 1u, 8 - (bits & 7));  // fill: ones
    }
    if (__syncthreads_or(bad) && t == 0) atomicOr(status + 2 * b + 1, 1u);
    // the interval's words to its scratch slot (bytes in stream order), counting 0xFF bytes
    if (act) {
        uint32_t *out = reinterpret_cast<uint32_t *>(scratch + ((long long)b * nint + kf + j) * slot);
        const int nby = ibytes[j], nw = min(slotw, (nby + 3) / 4);
        int cnt = 0;
        for (int i = t - t0; i < nw; i += nth) {
            const uint32_t word = ib[i];
            const int nbw = min(4, nby - 4 * i);
            cnt += __popc(__vcmpeq4(word, 0xffffffffu) & (0xffffffffu << (32 - 8 * nbw))) / 8;
            out[i] = __byte_perm(word, 0, 0x0123);
        }
        if (cnt) atomicAdd(iff + j, cnt);
    }
    __syncthreads();
    int n = 0;
    if (lastt) {
        const int k = kf + j;
        n = ibytes[j] + iff[j] + (k + 1 < nint ? 2 : 0);
        if (ibytes[j] > slot || n > slot) atomicOr(status + 2 * b + 1, 16u);  // raw fallback (not an error)
        len[(long long)b * nint + k] = n;
        ulen[(long long)b * nint + k] = ibytes[j];
    }
    if (n) atomicAdd(&csum_s, n);
    __syncthreads();
    if (t == 0) csum[(long long)b * gridDim.x + blockIdx.x] = csum_s;
}

// Interval k = 8 blockIdx.x + warp of payload blockIdx.y to its place in the payload.
// Its offset = the coder CTAs' sums before its CTA (`gi` intervals per coder CTA) plus
// the lengths before it inside that CTA; one warp copies the interval's bytes with the
// 0x00 stuffed after every 0xFF and appends the RSTm marker.  Header word 2 = nbytes |
// raw flag (bit 31) when a coder flagged the payload or the stream would not fit in the
// raw coefficients' 2 nv bytes; word 3 = number of blocks.  A raw payload gets its
// coefficients instead, split over the payload's CTAs.
constexpr int ST = 1024;  // marker-scan threads (decoder)
constexpr int PW = 8;     // warps (intervals) per CTA of jpeg_place
__global__ void __launch_bounds__(PW * 32) jpeg_place(uint8_t *const *pay, const int16_t *coef_base,
                                                      const uint8_t *scratch, const long long *len,
                                                      const long long *ulen, const long long *csum, int gi, int ncta,
                                                      int nint, int R, long long nv, const unsigned *status_in,
                                                      unsigned *status, long long *enc_bytes) {
    const int b = blockIdx.y, lane = threadIdx.x & 31;
    const int k = blockIdx.x * PW + (threadIdx.x >> 5);
    const long long *cs = csum + (long long)b * ncta, *lb = len + (long long)b * nint;
    const int c = min(k, nint - 1) / gi;  // the coder CTA of interval k
    long long pre = 0, tot = 0;
    for (int i = lane; i < ncta; i += 32) {
        const long long x = cs[i];
        tot += x;
        if (i < c) pre += x;
    }
    for (int i = c * gi + lane; i < k; i += 32) pre += lb[i];
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        pre += __shfl_xor_sync(~0u, pre, d);
        tot += __shfl_xor_sync(~0u, tot, d);
    }
    const bool raw = status_in[2 * b + 1] != 0 || tot > 2 * nv;
    if (k == 0 && lane == 0) {
        uint32_t *hdr = reinterpret_cast<uint32_t *>(pay[b]);
        hdr[2] = raw ? 0x80000000u : (uint32_t)tot;
        hdr[3] = (uint32_t)(nv / 64);
        status[2 * b] = hdr[2];
        if (enc_bytes) enc_bytes[b] = 16 + (raw ? 2 * nv : tot);
    }
    if (raw) {
        const uint4 *src = reinterpret_cast<const uint4 *>(coef_base + (long long)b * nv);
        uint4 *dst = reinterpret_cast<uint4 *>(pay[b] + 16);
        const long long n16 = nv / 8, per = (n16 + gridDim.x - 1) / gridDim.x;
        const long long e = min(n16, per * (blockIdx.x + 1));
        for (long long i = per * blockIdx.x + threadIdx.x; i < e; i += PW * 32) dst[i] = src[i];
        return;
    }
    if (k >= nint) return;
    const unsigned lt = (1u << lane) - 1u;
    const long long nu = ulen[(long long)b * nint + k];
    const uint8_t *src = scratch + ((long long)b * nint + k) * jpeg_slot(R);
    uint8_t *dst = pay[b] + 16 + pre;
    long long o = 0;
    for (long long i0 = 0; i0 < nu; i0 += 32) {
        const long long i = i0 + lane;
        const bool in = i < nu;
        const unsigned byte = in ? src[i] : 0u;
        const unsigned ff = __ballot_sync(~0u, in && byte == 0xffu);
        const long long q = o + lane + __popc(ff & lt);
        if (in) {
            dst[q] = (uint8_t)byte;
            if (byte == 0xffu) dst[q + 1] = 0;
        }
        o += min(32LL, nu - i0) + __popc(ff);
    }
    if (k + 1 < nint && lane == 0) {
        dst[o] = 0xFF;
        dst[o + 1] = (uint8_t)(0xD0 + (k & 7));
    }
}

// ---- decoder
// starts[b][k] = first byte of interval k: 0, then 2 past the k-th RSTm marker in
// stream order (markers are the only 0xFF not followed by 0x00).  One CTA per payload.
__global__ void __launch_bounds__(ST) jpeg_markers(uint8_t *const *pay, int nint, long long *starts,
                                                   unsigned *status) {
    using Scan = cub::BlockScan<int, ST>;
    __shared__ typename Scan::TempStorage tmp;
    const int b = blockIdx.x;
    const uint32_t w2 = reinterpret_cast<const uint32_t *>(pay[b])[2];
    if (w2 & 0x80000000u) return;  // raw payload
    const long long n = w2;
    const uint8_t *s = pay[b] + 16;
    const long long chunk = (n + ST - 1) / ST;
    const long long i0 = (long long)threadIdx.x * chunk, i1 = min(n, i0 + chunk);
    int cnt = 0;
    for (long long i = i0; i < i1; i++)
        if (s[i] == 0xFF && i + 1 < n && (s[i + 1] & 0xF8) == 0xD0) cnt++;
    int ex, tot;
    Scan(tmp).ExclusiveSum(cnt, ex, tot);
    long long *sb = starts + (long long)b * nint;
    if (threadIdx.x == 0) {
        sb[0] = 0;
        if (tot != nint - 1) atomicOr(status + 2 * b + 1, 2u);
    }
    if (tot != nint - 1) return;
    for (long long i = i0; i < i1; i++)
        if (s[i] == 0xFF && i + 1 < n && (s[i + 1] & 0xF8) == 0xD0) {
            if ((s[i + 1] & 7) != (ex & 7)) atomicOr(status + 2 * b + 1, 2u);
            sb[1 + ex++] = i + 2;
        }
}

// stream reader of one thread: a 64-bit buffer refilled bytewise (stuffed 0x00 after
// 0xFF skipped); bits beyond the interval read as zeros and are counted as an overrun
struct BitR {
    const uint8_t *in;
    long long pos, end;
    unsigned long long buf;
    int nb;
    long long real_bits, used;
    __device__ void refill() {
        while (nb <= 48) {
            unsigned byte = 0;
            if (pos < end) {
                byte = in[pos];
                pos += byte == 0xFFu ? 2 : 1;
                real_bits += 8;
            }
            buf |= (unsigned long long)byte << (56 - nb);
            nb += 8;
        }
    }
    __device__ unsigned peek(int n) const { return (unsigned)(buf >> (64 - n)); }
    __device__ void skip(int n) { buf <<= n; nb -= n; used += n; }
    __device__ int bits(int s) {
        if (s == 0) return 0;
        refill();
        const int v = (int)peek(s);
        skip(s);
        return v;
    }
};

// DECODE (T.81 F.2.2.3): 9-bit lookahead table, then the canonical MAXCODE search for
// longer codes
__device__ __forceinline__ int decode_symbol(BitR &r, const uint16_t *lut, const int32_t *mx, const int32_t *mn,
                                             const int32_t *ptr, const uint8_t *val) {
    r.refill();
    const unsigned p = r.peek(16);
    const unsigned e = lut[p >> 7];
    if (e) {
        r.skip((int)(e >> 8));
        return (int)(e & 0xffu);
    }
    for (int l = 10; l <= 16; l++) {
        const int code = (int)(p >> (16 - l));
        if (code <= mx[l]) {
            r.skip(l);
            return val[ptr[l] + code - mn[l]];
        }
    }
    return -1;
}

__global__ void __launch_bounds__(JT) jpeg_decode_k(const __grid_constant__ JpegTabs tab, uint8_t *const *pay,
                                                     int16_t *coef_base, long long nv, int R, int nint,
                                                     const long long *starts, unsigned *status) {
    __shared__ JpegTabs T;
    for (int i = threadIdx.x; i < (int)(sizeof(JpegTabs) / 4); i += JT)
        reinterpret_cast<uint32_t *>(&T)[i] = reinterpret_cast<const uint32_t *>(&tab)[i];
    __syncthreads();
    const int b = blockIdx.y;
    const int k = blockIdx.x * JT + threadIdx.x;
    if (k >= nint) return;
    const uint32_t w2 = reinterpret_cast<const uint32_t *>(pay[b])[2];
    if ((w2 & 0x80000000u) || status[2 * b + 1]) return;
    const long long n = w2;
    const long long *sb = starts + (long long)b * nint;
    BitR r{pay[b] + 16, sb[k], k + 1 < nint ? sb[k + 1] - 2 : n, 0ull, 0, 0, 0};
    const long long nblk = nv / 64;
    const long long b0 = (long long)k * R, b1 = min(nblk, b0 + R);
    int16_t *out = coef_base + (long long)b * nv;
    int pred = 0;
    for (long long bl = b0; bl < b1; bl++) {
        int16_t *c = out + bl * 64;
        int16_t v[64];
#pragma unroll
        for (int i = 0; i < 64; i++) v[i] = 0;
        const int s = decode_symbol(r, T.dc_lut, T.dc_max, T.dc_min, T.dc_ptr, T.dc_val);
        if (s < 0 || s > 11) { atomicOr(status + 2 * b + 1, 4u); return; }
        int d = r.bits(s);
        if (s && d < (1 << (s - 1))) d += 1 - (1 << s);  // EXTEND
        pred += d;
        v[0] = (int16_t)pred;
        for (int kk = 1; kk < 64; kk++) {
            const int rs = decode_symbol(r, T.ac_lut, T.ac_max, T.ac_min, T.ac_ptr, T.ac_val);
            if (rs < 0) { atomicOr(status + 2 * b + 1, 4u); return; }
            const int run = rs >> 4, sz = rs & 15;
            if (sz == 0) {
                if (run == 15) { kk += 15; continue; }
                break;
            }
            kk += run;
            if (kk > 63) { atomicOr(status + 2 * b + 1, 4u); return; }
            int a = r.bits(sz);
            if (a < (1 << (sz - 1))) a += 1 - (1 << sz);
            v[T.zz[kk]] = (int16_t)a;
        }
        uint4 *dst = reinterpret_cast<uint4 *>(c);
        const uint4 *src = reinterpret_cast<const uint4 *>(v);
#pragma unroll
        for (int q = 0; q < 8; q++) dst[q] = src[q];
    }
    if (r.used > r.real_bits) atomicOr(status + 2 * b + 1, 8u);
}

// raw payloads: coefficients straight from the payload
__global__ void jpeg_raw_in(uint8_t *const *pay, int16_t *coef_base, long long nv) {
    const int b = blockIdx.y;
    if (!(reinterpret_cast<const uint32_t *>(pay[b])[2] & 0x80000000u)) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(pay[b] + 16);
    uint4 *dst = reinterpret_cast<uint4 *>(coef_base + (long long)b * nv);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv / 8; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

}  // namespace

long long jpeg_payload_bytes(long long nv) { return 16 + 2 * nv; }
int jpeg_intervals(long long nv, int R) { return (int)((nv / 64 + R - 1) / R); }

void JpegWork::alloc(int P_, long long nv_, int R_) {
    P = P_; nv = nv_; R = R_;
    TQ_REQUIRE(R >= 1, "jpeg: restart interval must be >= 1 block");
    TQ_REQUIRE(nv % 64 == 0 && nv / 64 < (1LL << 30), "jpeg: payload must be whole 8x8 blocks");
    nint = jpeg_intervals(nv, R);
    const size_t np = (size_t)std::max(1, P);
    TQ_CHECK_CUDA(cudaMalloc(&coef, sizeof(int16_t) * nv * np));
    TQ_CHECK_CUDA(cudaMalloc(&len, sizeof(long long) * nint * np));
    TQ_CHECK_CUDA(cudaMalloc(&off, sizeof(long long) * nint * np));
    TQ_CHECK_CUDA(cudaMalloc(&ulen, sizeof(long long) * nint * np));
    TQ_CHECK_CUDA(cudaMalloc(&csum, sizeof(long long) * nint * np));
    TQ_CHECK_CUDA(cudaMalloc(&status, sizeof(unsigned) * 2 * np));
    TQ_CHECK_CUDA(cudaMalloc(&enc_bytes, sizeof(long long) * np));
    TQ_CHECK_CUDA(cudaMalloc(&scratch, (size_t)(128LL * R + 16) * nint * np));
    TQ_CHECK_CUDA(cudaMemset(enc_bytes, 0, sizeof(long long) * np));
}

void JpegWork::release() {
    for (void *p : {(void *)coef, (void *)len, (void *)off, (void *)ulen, (void *)csum, (void *)status, (void *)enc_bytes, (void *)scratch})
        if (p) cudaFree(p);
    *this = JpegWork();
}

int jpeg_encode(uint8_t *const *pay, JpegWork &w, cudaStream_t st) {
    if (w.P == 0) return 0;
    const JpegTabs &t = tabs();
    TQ_CHECK_CUDA(cudaMemsetAsync(w.status, 0, sizeof(unsigned) * 2 * w.P, st));
    int gi, ncta;  // intervals per coder CTA, coder CTAs per payload
    if (w.R <= JBK) {
        gi = JBK / w.R;
        ncta = ceil_div(w.nint, gi);
        jpeg_code_blocks<<<dim3(ncta, w.P), JB, gi * jpeg_slot(w.R), st>>>(t, w.coef, pay, w.nv, w.R, w.nint, w.len,
                                                                          w.ulen, w.csum, w.scratch, w.status);
    } else {
        gi = JW;
        ncta = ceil_div(w.nint, gi);
        TQ_CHECK_CUDA(cudaMemsetAsync(w.csum, 0, sizeof(long long) * ncta * w.P, st));
        jpeg_code_ring<<<dim3(ncta, w.P), JW * 32, 0, st>>>(t, w.coef, pay, w.nv, w.R, w.nint, w.len, w.ulen, w.csum,
                                                            w.scratch, w.status);
    }
    jpeg_place<<<dim3(ceil_div(w.nint, PW), w.P), PW * 32, 0, st>>>(pay, w.coef, w.scratch, w.len, w.ulen, w.csum,
                                                                    gi, ncta, w.nint, w.R, w.nv, w.status, w.status,
                                                                    w.enc_bytes);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 2;
}

int jpeg_decode(uint8_t *const *pay, JpegWork &w, cudaStream_t st) {
    if (w.P == 0) return 0;
    const JpegTabs &t = tabs();
    TQ_CHECK_CUDA(cudaMemsetAsync(w.status, 0, sizeof(unsigned) * 2 * w.P, st));
    jpeg_markers<<<w.P, ST, 0, st>>>(pay, w.nint, w.off, w.status);
    jpeg_decode_k<<<dim3(ceil_div(w.nint, JT), w.P), JT, 0, st>>>(t, pay, w.coef, w.nv, w.R, w.nint, w.off,
                                                                   w.status);
    jpeg_raw_in<<<dim3(std::max(1, std::min(16, (int)ceil_div(w.nv / 8, 256))), w.P), 256, 0, st>>>(
        pay, w.coef, w.nv);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 3;
}

}  // namespace tq
