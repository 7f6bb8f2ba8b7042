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
    uint16_t dc_co[16], ac_co[256];  // code by symbol
    uint8_t dc_si[16], ac_si[256];   // code length by symbol (0 = no code)
    uint8_t zz[64];                  // zig-zag position -> natural index
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
        done = true;
    }
    return t;
}

constexpr int JT = 32;   // threads (intervals) per CTA: one warp, so few intervals still spread over the SMs
constexpr int BLKP = 66; // int16 pitch of a thread's staged block: 33 words, conflict-free columns

// stream writer of one thread: bits MSB first, 0x00 stuffed after 0xFF, fill bits 1
struct BitW {
    uint8_t *out;  // bytes beyond cap are counted, not stored
    long long pos, cap;
    unsigned long long acc;
    int nb;
    __device__ void byte(unsigned b) {
        if (pos < cap) out[pos] = (uint8_t)b;
        pos++;
    }
    __device__ void put(unsigned code, int size) {
        acc = (acc << size) | code;
        nb += size;
        while (nb >= 8) {
            nb -= 8;
            const unsigned b = (unsigned)(acc >> nb) & 0xffu;
            byte(b);
            if (b == 0xffu) byte(0);
        }
    }
    __device__ void pad() {
        if (nb) put((1u << (8 - nb)) - 1u, 8 - nb);
    }
};

__device__ __forceinline__ int category(int v) { return 32 - __clz(v < 0 ? -v : v); }

// code blocks [b0, b1) of one payload (DC predictor starts at 0); status bit 1 set if
// a value falls outside the baseline categories
__device__ void code_interval(const JpegTabs &T, const int16_t *coef, long long b0, long long b1, BitW &w,
                              int16_t *blk, unsigned *bad) {
    int pred = 0;
    for (long long b = b0; b < b1; b++) {
        const uint4 *src = reinterpret_cast<const uint4 *>(coef + b * 64);
        uint32_t *dst = reinterpret_cast<uint32_t *>(blk);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint4 v = __ldg(src + q);
            dst[4 * q] = v.x; dst[4 * q + 1] = v.y; dst[4 * q + 2] = v.z; dst[4 * q + 3] = v.w;
        }
        const int dc = blk[0];
        const int diff = dc - pred;
        pred = dc;
        const int s = category(diff);
        if (s > 11) { atomicOr(bad, 1u); return; }
        w.put(T.dc_co[s], T.dc_si[s]);
        if (s) w.put((unsigned)(diff < 0 ? diff - 1 : diff) & ((1u << s) - 1u), s);
        // non-zero AC coefficients in zig-zag order as a bit mask, then one step per
        // non-zero coefficient (run = distance to the previous one)
        unsigned long long nz = 0;
#pragma unroll
        for (int k = 1; k < 64; k++) nz |= (unsigned long long)(blk[T.zz[k]] != 0) << k;
        int last = 0;
        while (nz) {
            const int k = __ffsll((long long)nz) - 1;
            nz &= nz - 1;
            int run = k - last - 1;
            last = k;
            while (run > 15) { w.put(T.ac_co[0xF0], T.ac_si[0xF0]); run -= 16; }
            const int v = blk[T.zz[k]];
            const int sz = category(v);
            if (sz > 10) { atomicOr(bad, 1u); return; }
            const int rs = (run << 4) | sz;
            w.put(T.ac_co[rs], T.ac_si[rs]);
            w.put((unsigned)(v < 0 ? v - 1 : v) & ((1u << sz) - 1u), sz);
        }
        if (last < 63) w.put(T.ac_co[0x00], T.ac_si[0x00]);  // EOB
    }
    w.pad();
}

__device__ __forceinline__ const int16_t *coef_of(uint8_t *const *pay, const int16_t *coef_base, int b,
                                                  long long nv) {
    return coef_base ? coef_base + (long long)b * nv : reinterpret_cast<const int16_t *>(pay[b] + 8);
}

// interval k of payload blockIdx.y coded into its scratch slot (SLOT(R) bytes: the raw
// size of its blocks; a longer interval makes the payload fall back to raw coefficients)
__device__ __forceinline__ long long jpeg_slot(int R) { return 128LL * R + 16; }
__global__ void __launch_bounds__(JT) jpeg_code(const __grid_constant__ JpegTabs tab, const int16_t *coef_base,
                                                uint8_t *const *pay, long long nv, int R, int nint, long long *len,
                                                uint8_t *scratch, unsigned *status) {
    __shared__ JpegTabs T;
    __shared__ __align__(16) int16_t blk[JT][BLKP];
    for (int i = threadIdx.x; i < (int)(sizeof(JpegTabs) / 4); i += JT)
        reinterpret_cast<uint32_t *>(&T)[i] = reinterpret_cast<const uint32_t *>(&tab)[i];
    __syncthreads();
    const int b = blockIdx.y;
    const int k = blockIdx.x * JT + threadIdx.x;
    if (k >= nint) return;
    const long long nblk = nv / 64;
    const long long b0 = (long long)k * R, b1 = min(nblk, b0 + R);
    const int16_t *coef = coef_of(pay, coef_base, b, nv);
    unsigned *st = status + 2 * b;
    const long long slot = jpeg_slot(R);
    BitW w{scratch + ((long long)b * nint + k) * slot, 0, slot, 0, 0};
    code_interval(T, coef, b0, b1, w, blk[threadIdx.x], st + 1);
    if (k + 1 < nint) { w.byte(0xFF); w.byte(0xD0 + (k & 7)); }
    if (w.pos > slot) atomicOr(st + 1, 16u);  // slot overflow: raw fallback (not an error)
    len[(long long)b * nint + k] = w.pos;
}

// one warp per interval: the scratch bytes to their scanned offset in the payload
__global__ void jpeg_copy(uint8_t *const *pay, const uint8_t *scratch, const long long *len, const long long *off,
                          int nint, int R, const unsigned *status) {
    const int b = blockIdx.y;
    if (status[2 * b] & 0x80000000u) return;
    const int k = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (k >= nint) return;
    const long long slot = jpeg_slot(R), n = len[(long long)b * nint + k];
    const uint8_t *src = scratch + ((long long)b * nint + k) * slot;
    uint8_t *dst = pay[b] + 16 + off[(long long)b * nint + k];
    for (long long i = lane; i < n; i += 32) dst[i] = src[i];
}

// exclusive scan of the interval lengths of payload blockIdx.x; header word 2 =
// nbytes | raw flag (bit 31) when the stream would not fit in the raw coefficients'
// 2 nv bytes; word 3 = number of blocks
constexpr int ST = 1024;
__global__ void __launch_bounds__(ST) jpeg_scan(const long long *len, long long *off, int nint, long long nv,
                                                uint8_t *const *pay, unsigned *status, long long *enc_bytes) {
    using Scan = cub::BlockScan<long long, ST>;
    __shared__ typename Scan::TempStorage tmp;
    const int b = blockIdx.x;
    long long carry = 0;
    for (int c0 = 0; c0 < nint; c0 += ST) {
        const int k = c0 + threadIdx.x;
        const long long x = k < nint ? len[(long long)b * nint + k] : 0;
        long long ex, tot;
        Scan(tmp).ExclusiveSum(x, ex, tot);
        if (k < nint) off[(long long)b * nint + k] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const bool bad = status[2 * b + 1] != 0;  // category overflow (1) or slot overflow (16)
        const bool raw = bad || carry > 2 * nv;
        uint32_t *hdr = reinterpret_cast<uint32_t *>(pay[b]);
        hdr[2] = raw ? 0x80000000u : (uint32_t)carry;
        hdr[3] = (uint32_t)(nv / 64);
        status[2 * b] = hdr[2];
        if (enc_bytes) enc_bytes[b] = 16 + (raw ? 2 * nv : carry);
    }
}

// raw fallback: coefficients (16-byte chunks) into the payload after the header
__global__ void jpeg_raw_copy(const int16_t *coef_base, uint8_t *const *pay, long long nv, const unsigned *status) {
    const int b = blockIdx.y;
    if (!(status[2 * b] & 0x80000000u)) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(coef_base + (long long)b * nv);
    uint4 *dst = reinterpret_cast<uint4 *>(pay[b] + 16);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv / 8; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
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
    TQ_CHECK_CUDA(cudaMalloc(&status, sizeof(unsigned) * 2 * np));
    TQ_CHECK_CUDA(cudaMalloc(&enc_bytes, sizeof(long long) * np));
    TQ_CHECK_CUDA(cudaMalloc(&scratch, (size_t)(128LL * R + 16) * nint * np));
    TQ_CHECK_CUDA(cudaMemset(enc_bytes, 0, sizeof(long long) * np));
}

void JpegWork::release() {
    for (void *p : {(void *)coef, (void *)len, (void *)off, (void *)status, (void *)enc_bytes, (void *)scratch})
        if (p) cudaFree(p);
    *this = JpegWork();
}

int jpeg_encode(uint8_t *const *pay, JpegWork &w, cudaStream_t st) {
    if (w.P == 0) return 0;
    const JpegTabs &t = tabs();
    TQ_CHECK_CUDA(cudaMemsetAsync(w.status, 0, sizeof(unsigned) * 2 * w.P, st));
    const dim3 grid(ceil_div(w.nint, JT), w.P);
    jpeg_code<<<grid, JT, 0, st>>>(t, w.coef, pay, w.nv, w.R, w.nint, w.len, w.scratch, w.status);
    jpeg_scan<<<w.P, ST, 0, st>>>(w.len, w.off, w.nint, w.nv, pay, w.status, w.enc_bytes);
    jpeg_copy<<<dim3(ceil_div(w.nint, 8), w.P), 256, 0, st>>>(pay, w.scratch, w.len, w.off, w.nint, w.R, w.status);
    jpeg_raw_copy<<<dim3(std::max(1, std::min(16, (int)ceil_div(w.nv / 8, 256))), w.P), 256, 0, st>>>(
        w.coef, pay, w.nv, w.status);
    TQ_CHECK_CUDA(cudaGetLastError());
    return 4;
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
