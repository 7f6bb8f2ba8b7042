// codecs.cuh -- the two quantizers Q of PAPER.md:268 (eq-compact:conc3), batched over
// P payloads of nv fp32 values each.  Inputs, payloads and outputs are addressed
// through device arrays of pointers (one entry per payload), so a batch can mix local
// iterates, received payloads and segments of the consensus image.
//
// K-means (Alg. 5; exact rules DESIGN.md R-16): LSD radix sort of the
// payload keys on their top 24 bits (low byte resolved per query), quantile init as exact order statistics, E_q Lloyd steps as upper
// bounds + fixed-point prefix sums on the sorted keys (exact, deterministic), final
// assignment, labels packed as ceil(log2 K) bit-planes per 32-element group.
// Payload: [K fp32 centres][ceil(nv/32) * B uint32 planes, group-major].
//
// DCT (R-18): per-payload [min,max], fp64 8-bit map, exact integer two-pass
// 8x8 DCT, IJG-scaled Annex K table, round half away from zero -> int16.
// Payload: [min, max fp32][nv int16 coefficients in [block][u][v] order].
#pragma once
#include "common.cuh"

namespace tq {

int kmeans_bits(int K);
long long kmeans_payload_bytes(int K, long long nv);
long long dct_payload_bytes(long long nv);

struct KmeansWork {
    int P = 0, K = 0, B = 0, T = 0;  // payloads, clusters, bits per label, 2048-key tiles per payload
    long long nv = 0;
    uint32_t *keysA = nullptr;      // [P][T*2048] order-preserving keys (sorted in place)
    uint32_t *keysB = nullptr;      // radix-sort ping-pong buffer
    uint32_t *hist = nullptr;       // [P][T][256] per-tile digit counts -> offsets within the digit
    uint32_t *dtot = nullptr;       // [P][256] digit totals
    long long *csum = nullptr;      // [P][T*32] fixed-point sums of 64-key chunks of the sorted keys
    long long *cpre = nullptr;      // [P][T*32] their exclusive prefix
    float *cen = nullptr;           // [P][K]
    float *thr = nullptr;           // [P][K]
    int *fexp = nullptr;            // [P] fixed-point exponent F
    int *lut = nullptr;             // [P][1025] final-assignment bucket table (km_lloyd)
    uint32_t *heads = nullptr;      // [P][<= 8192] first key of each Lloyd super-chunk (km_csum)
    float *lutmap = nullptr;        // [P][2] bucket map: lo, scale
    void alloc(int P, int K, long long nv);
    void release();
};

// vin[b]: nv floats; pay[b]: payload bytes; labels: table of int32[nv] or null table
// dec_out (optional): per payload, the decoded values c[label] written by the final pass
// (elements of float for prec 0, double for prec 1) -- the decode of a local payload fused
int kmeans_encode(const float *const *vin, KmeansWork &ws, int lloyd, uint8_t *const *pay,
                  int32_t *const *labels, cudaStream_t st, void *const *dec_out = nullptr, int prec = 0);
// out[b]: nv elements of float (prec 0) or double (prec 1)
int kmeans_decode(const uint8_t *const *pay, int P, long long nv, int K, int prec,
                  void *const *out, cudaStream_t st);

struct DctWork {
    int P = 0;
    float *minmax = nullptr;       // [P][2]
    unsigned *counter = nullptr;   // [P]
    float *partial = nullptr;      // [P][part_stride]
    int part_stride = 0;
    void alloc(int P, long long nv);
    void release();
};

// Baseline JPEG Huffman entropy coding of the DCT coefficients (SURVEY NEXT-2, T.81
// Annex F with the Annex K luminance tables, an RSTm marker every R blocks; R-25).
// Entropy payload: [mn f32][mx f32][u32 nbytes | raw flag bit 31][u32 blocks] then the
// entropy-coded segment -- or, when it would exceed the 2 nv bytes of the plain
// coefficients (raw flag), the int16 coefficients.  Capacity 16 + 2 nv bytes.
struct JpegWork {
    int P = 0, R = 0, nint = 0;
    long long nv = 0;
    int16_t *coef = nullptr;        // [P][nv] coefficients (encode input / decode output)
    long long *len = nullptr;       // [P][nint] interval bytes after stuffing, marker included (encode)
    long long *ulen = nullptr;      // [P][nint] interval bytes before stuffing (encode)
    long long *csum = nullptr;      // [P][coder CTAs] stuffed bytes per coder CTA (encode)
    long long *off = nullptr;       // [P][nint] interval starts (decode)
    unsigned *status = nullptr;     // [P][2]: header word, flags (1 category, 16 slot overflow -> raw;
                                    // decode: 2 markers, 4 code, 8 overrun)
    long long *enc_bytes = nullptr; // [P] payload bytes of the last encode (header included)
    uint8_t *scratch = nullptr;     // [P][nint][128 R + 16] per-interval stream before stuffing (encode)
    void alloc(int P, long long nv, int R);
    void release();
};
long long jpeg_payload_bytes(long long nv);
int jpeg_intervals(long long nv, int R);
// pay[b]: payload with mn/mx in bytes 0..7 already; coefficients in w.coef
int jpeg_encode(uint8_t *const *pay, JpegWork &w, cudaStream_t st);
// coefficients of the payloads into w.coef (status bits set on a malformed stream)
int jpeg_decode(uint8_t *const *pay, JpegWork &w, cudaStream_t st);

// jw == nullptr: plain payload [mn][mx][int16 coefficients]; otherwise the entropy
// payload above, the coefficients passing through jw->coef
int dct_encode(const float *const *vin, int P, int rows, int cols, int quality, DctWork &ws,
               uint8_t *const *pay, cudaStream_t st, JpegWork *jw = nullptr);
int dct_decode(const uint8_t *const *pay, int P, int rows, int cols, int quality, int prec,
               void *const *out, cudaStream_t st, JpegWork *jw = nullptr);

// host reference tables (independent of the oracle): Annex K table scaled to quality,
// and the integer DCT matrix round(2^14 alpha(u) cos((2x+1) u pi / 16))
void dct_host_tables(int quality, int *C64, int *Q64);

}  // namespace tq
