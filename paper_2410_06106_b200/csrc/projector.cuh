// projector.cuh -- Joseph forward projector A and matched backprojector A^T for sm_100a,
// with the inner-solver epilogues fused into A^T.
//
// Operator (R-1): P[(a,j),p] = max(0, 1-|t_j-t_p|/m_a)/m_a.
//
// Siddon (R-26): on each major-axis line (a band one pixel thick) the
// ray covers the cross interval [c - w/2, c + w/2], w = |B| <= 1 the cross drift per
// line, with length 1/m_a; it meets pixels a = floor(c) and a + 1 only, and pixel a + 1
// receives the fraction g = sat((u - 1/2) / w + 1/2), u = c - a (g = u is Joseph).  The
// same tiles, windows and reduction serve both; w = 0 (axis rays, exact trig) uses the
// slope 2^22 so that u = 1/2 (a ray on a pixel edge) gives exactly 1/2.  The transpose
// weight of bin distance s is sat(a0 - s a1), a1 = 1/(m w), a0 = (1 + 1/w)/2 (Joseph:
// a1 = 1/m, a0 = 1), times the 1/m pre-scale of the staged bins.
//
// Forward (A), "image-tile stationary": one CTA stages a TH x TW tile of one node's
// image in shared memory (zero halo on both sides of the cross axis) and walks, for
// EVERY angle of that node whose major axis matches the tile orientation, all rays
// that cross the tile: per line of the tile one bilinear sample (2 taps) from shared
// memory.  Each ray's partial sum over the tile goes to a dense scratch slot indexed by
// (ray row, line band, parity of the cross tile, bin): a ray meets at most two cross
// tiles per band, and they differ in parity, so no slot has two writers.  fp_reduce
// adds a ray's slots in band order (deterministic, no atomics) and applies 1/m_a and
// the residual.  y-major angles walk rows of a wide
// tile, x-major angles walk columns of a tall tile (the transposed staging), so the
// rays a tile touches are mostly full-length segments.  Each image pixel is read from
// HBM/L2 once per orientation per application, for all angles of its node.
//
// Backward (A^T), pixel-driven: one CTA owns a 64 x 64 pixel tile, stages for every
// angle of its node the window of <= 96 sinogram bins the tile projects onto
// (pre-scaled by 1/m_a), and each thread gathers the <= 2 bins under each of its 16
// pixels per angle (2 shared-memory taps + 2 saturating FMAs for the weights).
#pragma once
#include "common.cuh"

namespace tq {

enum BpEpi { EPI_PLAIN = 0, EPI_CGQ = 1, EPI_RESID = 2, EPI_GD = 3, EPI_CGR = 4 };
// zero elements before and after a backprojector input (rows with zero guard bins at 0 and
// n_det + 1): the 96-bin windows are staged without bounds checks; slots outside
// [-1, n_det] only feed pixels outside the image
constexpr int SPAD = 256;
enum ScalSlot { S_RR = 0, S_PQ = 1, S_ALPHA = 2, S_RRNEW = 3, S_BETA = 4, S_NORM = 5, S_PP = 6, S_NSLOT = 8 };

// forward tile geometry
constexpr int FP_TH = 32;                 // lines (major-axis steps) per tile
constexpr int FP_TW = 128;                // cross-axis extent of a tile
constexpr int FP_HALO = FP_TH + 6;        // zero columns each side: covers a ray's drift over TH lines
constexpr int FP_WMAX = FP_TW + FP_TH + 8;  // max rays crossing one tile for one angle
constexpr int FP_THREADS = 256;
constexpr int FP_MAXA = 64;               // angles per shared-memory batch
constexpr int FPP_MAXA = 32;              // angles per batch of the persistent fp32 forward kernel

// Static per-(ray row, tile) geometry of the forward tiles, computed once (fp_setup):
// the window of rays [jlo, jlo + W) that cross the tile and the shared-memory cross
// coordinate kap of ray jlo on the tile's first line (ray jlo + w sits at kap + w*at).
struct FpWin {
    double kap;
    int jlo, W;
};
struct FpRowGeo {   // per ray row: cross step per bin and per line, cross coordinate of bin c0 on line 0
    double at, B, a0;
};

// The same, per (tile, position in the orientation-grouped row list `olist`), laid out
// so that one forward work unit (node, orientation, tile) reads its records as one
// contiguous run (prefetched with cp.async by the persistent fp32 kernel).
struct FpRec {
    double kap;  // shared-memory cross coordinate of ray jlo on the tile's first line, minus FP2 origin
    double at;   // cross step per bin
    float B;     // cross step per line
    int jlo, W, row;
};

// Static per-unit item plan of the persistent fp32 forward kernel (first batch of <= 32
// angles of a unit).  Work is split into half-warp items of nh_k consecutive rays of one
// angle k, nh_k = min(16, floor(15 / at_k) + 1), so the 16 lanes of a half-warp read one
// line's (e, d) pairs within a window of 16 consecutive 8-byte slots: every LDS.64 of the
// ray walk is conflict-free (2 wavefronts per warp).  hpre = exclusive prefix of the
// half-item counts ceil(W_k / nh_k); hk = per half-item k | nh_k << 5 | (its index within
// angle k) << 10, so an item learns its angle, width and first ray from one load.
// Bulk-copied with the unit's records.
constexpr int FPP_HMAX = 512;  // >= FPP_MAXA * ceil(FP_WMAX / 11) half-items per batch
struct FpUnitTab {
    int hpre[FPP_MAXA + 1];
    unsigned char nh[FPP_MAXA];
    unsigned short hk[FPP_HMAX];
    int pad[3];
};
__host__ __device__ inline unsigned short fp_hk_pack(int k, int nh, int rank) {
    return (unsigned short)(k | (nh << 5) | (rank << 10));
}
static_assert(FPP_MAXA <= 32 && (FP_WMAX + 10) / 11 <= 64, "half-item packing (5 | 5 | 6 bits)");
static_assert(sizeof(FpUnitTab) % 16 == 0, "bulk-copy granularity");
static_assert(FPP_MAXA * ((FP_WMAX + 10) / 11) <= FPP_HMAX, "half-item table too small");

template <typename T>
struct FpArgs {
    const T *img;          // [L][n] node-major images
    long long n;
    int N, n_det;
    const int *olist;      // ray rows grouped by (node, orientation)
    const int *oofs;       // [2L+1] offsets into olist; group g = 2*node + orientation
    const FpWin *wins;     // [n_rows][ntiles]
    const FpRowGeo *rgeo;  // [n_rows]
    T *partial;            // [n_rows][nt_line][2][n_det]: band lt, cross-tile parity ct & 1
    int nt_line, nt_cross; // tiles along the major / cross axis (same for both orientations)
    uint32_t magic;        // = 0x4B000000 << 2 (mod 2^32), see projector.cu magic_base
    const FpRec *recs;     // [ntiles][n_olist] (fp32 persistent kernel)
    int n_olist, L;
    const FpUnitTab *utab; // [2 * L_all * ntiles] (fp32 persistent kernel)
    int siddon;            // 1: Siddon weights (R-26) -- generic tile kernel
    // node group (persistent fp32 kernel): the launch covers nodes [node0, node0 + L) of the
    // L_all nodes the unit tables were built for; img and oofs point at node0's entries
    int node0, L_all;
};

// per ray row of a context: (cos, sin, m, 1/w) of its angle for the backprojector (one load
// instead of the rows -> angle -> trig / xmaj chain); 1/w only for Siddon (R-26)
void launch_bp_rowc(const RayRow *rows, const double2 *trig, const int *xmaj, int n_rows, double4 *rowc,
                    cudaStream_t st);

// row stride (bins) of the forward partial slots: n_det rounded up to a multiple of 4
__host__ __device__ inline int fp_ps(int n_det) { return (n_det + 3) & ~3; }

template <typename T>
struct FpRedArgs {
    const T *partial;      // as FpArgs::partial; slots no tile writes stay zero
    const RayRow *rows;
    const double2 *trig;
    const int *xmaj;
    const T *d;            // RESID: data [n_rows][n_det]
    T *out;                // [n_rows][out_stride] + out_off
    int out_stride, out_off;
    int N, n_det, nt_line;
    const double4 *rowc;   // [n_rows] as BpArgs::rowc (m in .z), or null
    const FpRowGeo *rgeo;  // [n_rows] (fp32): skip the slots no tile of the row writes; null: read all
    int nt_cross;
    // CG step (cg != 0, not RESID): each CTA's sum of squared outputs into cgs[node][k *
    // gridDim.x + blockIdx.x] (k = the row's angle within its node): ||A p||^2 for cg_alpha
    int cg;
    double *cgs;           // [L][part_stride]
    int part_stride;
    int row_base;          // the launch reduces rows [row_base, row_base + gridDim.y) (a node group)
};

template <typename T>
struct BpArgs {
    const T *s;              // [n_rows][s_stride] + s_off; s_off >= 1 zero guard bins each side,
                             // SPAD zero elements before row 0 and after the last row
    int s_stride, s_off;
    const int *node_row0;    // [L] first ray row of each node
    const int *node_nang;    // [L]
    const RayRow *rows;      // [n_rows]
    const double2 *trig;
    const int *xmaj;
    int N, n_det;
    long long n;
    // epilogue operands (node-major [L][n])
    T *out;                  // PLAIN: g; CGQ: q; RESID: r; GD: x (in place); CGR: r - alpha q
    T *out2;                 // RESID: p (= r)
    const T *vin;            // CGQ/CGR: p; RESID/GD: x
    const T *bprime;         // RESID/GD: b'; CGR: r
    const double *cnode;     // [L] c_i
    const double *eta;       // [L] GD step
    double *partial;         // [L][part_stride]
    unsigned *counter;       // [L]
    double *scal;            // [L][S_NSLOT]
    int part_stride;
    uint32_t magic;          // = 0x4B000000 << 2 (mod 2^32)
    int siddon;              // 1: Siddon weights (R-26)
    const double4 *rowc;     // [n_rows] (cos, sin, m, 1/w) per ray row, or null (from rows/trig/xmaj)
};

constexpr uint32_t kMagicBits4 = 0x2C000000u;  // (0x4B000000 << 2) mod 2^32
void projector_setup();                   // per-device kernel attributes (not capturable)
int fp_ntiles(int N);                     // tiles per orientation
int bp_tiles(int N);
// forward: tile pass over L nodes then the fixed-order reduction over n_rows rows
void launch_fp(int prec, const void *args, int L, cudaStream_t st);
// static forward geometry of n_rows rows (once per context)
void launch_fp_setup(const RayRow *rows, const int *xmaj, const double2 *trig, int n_rows, int N, int n_det,
                     FpWin *wins, FpRowGeo *rgeo, const int *olist, int n_olist, FpRec *recs, const int *oofs, int L,
                     FpUnitTab *utab, cudaStream_t st);
void launch_fp_reduce(int prec, bool resid, const void *args, int n_rows, int n_det, cudaStream_t st);
int fp_reduce_blocks(int prec, int n_det);  // CTAs per row of launch_fp_reduce
void launch_bp(int prec, int epi, const void *args, int L, int N, cudaStream_t st);

}  // namespace tq
