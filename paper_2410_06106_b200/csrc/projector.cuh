// projector.cuh -- Joseph forward projector A (ray-driven) and matched backprojector
// A^T (pixel-driven) for sm_100a, with the inner-solver epilogues fused into A^T.
//
// Operator (R-1): P[(a,j),p] = max(0, 1-|t_j-t_p|/m_a)/m_a.
// Forward: each thread owns one ray (a, j) and walks the N lines of the ray's major
// axis, interpolating linearly between the two pixels it passes between (2 taps per
// voxel-update, "VU").  Backward: each thread owns PX pixels and, per angle of its
// node, gathers the <= 2 bins whose triangle covers the pixel.  No atomics: every
// output is summed by one thread in a fixed order, so results are deterministic.
#pragma once
#include "common.cuh"

namespace tq {

enum BpEpi { EPI_PLAIN = 0, EPI_CGQ = 1, EPI_RESID = 2, EPI_GD = 3 };
enum ScalSlot { S_RR = 0, S_PQ = 1, S_ALPHA = 2, S_RRNEW = 3, S_BETA = 4, S_NORM = 5, S_NSLOT = 8 };

template <typename T>
struct FpArgs {
    const T *img;          // [L][n], image of local node r.node
    const T *d;            // RESID: data rows [n_rows][n_det]
    T *out;                // [n_rows][out_stride] + out_off
    const RayRow *rows;    // [n_rows]
    const double2 *trig;   // [n_angles] (cos, sin)
    const int *xmaj;       // [n_angles]
    int N, n_det, out_stride, out_off;
    long long n;
};

template <typename T>
struct BpArgs {
    const T *s;              // [n_rows][s_stride] + s_off
    int s_stride, s_off;
    const int *node_row0;    // [L] first ray row of each node
    const int *node_nang;    // [L]
    const RayRow *rows;      // [n_rows]
    const double2 *trig;
    const int *xmaj;
    int N, n_det;
    long long n;
    // epilogue operands (node-major [L][n])
    T *out;                  // PLAIN: g; CGQ: q; RESID: r; GD: x (in place)
    T *out2;                 // RESID: p (= r)
    const T *vin;            // CGQ: p; RESID/GD: x
    const T *bprime;         // RESID/GD
    const double *cnode;     // [L] c_i
    const double *eta;       // [L] GD step
    double *partial;         // [L][part_stride]
    unsigned *counter;       // [L]
    double *scal;            // [L][S_NSLOT]
    int part_stride;
};

void launch_fp(int prec, bool resid, const void *args, int n_rows, int n_det, cudaStream_t st);
void launch_bp(int prec, int epi, const void *args, int L, int N, cudaStream_t st);
int bp_tiles(int N);

}  // namespace tq
