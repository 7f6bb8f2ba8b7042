// solver.cuh -- device geometry tables and the batched inner solver: every local node
// i solves min 1/2||A_i x - d_i||^2 + c_i/2 ||x||^2 - b_i'^T x (PAPER.md:158
// eq:solve_u; R-7) by E1 steps of GD (Alg. 2) or CG (R-8), all
// nodes of the rank in the same launches.
#pragma once
#include "common.cuh"
#include "projector.cuh"
#include "vec.cuh"

namespace tq {

// device geometry shared by all nodes of a context
struct DevGeom {
    int N = 0, n_ang = 0, n_det = 0, proj = 0;  // proj: 0 Joseph, 1 Siddon
    long long n = 0;
    double2 *trig = nullptr;  // [n_ang]
    int *xmaj = nullptr;      // [n_ang]
    std::vector<int> xmaj_h;
    void init(int N, int n_ang, int n_det, int proj = 0, const double *angles_rad = nullptr);
    void release();
};

enum AxMode { AX_OFF = 0, AX_REFRESH = 1, AX_CACHED = 2 };

struct Inner {
    int prec = 0, L = 0, n_rows = 0, sp = 0, part_stride = 0;
    long long n = 0;
    RayRow *rows = nullptr;    // [n_rows]
    int *row0 = nullptr;       // [L]
    int *nang = nullptr;       // [L]
    int *olist = nullptr;      // ray rows grouped by (node, major axis) for the forward tiles
    int *oofs = nullptr;       // [2L+1]
    void *fpart = nullptr;     // forward partial sums [n_rows][nt_line][2][n_det] (zeroed once)
    FpWin *fwin = nullptr;     // [n_rows][fp_ntiles] static ray windows of the forward tiles
    FpRowGeo *frg = nullptr;   // [n_rows]
    FpRec *frec = nullptr;     // [fp_ntiles][n_olist] (persistent fp32 forward kernel)
    FpUnitTab *futab = nullptr; // [2 L fp_ntiles]
    int n_olist = 0;
    int nt_line = 0, nt_cross = 0;
    void *X = nullptr, *R = nullptr, *P = nullptr, *Q = nullptr, *BP = nullptr;  // [L][n]
    void *D = nullptr;         // [n_rows][n_det]
    void *AX = nullptr;        // [n_rows][n_det] A x of the current X (CG, ax mode != AX_OFF)
    void *S = nullptr;         // [n_rows][sp], guard column at 0 and n_det+1 (inside S_base)
    void *S_base = nullptr;    // S with SPAD zero elements before and after
    double *cnode = nullptr, *eta = nullptr;  // [L]
    double *scal = nullptr;    // [L][S_NSLOT]
    double *partial = nullptr; // [L][part_stride]
    double *cgs = nullptr, *cgp = nullptr;  // [L][part_stride] CG step: ||A p||^2 / ||p||^2 partials (cg_alpha)
    unsigned *counter = nullptr;
    double4 *rowc = nullptr;     // [n_rows] backprojector per-row angle constants
    std::vector<RayRow> rows_h;
    std::vector<int> row0_h, nang_h;
    // angle lists per local node (global angle ids, increasing)
    void init(int prec, const DevGeom &g, const std::vector<std::vector<int>> &angles);
    void release();
    size_t esize() const { return prec ? 8 : 4; }
    void *xrow(void *base, int i) const { return (char *)base + esize() * n * i; }
    // launches; return the number of kernels launched
    // ax: AX_OFF = residual projection of X every solve; AX_REFRESH = project X into AX first;
    // AX_CACHED = residual d - AX (AX = A x maintained by the CG steps: A x += alpha A p)
    // n0, cnt: only the node group [n0, n0 + cnt) (cnt < 0: to the last node); every launch of a
    // group touches only that group's vectors, tables and ray rows (fp32, persistent forward kernel)
    int cg(const DevGeom &g, int e1, cudaStream_t st, int ax = 0, int n0 = 0, int cnt = -1);
    int gd(const DevGeom &g, int e1, cudaStream_t st);
    int norm2(cudaStream_t st);
    // S = (D -) A img (2 tile launches + 1 reduction); out/out_stride/out_off override S;
    // cg: the reduction also sets alpha of a CG step from ||S||^2 (see cg())
    int project(const DevGeom &g, const void *img, bool resid, cudaStream_t st, void *out = nullptr,
                int out_stride = 0, int out_off = 0, bool cg = false, int n0 = 0, int cnt = -1);
    // rin: the residual r read by EPI_CGR (out may alias it)
    int backproject(const DevGeom &g, int epi, void *out, void *out2, const void *vin, cudaStream_t st,
                    const void *rin = nullptr, int n0 = 0, int cnt = -1);
};

}  // namespace tq
