// vec.cuh -- streaming vector kernels of the inner CG solver (fp64 scalars from the
// per-node scalar table, fp64 arithmetic in registers, T storage) and small helpers.
#pragma once
#include "common.cuh"
#include "projector.cuh"

namespace tq {

// alpha = rr / p.q of a CG step with p.q = ||A p||^2 + c ||p||^2 (R-8), one CTA per
// node: the forward reduction's per-CTA partials of ||A p||^2 (nfs_pa per angle of the node,
// cgs) and the previous vector pass's per-CTA partials of ||p||^2 (npp of them in cgp; npp = 0:
// scal[S_PP], p0 = r0), each summed in a fixed order -> scal[S_PQ], scal[S_ALPHA]
void launch_cg_alpha(int L, double *scal, const double *cgs, int nfs_pa, const int *nang, const double *cgp,
                     int npp, const double *cnode, int part_stride, cudaStream_t st);
// sinogram-space A x kept by the CG steps (ax == null: none): ax[row] += alpha s[row] for the
// node's rows, s = A p of the step ([n_rows][sp], bin j at j + 1)
struct AxUpdate {
    void *ax;
    const void *s;
    const int *row0, *nang;
    int n_det, sp;
};
// x += alpha p, then (with_p) p = r + beta p and each CTA's ||p||^2 into pp_out[node][block],
// else scal[node][S_NORM] = ||x||^2 (last CG step); and the A x update above
void launch_cg_update_px(int prec, void *x, void *p, const void *r, long long n, int L, double *scal,
                         double *partial, int part_stride, unsigned *counter, bool with_p, double *pp_out,
                         const AxUpdate &au, cudaStream_t st);
// s[row][j + 1] = d[row][j] - ax[row][j]: the CG residual's sinogram term from the kept A x
void launch_resid_from_ax(int prec, const void *d, const void *ax, void *s, int n_rows, int n_det, int sp,
                          cudaStream_t st);
// scal[node][S_NORM] = ||x_node||^2
void launch_norm2(int prec, const void *x, long long n, int L, double *scal, double *partial,
                  int part_stride, unsigned *counter, cudaStream_t st);
// dst[i] = (Tdst) src[i]  (float <-> double conversions / copies)
void launch_convert(int src_prec, const void *src, int dst_prec, void *dst, long long n,
                    cudaStream_t st);
int vec_blocks(long long n);
// tq_params.stop_tol: out[2v] = ||cur_tab[v] - prev_v||^2, out[2v+1] = ||cur_tab[v]||^2 (fp64,
// fixed order), then prev_v = cur_tab[v]; prev [V][n]; partial [V][2 part_stride]; counter [V]
void launch_rel_change(int prec, const void *const *cur_tab, void *prev, long long n, int V, double *out,
                       double *partial, int part_stride, unsigned *counter, cudaStream_t st);

}  // namespace tq
