// vec.cuh -- streaming vector kernels of the inner CG solver (fp64 scalars from the
// per-node scalar table, fp64 arithmetic in registers, T storage) and small helpers.
#pragma once
#include "common.cuh"
#include "projector.cuh"

namespace tq {

// r -= alpha q; rr_new = r.r (per node, deterministic); last block: beta = rr_new / rr,
// rr = rr_new.  (The matching x += alpha p is deferred to launch_cg_update_px, which reads
// p anyway: one pass over x, p fewer per CG step, identical arithmetic.)
void launch_cg_update_r(int prec, void *r, const void *q, long long n, int L, double *scal, double *partial,
                        int part_stride, unsigned *counter, cudaStream_t st);
// x += alpha p, then (with_p) p = r + beta p, else scal[node][S_NORM] = ||x||^2 (last CG step)
void launch_cg_update_px(int prec, void *x, void *p, const void *r, long long n, int L, double *scal,
                         double *partial, int part_stride, unsigned *counter, bool with_p, cudaStream_t st);
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
