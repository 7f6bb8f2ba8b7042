// vec.cuh -- streaming vector kernels of the inner CG solver (fp64 scalars from the
// per-node scalar table, fp64 arithmetic in registers, T storage) and small helpers.
#pragma once
#include "common.cuh"
#include "projector.cuh"

namespace tq {

// x += alpha p; r -= alpha q; rr_new = r.r (per node, deterministic); last block:
// beta = rr_new / rr, rr = rr_new.
void launch_cg_update_xr(int prec, void *x, void *r, const void *p, const void *q, long long n,
                         int L, double *scal, double *partial, int part_stride, unsigned *counter,
                         cudaStream_t st);
// p = r + beta p
void launch_cg_update_p(int prec, void *p, const void *r, long long n, int L, const double *scal,
                        cudaStream_t st);
// scal[node][S_NORM] = ||x_node||^2
void launch_norm2(int prec, const void *x, long long n, int L, double *scal, double *partial,
                  int part_stride, unsigned *counter, cudaStream_t st);
// dst[i] = (Tdst) src[i]  (float <-> double conversions / copies)
void launch_convert(int src_prec, const void *src, int dst_prec, void *dst, long long n,
                    cudaStream_t st);
int vec_blocks(long long n);

}  // namespace tq
