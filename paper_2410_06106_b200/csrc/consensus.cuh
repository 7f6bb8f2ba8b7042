// consensus.cuh -- the consensus / dual steps of both ADMM rules (elementwise, HBM
// streams), fused with the next right-hand side b' of the local problems.
#pragma once
#include "common.cuh"

namespace tq {

// rule=graph (R-7): for local node i with public value xh_i = Q(x_i) and
// neighbour sum S_i = sum_j xh_j:  alpha_i += rho (deg_i xh_i - S_i);
// b'_i = -alpha_i + rho (deg_i xh_i + S_i).  update_alpha = 0 only recomputes b'.
int launch_graph_dual(int prec, const void *const *own_ptr, const void *const *nbr_ptr, const int *nbr_off,
                      void *alpha, void *bprime, long long n, int L, double rho,
                      int update_alpha, cudaStream_t st);

// rule=paper, Alg. 3 on node i's own segment [lo_i, lo_i + len) of its
// slice's consensus image xg_tab[i]:  E2 times  x <- x - eta2 rho (x - u - lambda/rho).
// Result to seg_tab[i] (fp32, to be quantized) or, if seg_tab == null, in place in xg.
int launch_paper_alg3(int prec, const void *u, const void *lam, void *const *xg_tab,
                      const long long *lo, const long long *len, long long max_len,
                      float *const *seg_tab, long long n, int L, double rho, double eta2, int e2,
                      cudaStream_t st);

// rule=paper, eq:solve_lamda and the next b' = rho x - lambda:
// lambda += rho (u - x) (update_lam = 1), b' = rho x - lambda.
int launch_paper_dual(int prec, const void *u, void *lam, void *bprime, const void *const *xg_tab,
                      long long n, int L, double rho, int update_lam, cudaStream_t st);

// rule=consensus (eq-compact:solve_x): csum[s][p] = sum over the local nodes of
// local slice js (slice_of[js], local node indices [first[js], first[js] + cnt[js]), node
// order) of u + lambda/rho, in fp64.  Slices without local nodes keep their zeros.
int launch_consensus_partial(int prec, const void *u, const void *lam, double *csum, const int *slice_of,
                             const int *first, const int *cnt, int n_local_slices, long long n, double rho,
                             cudaStream_t st);
// x[m] = csum[slice][segment m] / M for each local node: to seg_tab[i] (fp32, quantized) or in
// place into the consensus image xg_tab[i] (seg_tab == null)
int launch_consensus_segment(int prec, const double *csum, const int *node_slice, void *const *xg_tab,
                             const long long *lo, const long long *len, long long max_len, float *const *seg_tab,
                             long long n, int L, int M, cudaStream_t st);

// dst_tab[i][p] = (float) src_tab[i][p]  (quantizer input = the fp32 wire format)
int launch_to_float(int prec, const void *const *src_tab, float *const *dst_tab, long long n, int L,
                    cudaStream_t st);

}  // namespace tq
