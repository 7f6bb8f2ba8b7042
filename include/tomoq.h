/*
 * tomoq.h -- C-ABI of libtomoq.so, the B200 (sm_100a) hot path of decentralized
 * quantized ADMM for parallel-beam tomography (arXiv 2410.06106, "PAPER.md").
 *
 * Citations: "P:n" = PAPER.md line n.  "R-k" = a reading of the paper listed in
 * DESIGN.md ("Readings").  The library never aborts: every call returns a
 * tq_status; on failure tq_last_error() (per context) / tq_last_error_global()
 * (for calls without a context) return a one-line message.  Not thread-safe per
 * context.  The caller owns every pointer it passes; the library copies what it
 * keeps and owns all device state it allocates until tq_destroy().
 *
 * Geometry (R-1..R-3): image N x N, row-major, row 0 on top, pixel centres
 * x_c = c-(N-1)/2, y_r = (N-1)/2-r; angles theta_a = pi a / n_angles;
 * bins t_j = j-(n_det-1)/2, unit spacing; n_det >= ceil(N sqrt 2) so every ray
 * through the grid is measured.  A sinogram is [angle][bin] row-major.
 * The system matrix P of P:47-77 is Joseph's: P[(a,j),p] = max(0, 1-|t_j-t_p|/m_a)/m_a,
 * t_p = x_c cos + y_r sin, m_a = max(|cos|,|sin|) with the major axis chosen by
 * the integer rule 4a in [n_angles, 3 n_angles] -> x-major.
 *
 * Precision: 0 = fp32 storage/arithmetic with fp64 dots and epilogues (production);
 * 1 = fp64 everywhere (verification mode, same kernels instantiated for double).
 * Quantizers always see the fp32-rounded iterate (the wire format, R-16/R-18).
 */
#ifndef TOMOQ_H
#define TOMOQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TQ_OK = 0,
    TQ_EINVAL = 1,     /* bad argument / geometry / graph */
    TQ_ENOMEM = 2,     /* device or host allocation failed */
    TQ_ECUDA = 3,      /* CUDA runtime error (message has the CUDA string) */
    TQ_ENCCL = 4,      /* NCCL missing or failed */
    TQ_EDIVERGED = 5,  /* some node's ||x||_2 exceeded 1e12 (SPEC "divergence guard") */
    TQ_ESTATE = 6      /* call out of order (e.g. tq_run before tq_set_sinogram) */
} tq_status;

typedef struct tq_ctx tq_ctx;

typedef struct {
    int32_t image_side;  /* N, multiple of 8, >= 8 */
    int32_t n_angles;    /* angles evenly spaced in [0, pi) */
    int32_t n_det;       /* detector bins, >= ceil(N sqrt 2) */
    int32_t projector;   /* TQ_PROJ_JOSEPH (R-1, default) or TQ_PROJ_SIDDON: exact intersection
                            lengths P_ji = |ray j inside pixel i| (SURVEY NEXT-3,
                            R-26: trig exact at 0 and pi/2, a ray on a pixel edge counts half
                            in each of the two pixels) */
    const double *angles_rad; /* NULL: theta_a = pi a / n_angles ("evenly distributed from
                            0 to 180 degrees"), major axis by the integer rule above (R-3).
                            Else n_angles explicit angles in [0, pi) (radians, any order, copied),
                            ray (theta, t) = {x cos + y sin = t} as P:42; major axis x iff
                            |sin theta| >= |cos theta| in fp64 (R-3 for explicit lists); Siddon
                            takes trig exact where theta == 0 or theta == fl64(pi/2) (R-26). */
} tq_geometry;

enum { TQ_PROJ_JOSEPH = 0, TQ_PROJ_SIDDON = 1 };

enum { TQ_SPLIT_ROUND_ROBIN = 0, TQ_SPLIT_CONTIGUOUS = 1 };
enum { TQ_RULE_GRAPH = 0, TQ_RULE_PAPER = 1, TQ_RULE_CONSENSUS = 2 };
enum { TQ_INNER_GD = 0, TQ_INNER_CG = 1 };
enum { TQ_Q_NONE = 0, TQ_Q_KMEANS = 1, TQ_Q_DCT = 2, TQ_Q_ALTERNATE = 3 };

/* The communication graph of ONE slice (every slice uses the same graph).
 * rule TQ_RULE_GRAPH: decentralized consensus ADMM over the edges (R-7, default).
 * rule TQ_RULE_PAPER: the segment-owner dADMM of P:158-166 (edges unused; every
 * node needs every segment -- an all-gather).
 * rule TQ_RULE_CONSENSUS: the standard consensus ADMM of P:121-131 with x sharded in
 * the same segments: x[m] = mean over all nodes of (u + lambda/rho)[m] (an all-reduce
 * of per-rank partial sums across ranks), Q per segment, all-gather. */
typedef struct {
    int32_t n_nodes;          /* M ADMM nodes per slice, 1 <= M <= n_angles */
    int32_t n_edges;
    const int32_t *edges;     /* 2*n_edges node ids, undirected, no self loops / duplicates;
                                 every node degree <= 64 (TQ_EINVAL otherwise) */
    int32_t angle_split;      /* TQ_SPLIT_* (P:319-320 round-robin; R-5 contiguous) */
    const int32_t *node_rank; /* [n_nodes] rank owning node i (all slices); NULL => i mod world */
    int32_t rule;             /* TQ_RULE_* */
} tq_graph;

typedef struct {
    double rho;            /* penalty rho > 0 */
    int32_t inner;         /* TQ_INNER_GD (Alg. 2) or TQ_INNER_CG (R-8) */
    int32_t e1;            /* inner steps E1 >= 0 */
    const double *eta1;    /* [n_nodes] GD step per node, or NULL => 1/(2 a_i N + c_i) (R-8) */
    int32_t e2;            /* Alg. 3 steps (paper rule) */
    double eta2;           /* Alg. 3 step, 0 < eta2 rho < 2 */
    double stop_tol;       /* 0: run exactly the requested iterations.  > 0: the stopping
                              criterion of P:330 ("stopping criterion of 1e-6", R-13): after
                              every iteration k the relative change
                                r_k = max ||x^{k+1} - x^k||_2 / ||x^{k+1}||_2   (0/0 := 0)
                              over the iterates -- graph rule: every node's private x_i; paper /
                              consensus rule: the consensus x of every slice -- maximised over
                              ranks; the run stops after the first iteration with r_k <= stop_tol.
                              Every iteration then synchronises the host (tq_run_async becomes
                              blocking).  tq_stats.iters_last_run / rel_change_last report it. */
} tq_params;

typedef struct {
    int32_t kind;         /* TQ_Q_*; ALTERNATE = K-means on even slices, DCT on odd (R-20) */
    int32_t k;            /* K-means clusters, 1..256 (Alg. 5) */
    int32_t lloyd_iters;  /* Lloyd iterations after the quantile init (R-16) */
    int32_t quality;      /* DCT quality 1..100, IJG scaling of the Annex K table (R-18) */
    int32_t keep_labels;  /* 1: keep the last K-means labels for tq_export_labels (parity) */
    int32_t jpeg_restart; /* DCT payloads: 0 = plain int16 coefficients; R >= 1 = baseline JPEG
                             Huffman entropy coding (T.81 Annex F, Annex K luminance tables)
                             with an RSTm marker every R 8x8 blocks;
                             lossless, so iterates are unchanged; payload bytes shrink */
} tq_quant;

typedef struct {
    int64_t iters;                 /* ADMM iterations run so far */
    int32_t local_nodes;           /* (slice, node) pairs on this rank */
    int32_t world;
    int64_t payload_bytes_logical; /* last iteration: sum over local nodes of bytes each
                                      node sent (graph: deg x payload; paper: (M-1) x segment) */
    int64_t nccl_bytes_sent;       /* last iteration, this rank, over NCCL */
    int64_t nccl_bytes_recv;
    int64_t kernel_launches;       /* kernels launched by the last tq_run (all iterations) */
    double ms_last_run;            /* device time of the last tq_run (CUDA events) */
    int64_t iters_last_run;        /* iterations the last run performed (fewer than requested
                                      when tq_params.stop_tol stopped it) */
    double rel_change_last;        /* r_k of the last iteration (stop_tol > 0), else -1 */
    int32_t phase_valid;           /* 1: phase_ms holds the last run's phases (tq_set_profiling) */
    int32_t node_groups;           /* concurrent node groups of the last run's iteration graph: 1, or
                                      TQ_GROUPS / its default where they apply (see TQ_GROUPS below;
                                      DESIGN.md 6.1 "node groups") */
    double phase_ms[4];            /* device ms of the last run, summed over its iterations:
                                      [0] inner solves (A3: the E1 CG / GD steps of every local
                                      node; plus Alg. 3 / the consensus partial sums and their
                                      cross-rank reduction), [1] encode (A5 / A6 quantizers),
                                      [2] exchange (A7), [3] decode + dual / next b' (A4) */
} tq_stats;

/* ---------------------------------------------------------------- context API */
/* Transport ids for world > 1 (the exchange of P:188 / P:248-252 between ranks).
 * tq_nccl_unique_id: an NCCL unique id (rank 0 creates it, the caller broadcasts it); one
 *   process per GPU; payloads move with ncclSend / ncclRecv, the consensus sums with ncclReduce.
 * tq_loopback_id: an in-process world: the `world` contexts created with it live in THIS
 *   process (one host thread per rank, calling the same sequence of context calls, as NCCL
 *   ranks would), on one GPU or several.  Each receiver pulls every planned payload with its
 *   own cudaMemcpyAsync from the sender's buffer; the consensus segment sums are a fixed-order
 *   (rank 0, 1, ...) kernel at the segment owner.  A rank that does not reach a rendezvous
 *   within TQ_LOOPBACK_TIMEOUT_S seconds (default 120) makes every rank fail with TQ_ENCCL.
 *   Results equal the world == 1 run bit for bit (graph and paper rules). */
tq_status tq_nccl_unique_id(uint8_t id[128]);
tq_status tq_loopback_id(uint8_t id[128]);

/* One context per rank, owning every (slice, node) mapped to this rank.
 * nccl_id: a transport id (above) from rank 0, the same on every rank; NULL if world == 1.
 * device: CUDA device ordinal to use. */
tq_status tq_create(const tq_geometry *geom, const tq_graph *graph, int32_t n_slices,
                    int32_t rank, int32_t world, const uint8_t *nccl_id, int32_t precision,
                    int32_t device, tq_ctx **out);
tq_status tq_set_params(tq_ctx *ctx, const tq_params *p);
tq_status tq_set_quantizer(tq_ctx *ctx, const tq_quant *q);

/* Sinogram of one slice.  node >= 0: that node's shard ([a_node][n_det], its angles in
 * increasing order); node == -1: the full slice sinogram [n_angles][n_det] and the
 * library keeps the rows of its local nodes.  Ignored for nodes not on this rank.
 * len is in floats; on_device: d is a device pointer, which must hold its final values when
 * the call is made (no write to it still pending on any stream -- use tq_set_sinogram_stream
 * for a buffer written asynchronously).  Returns once d has been copied (the caller may reuse
 * it); the new rows replace the old ones after any enqueued run. */
tq_status tq_set_sinogram(tq_ctx *ctx, int32_t slice, int32_t node, const float *d,
                          int64_t len, int32_t on_device);
/* The same for a device buffer d written on the caller's `stream` (NULL = legacy default
 * stream): the library's copy of d is ordered after everything already enqueued on `stream`
 * (an event recorded there).  Returns once d has been copied. */
tq_status tq_set_sinogram_stream(tq_ctx *ctx, int32_t slice, int32_t node, const float *d,
                                 int64_t len, void *stream);

/* Enqueue `iters` ADMM iterations (Alg. 4) on `stream` (NULL = the
 * context's own stream) and wait for them; returns TQ_EDIVERGED if any node's norm
 * exceeds 1e12 after the last iteration. */
tq_status tq_run(tq_ctx *ctx, int32_t iters, void *stream);
/* The same iterations, enqueued and not waited for: returns once they are on `stream`.
 * tq_set_sinogram, tq_get_image_async and a further tq_run_async may follow at once (they
 * order themselves after it on the device); every other call first waits for it.  Its
 * statistics and divergence check (TQ_EDIVERGED) are reported by the first call that waits
 * -- tq_wait, tq_run, tq_get_image, tq_get_stats, tq_export_state, ... */
tq_status tq_run_async(tq_ctx *ctx, int32_t iters, void *stream);
/* Wait for the last enqueued run; TQ_EDIVERGED as tq_run.  TQ_OK at once if none. */
tq_status tq_wait(tq_ctx *ctx);

/* node >= 0: that node's private iterate (graph) / u_m (paper) -- must be local.
 * node == -1: graph rule: mean over the slice's nodes of x_i (all must be local, R-22);
 *             paper rule: the consensus x.  out: N*N floats (host or device). */
tq_status tq_get_image(tq_ctx *ctx, int32_t slice, int32_t node, float *out, int64_t len,
                       int32_t on_device);
/* The same image, enqueued instead of waited for: the library snapshots it into one of two
 * device staging buffers (on its own stream, after the last tq_run) and enqueues the copy to
 * `out` on `stream` (a CUDA stream of the caller's; NULL = the legacy default stream).  The
 * call returns at once; `out` (page-locked host or device memory) holds the image once
 * `stream` has completed the copy, and must stay valid until then.  A third call waits for
 * the copy of the first before reusing its staging buffer, so at most two are in flight --
 * the next tq_run can overlap the transfer. */
tq_status tq_get_image_async(tq_ctx *ctx, int32_t slice, int32_t node, float *out, int64_t len,
                             int32_t on_device, void *stream);

/* State of one local node as 3*N*N doubles: graph rule [x_i | alpha_i | xhat_i];
 * paper rule [u_m | lambda_m | x].  Import recomputes the next right-hand side. */
tq_status tq_export_state(tq_ctx *ctx, int32_t slice, int32_t node, double *buf, int64_t len);
tq_status tq_import_state(tq_ctx *ctx, int32_t slice, int32_t node, const double *buf, int64_t len);
/* Pre-quantization labels of the last encode of a local node (K-means only), int32 [N*N]. */
tq_status tq_export_labels(tq_ctx *ctx, int32_t slice, int32_t node, int32_t *buf, int64_t len);

/* Profiling hook: enqueue `reps` launches of one component of the iteration over all
 * local nodes on `stream` (no synchronisation), with the context's own buffers, so a
 * caller can time it with events on that stream.  Components: 0 forward projector
 * S = A P, 1 backprojector with the CG epilogue Q = A^T S + c P, 2 forward residual
 * S = D - A X, 3 the K-means encode of the quantized slices, 4 the DCT encode,
 * 5 the consensus/dual kernel without the dual update (b' only).  Overwrites only
 * scratch (S, Q, payloads and the decoded public values of local K-means payloads,
 * b' is recomputed identically); x and alpha are unchanged.
 * Returns TQ_EINVAL for a component the context does not have.  *units = algorithmic
 * work per launch (voxel-updates for 0-2, elements for 3-5). */
tq_status tq_launch_component(tq_ctx *ctx, int32_t component, int32_t reps, void *stream,
                              int64_t *units);

tq_status tq_get_stats(const tq_ctx *ctx, tq_stats *out);
/* Environment knob read by tq_create: TQ_AX_MAXAGE (default 16) -- the graph-rule CG keeps the
 * residual's A x in sinogram space across inner solves (A x += alpha A p; R-8) and
 * recomputes it by a forward projection when stale and at least every TQ_AX_MAXAGE iterations;
 * 0 projects x in every solve (the oracle's order of operations).
 * Environment knob read when the exchange state is built (first run after tq_create /
 * tq_set_quantizer): TQ_GROUPS (at most 8; 1 disables; default one group per local node, up to
 * 8, for N >= 512, else 1) -- with the graph rule and fp32, the inner solves and encodes (K-means,
 * DCT, JPEG-coded DCT) of an iteration run as that many concurrent launch chains over contiguous
 * node ranges, joined before the exchange.  Results are bitwise those of one chain (per-node arithmetic is unchanged);
 * tq_stats.node_groups reports what the last run used. */

/* Debug aid (no compute-sanitizer on the GPU pool): with TQ_GUARD=1 in the environment of the
 * process, every device allocation of the library carries 256-byte guard bands (checked after
 * every run: TQ_ECUDA on an out-of-bounds write) and starts poisoned with 0xff bytes, so reads
 * of never-written memory change results.  This call checks every live allocation's guards now
 * (TQ_OK when TQ_GUARD is unset). */
tq_status tq_debug_guard_check(void);
/* Transport self-check (the A7 exchange layer alone): creates the transport of
 * `id` (tq_nccl_unique_id or tq_loopback_id) for (rank, world) on `device`, and `rounds` times
 * runs each of its operations on a synthetic plan: every rank sends `bytes` bytes to every rank
 * INCLUDING ITSELF (so NCCL's grouped ncclSend / ncclRecv, ncclReduce and ncclAllReduce all run
 * even at world == 1, e.g. on a one-GPU box, where NCCL refuses two ranks per device), then the
 * ranks' `n_doubles`-element fp64 buffers are summed onto segment owners (segment g of `world`,
 * owner g, as the consensus rule's reduce), then the maximum of the rank ids is taken.  Every
 * received byte and owned sum is compared with its exact host value.  Called by every rank of
 * the world (loopback: one host thread per rank of this process).  Blocking; allocates and
 * frees its own buffers.  TQ_OK when everything matched; TQ_ENCCL (message in
 * tq_last_error_global) on a mismatch or a transport error; TQ_EINVAL on bad arguments. */
tq_status tq_debug_transport_check(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                                   int64_t bytes, int64_t n_doubles, int32_t rounds);
/* Phase timing (tq_stats.phase_ms): on = 1 makes later runs launch each phase as its own CUDA
 * graph with timing events in between (slightly slower than the default whole-iteration
 * graph; off by default).  Waits for an enqueued run. */
tq_status tq_set_profiling(tq_ctx *ctx, int32_t on);
/* Bytes one local node (slice, node) sent and received in the last iteration, as the method
 * moves them (the per-node communication of P:248-252, independent of where nodes are placed):
 * graph rule: sent = deg_i x its payload, received = the sum of its neighbours' payloads;
 * paper rule: sent = (M-1) x its segment payload, received = the other M-1 segment payloads
 * (with TQ_Q_NONE: sent + received = 2 (M-1)/M X, X = the image bytes); consensus rule:
 * the paper rule's segment traffic plus the fp64 partial sums (8 B per element) of the other
 * nodes' segments sent to their owners and received from the other M-1 nodes for its own.
 * Entropy-coded DCT payloads count their coded size (header included).  Waits for a run. */
tq_status tq_get_node_bytes(tq_ctx *ctx, int32_t slice, int32_t node, int64_t *sent, int64_t *recv);
const char *tq_last_error(const tq_ctx *ctx);
const char *tq_last_error_global(void);
void tq_destroy(tq_ctx *ctx);

/* ---------------------------------------------------------------- host-side plans
 * Pure host functions (no GPU needed). */
/* Angle partition of P:319-320 / R-5: offsets[n_nodes+1], idx[n_angles]. */
tq_status tq_partition_angles(int32_t n_angles, int32_t n_nodes, int32_t split,
                              int32_t *offsets, int32_t *idx);
/* Exchange plan of `rank` for one iteration: sends = (node, peer) pairs this rank
 * sends node's payload to; recvs = (node, peer) pairs it receives.  Capacity in
 * pairs; *n_* returns the counts (TQ_EINVAL if capacity is too small). */
tq_status tq_exchange_plan(const tq_graph *graph, int32_t rank, int32_t world,
                           int32_t *sends, int32_t cap_sends, int32_t *n_sends,
                           int32_t *recvs, int32_t cap_recvs, int32_t *n_recvs);
/* Payload bytes of one encoded vector of n elements (Q kind for the slice). */
int64_t tq_payload_bytes(int32_t kind, int32_t k, int64_t n, int32_t precision);

/* ---------------------------------------------------------------- stateless kernels
 * Device pointers, caller-owned; precision selects float (0) / double (1) elements;
 * stream NULL = default stream; calls are asynchronous. */
/* sino[k][j] = (A img)[(sel[k], j)]  (Eq. 2). sel: host array of n_sel angle ids. */
tq_status tq_project(const tq_geometry *g, const int32_t *sel, int32_t n_sel, const void *img,
                     void *sino, int32_t precision, void *stream);
/* img = A^T sino over the selected angles (the transpose of Alg. 2 line 3). */
tq_status tq_backproject(const tq_geometry *g, const int32_t *sel, int32_t n_sel,
                         const void *sino, void *img, int32_t precision, void *stream);
/* One node's inner solve of min 1/2||A x - d||^2 + c/2||x||^2 - b'^T x, E1 GD (eta) or
 * CG steps, warm start x (in/out).  d: [n_sel][n_det]. Synchronous. */
tq_status tq_local_solve(const tq_geometry *g, const int32_t *sel, int32_t n_sel,
                         const void *d, const void *bprime, double c, int32_t inner,
                         int32_t e1, double eta, void *x, int32_t precision, void *stream);
/* K-means encode (Alg. 5 made exact, R-16) of n fp32 values: centers[k] fp32,
 * planes[ceil(n/32) * ceil(log2 k)] uint32 bit-planes (group-major), labels (int32,
 * optional, may be NULL). */
tq_status tq_kmeans_encode(const float *v, int64_t n, int32_t k, int32_t iters, float *centers,
                           uint32_t *planes, int32_t *labels, void *stream);
tq_status tq_kmeans_decode(const float *centers, const uint32_t *planes, int64_t n, int32_t k,
                           float *out, void *stream);
/* DCT codec (R-18) of a rows x cols fp32 array (8 | rows, 8 | cols): coef[rows*cols] int16
 * in [block][u][v] order, minmax[2] fp32. */
tq_status tq_dct_encode(const float *v, int32_t rows, int32_t cols, int32_t quality,
                        int16_t *coef, float *minmax, void *stream);
tq_status tq_dct_decode(const int16_t *coef, const float *minmax, int32_t rows, int32_t cols,
                        int32_t quality, float *out, void *stream);
/* Baseline JPEG Huffman entropy coding (ITU-T T.81 Annex C code
 * generation, F.1.2 DC-difference / AC run-length coding with ZRL and EOB, F.1.2.3 byte
 * stuffing and 1-fill, F.1.4.4 RSTm markers every `restart` >= 1 blocks with the DC
 * predictor reset; Annex K Tables K.3 / K.5 luminance Huffman tables; R-25) of
 * n_blocks 8x8 blocks of coefficients in the order tq_dct_encode writes them (raster
 * blocks, natural order inside a block).  Device pointers, caller-owned.
 * Encode writes the entropy-coded segment (no JPEG headers) to out[cap] and its length to
 * *nbytes (host pointer); TQ_EINVAL if a value lies outside the baseline categories (DC
 * difference > 11 bits, AC > 10 bits), or if the stream would exceed 2 bytes per
 * coefficient or cap.  Decode reads nbytes of such a segment and writes the
 * coefficients; TQ_EINVAL on a malformed stream (bad code, missing or misnumbered RSTm,
 * truncated data).  Both synchronise the stream. */
tq_status tq_jpeg_encode(const int16_t *coef, int64_t n_blocks, int32_t restart, uint8_t *out,
                         int64_t cap, int64_t *nbytes, void *stream);
tq_status tq_jpeg_decode(const uint8_t *in, int64_t nbytes, int64_t n_blocks, int32_t restart,
                         int16_t *coef, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TOMOQ_H */
