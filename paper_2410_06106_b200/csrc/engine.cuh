// engine.cuh -- the ADMM context behind the C-ABI: per-rank device state for every
// (slice, node) mapped to this rank, the outer loop of Alg. 4
// for the three consensus rules, the quantized exchange (NCCL send/recv between ranks,
// pointers within a rank) and CUDA-graph replay of whole iterations.
#pragma once
#include <map>
#include <memory>

#include "codecs.cuh"
#include "consensus.cuh"
#include "solver.cuh"
#include "transport.cuh"

namespace tq {


// exchange plan of one rank for one slice-independent graph
void exchange_plan(int M, const std::vector<int> &edges, const std::vector<int> &node_rank, int rule,
                   int rank, int world, std::vector<std::pair<int, int>> &sends,
                   std::vector<std::pair<int, int>> &recvs);

struct Ctx {
    // ---- problem
    int N = 0, n_ang = 0, n_det = 0, S = 1, M = 1, rank = 0, world = 1, prec = 0, device = 0;
    int rule = 0, split = 0;
    long long n = 0;
    std::vector<int> edges, node_rank, aoff, aidx, row_off;
    std::vector<std::vector<int>> adj;
    // ---- local (slice, node) pairs, slice-major
    std::vector<std::pair<int, int>> loc;
    std::vector<int> loc_of;  // [S*M] -> local index or -1
    int L = 0;
    DevGeom geo;
    Inner in;
    void *ALPHA = nullptr;      // [L][n] alpha_i (graph) / lambda_m (paper)
    void *XG = nullptr;         // paper / consensus: [S][n] consensus x
    double *CSUM = nullptr;     // consensus: [S][n] sum of u + lambda/rho over nodes (fp64)
    // ---- settings
    tq_params prm{};
    std::vector<double> eta1;
    bool have_params = false;
    tq_quant q{TQ_Q_NONE, 16, 10, 50, 0, 0};
    std::vector<char> sino_set;
    bool need_rhs = false;      // recompute b' from the state before the next iteration
    // sinogram-space A x kept across CG solves (graph rule: x changes only in the solve, by
    // x += alpha p, so A x += alpha A p); recomputed when stale or every AX_MAXAGE iterations
    bool ax_valid = false;
    int ax_age = 0;
    int ax_maxage = 16;         // TQ_AX_MAXAGE (0: no kept A x, the residual projection every solve)
    bool use_ax() const;
    void ax_before(int iters, cudaStream_t s);
    // ---- quantizer / exchange state (rebuilt by setup_exchange)
    bool xready = false;
    int kind_of_slice(int s) const;
    long long dct_bytes(long long nv) const;   // payload capacity of a DCT payload
    JpegWork *jw_enc() { return jenc.P ? &jenc : nullptr; }
    long long payload_len = 0;                // elements per payload (n or segment)
    struct Pay { int slice, node; uint8_t *buf; bool local; int kind; };
    std::vector<Pay> pays;                    // every payload this rank touches
    std::map<std::pair<int, int>, int> pay_of;
    std::vector<void *> owned;                // device allocations of the exchange state
    // encode batches (local payloads) and decode batches (all payloads) per kind
    struct Batch {
        int kind = 0, P = 0;
        const float **vin = nullptr;          // device tables
        uint8_t **pay = nullptr;
        int32_t **labels = nullptr;
        void **out = nullptr;
        void **dec_out = nullptr;             // K-means: fused decode outputs of the local payloads
        std::vector<int> members;             // pays index
        std::vector<const void *> conv_src;   // to_float sources
        const void **conv_src_d = nullptr;
        float **conv_dst_d = nullptr;
        bool need_conv = false;
    };
    Batch enc[3], dec[3];
    KmeansWork kmw;
    DctWork dctw;
    JpegWork jenc, jdec;                      // DCT entropy coding (q.jpeg_restart > 0)
    long long logical_fixed = 0;              // logical bytes of the fixed-size payloads
    std::vector<long long> jmult;             // per jenc payload: times it is sent per iteration
    float *fstage = nullptr;                  // float staging for quantizer inputs
    int32_t *labels_buf = nullptr;            // [L][payload_len] when keep_labels
    std::vector<int> label_row;               // local idx -> row in labels_buf or -1
    // graph rule dual tables
    const void **xh_tab = nullptr;
    int *own_slot = nullptr, *nbr_off = nullptr, *nbr_slot = nullptr;
    const void **own_ptr = nullptr, **nbr_ptr = nullptr;  // xh_tab[own_slot[i]], xh_tab[nbr_slot[k]]
    // paper / consensus rule tables
    int *cs_slice = nullptr, *cs_first = nullptr, *cs_cnt = nullptr, *node_slice = nullptr;
    void **xg_tab = nullptr;
    long long *seg_lo = nullptr, *seg_len = nullptr;
    long long seg_max = 0;
    float **seg_tab = nullptr;
    // communication between ranks (world > 1): NCCL or the in-process loopback
    std::unique_ptr<Transport> tr;
    std::vector<XferDesc> sends, recvs;       // this rank's plan entries, sorted by (peer, node)
    std::vector<SumSeg> sum_segs;             // consensus rule: the segment sums and their owners
    // ---- execution
    cudaStream_t stream = nullptr;
    // an iteration = graph segments separated by communication steps (none when world == 1)
    enum Comm { COMM_NONE = 0, COMM_REDUCE = 1, COMM_EXCHANGE = 2 };
    struct Seg { cudaGraphExec_t exec; int launches, comm; };
    std::vector<Seg> segs;
    static constexpr int MULTI = 4;
    Seg seg2{nullptr, 0, COMM_NONE};  // world == 1: MULTI iterations in one graph
    // tq_set_profiling: one graph per phase (inner | encode | decode + dual), events between
    bool profiling = false;
    std::vector<Seg> psegs;
    std::vector<cudaEvent_t> pev;    // 5 per iteration of the profiled run
    int prof_iters = 0;
    void set_profiling(bool on);
    // tq_params.stop_tol: previous iterates and the fp64 sums of the relative change
    void *XPREV = nullptr;
    double *chg_out = nullptr, *chg_part = nullptr, *chg_host = nullptr;
    unsigned *chg_cnt = nullptr;
    const void **chg_tab = nullptr;
    int chg_V = -1;
    std::vector<void *> chg_owned;
    void setup_stop_test(cudaStream_t s);
    double stop_test(cudaStream_t s);
    void free_stop_test();
    void node_bytes(int slice, int node, long long &sent, long long &recv);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    tq_stats st{};
    std::string err;

    void create(const tq_geometry &g, const tq_graph &gr, int n_slices, int rank, int world,
                const uint8_t *nccl_id, int precision, int device);
    void destroy();
    void set_params(const tq_params &p);
    void set_quant(const tq_quant &qq);
    void set_sinogram(int slice, int node, const float *d, long long len, bool on_device,
                      cudaStream_t src_s = nullptr, bool has_src_s = false);
    void run(int iters, cudaStream_t user);        // enqueue + finish
    void run_async(int iters, cudaStream_t user);  // enqueue only; finish() reports later
    void finish();  // wait for an enqueued run; its stats and divergence check (may fail)
    void get_image(int slice, int node, float *out, long long len, bool on_device);
    void get_image_async(int slice, int node, float *out, long long len, bool on_device, cudaStream_t s);
    void export_state(int slice, int node, double *buf, long long len);
    void import_state(int slice, int node, const double *buf, long long len);
    void export_labels(int slice, int node, int32_t *buf, long long len);
    long long launch_component(int component, int reps, cudaStream_t s);
    // tq_set_sinogram: NSTAGE device staging buffers filled on the upload stream; the gathers
    // into D are deferred to the stream of the next run (flush_gathers), so a new sinogram
    // costs no cross-stream round trip between two runs
    static constexpr int NSTAGE = 4;  // uploads in flight: the host may run this many calls ahead
    float *sino_stage[NSTAGE] = {};
    long long sino_stage_len[NSTAGE] = {};
    int stage_buf = 0;
    cudaEvent_t stage_copied[NSTAGE] = {}, stage_free[NSTAGE] = {};
    struct PendGather { int buf; int *pairs; int count; };
    std::vector<PendGather> pend_gathers;
    void flush_gathers(cudaStream_t s);
    cudaEvent_t gathers_done = nullptr;  // end of the last flushed gathers (on gathers_s)
    cudaStream_t gathers_s = nullptr;
    bool gathers_live = false;
    void order_after_gathers(cudaStream_t s);
    cudaEvent_t src_ready = nullptr;     // tq_set_sinogram_stream: the caller's stream position
    struct GatherMap { int *pairs; int count; };
    std::map<std::pair<int, int>, GatherMap> gather_maps;  // (slice, node) -> sinogram row pairs
    float *img_stage = nullptr;    // persistent staging of tq_get_image
    float *img_async[2] = {nullptr, nullptr};  // tq_get_image_async staging (double-buffered)
    cudaEvent_t img_ready[2] = {nullptr, nullptr}, img_done[2] = {nullptr, nullptr};
    int img_buf = 0;
    bool img_used[2] = {false, false};
    // asynchronous runs: run_done marks the end of the last enqueued run on its stream run_s
    // (valid while the run is pending); image snapshots go on that stream behind it
    cudaEvent_t run_done = nullptr;
    cudaStream_t up_stream = nullptr;  // tq_set_sinogram's host-to-device copies
    cudaStream_t run_s = nullptr;
    cudaStream_t img_s[2] = {nullptr, nullptr};  // stream of each staging buffer's snapshot
    bool pending = false;
    double *norm_host = nullptr;   // pinned [L][S_NSLOT] scalar table of the last run
    int pending_iters = 0;
    // the snapshot kernel of get_image / get_image_async into d (fp32) on `stream`
    void snapshot_image(int slice, int node, float *d, cudaStream_t s);

   private:
    void invalidate();
    void setup_exchange();
    void free_exchange();
    bool segmented() const { return rule != TQ_RULE_GRAPH; }
    int stage(int id, cudaStream_t s);  // 0: inner solves (+ Alg. 3 / partial sums), 1: x + encode,
                                        // 2: decode + dual (phase_b)
    // Node groups (DESIGN.md 6.1 "node groups"): stages 0 + 1 of the graph rule's fp32 CG path
    // captured as G independent chains over contiguous node ranges (TQ_GROUPS; by default one per
    // node, up to MAXG, for N >= 512; group 0 on the iteration's
    // stream, group g on sg[g]), joined before the exchange / dual, so one group's kernel tails,
    // CG scalar kernels and Lloyd steps overlap the others' work.  Per-node arithmetic is unchanged.
    static constexpr int MAXG = 8;
    int ngroups = 1;
    int grp_n0[MAXG] = {}, grp_cnt[MAXG] = {};
    KmeansWork kmw_g[MAXG];
    DctWork dctw_g[MAXG];
    JpegWork jenc_g[MAXG];            // tq_quant.jpeg_restart > 0: each group's entropy coder
    int grp_b0[3][MAXG] = {}, grp_bc[3][MAXG] = {};  // [codec kind][group]: the group's subrange of enc[kind]
    cudaStream_t sg[MAXG] = {};       // sg[0] unused: group 0 runs on the iteration's stream
    cudaEvent_t ev_fork = nullptr, ev_join[MAXG] = {};
    bool grouped() const;
    int stage01_grouped(cudaStream_t s);
    int stages(const std::vector<int> &ids, cudaStream_t s);  // stage() of each id, 0 + 1 grouped
    void reduce_sums(cudaStream_t s);   // consensus, world > 1: segment sums to their owners
    void exchange(cudaStream_t s);
    bool has_exchange() const;
    int phase_b(cudaStream_t s);  // decode + dual / next b'
    int prepare_rhs(cudaStream_t s);
    void enqueue(int iters, cudaStream_t user);
    void *dev_alloc(size_t bytes);
    int local(int slice, int node) const;
};

}  // namespace tq
