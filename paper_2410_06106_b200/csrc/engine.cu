// engine.cu -- see engine.cuh.
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>

#include <nvtx3/nvToolsExt.h>

#include "engine.cuh"

namespace tq {

// NVTX ranges (header-only NVTX v3; free when no tool is attached): host phases of the API
// and, around each graph launch, the ADMM phase its kernels belong to, so `ncu --nvtx
// --nvtx-include "tq:encode/"` (or a timeline tool) selects one phase's kernels
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

[[noreturn]] void fail(tq_status code, const std::string &msg) { throw Error{code, msg}; }

// ---------------------------------------------------------------- exchange plan
// graph rule: a node's payload goes to every rank owning one of its neighbours
// (deduplicated per (node, peer)); paper / consensus rule: every node's segment
// payload goes to every other rank that owns nodes (the all-gather of P:188).  Sorted by
// (peer, node) so both ends of every pair post matching send/recv sequences.
void exchange_plan(int M, const std::vector<int> &edges, const std::vector<int> &node_rank, int rule,
                   int rank, int world, std::vector<std::pair<int, int>> &sends,
                   std::vector<std::pair<int, int>> &recvs) {
    std::set<std::pair<int, int>> S, R;  // (peer, node)
    if (rule == TQ_RULE_GRAPH) {
        for (size_t e = 0; e + 1 < edges.size(); e += 2) {
            const int i = edges[e], j = edges[e + 1];
            const int ri = node_rank[i], rj = node_rank[j];
            if (ri == rj) continue;
            if (ri == rank) { S.insert({rj, i}); R.insert({rj, j}); }
            if (rj == rank) { S.insert({ri, j}); R.insert({ri, i}); }
        }
    } else {
        std::set<int> owners(node_rank.begin(), node_rank.end());
        for (int m = 0; m < M; m++) {
            const int rm = node_rank[m];
            for (int r : owners) {
                if (r == rm) continue;
                if (rm == rank) S.insert({r, m});
                if (r == rank) R.insert({rm, m});
            }
        }
    }
    (void)world;
    sends.clear();
    recvs.clear();
    for (auto &p : S) sends.push_back({p.second, p.first});
    for (auto &p : R) recvs.push_back({p.second, p.first});
}

// ---------------------------------------------------------------- small kernels
namespace {

// row pairs[2 r] of src -> row pairs[2 r + 1] of dst
template <typename T>
__global__ void gather_rows(const float *src, const int *pairs, T *dst, int n_det) {
    const int r = blockIdx.y;
    const float *s = src + (long long)pairs[2 * r] * n_det;
    T *d = dst + (long long)pairs[2 * r + 1] * n_det;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_det; j += gridDim.x * blockDim.x) d[j] = (T)s[j];
}

template <typename T>
__global__ void mean_rows(const T *base, int rows, long long n, float *out) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < rows; r++) s += (double)base[(long long)r * n + p];
        out[p] = (float)(s / rows);
    }
}

}  // namespace

// ---------------------------------------------------------------- context
int Ctx::local(int slice, int node) const {
    if (slice < 0 || slice >= S || node < 0 || node >= M) return -1;
    return loc_of[(size_t)slice * M + node];
}

long long Ctx::dct_bytes(long long nv) const {
    return q.jpeg_restart > 0 ? jpeg_payload_bytes(nv) : dct_payload_bytes(nv);
}

int Ctx::kind_of_slice(int s) const {
    if (q.kind == TQ_Q_ALTERNATE) return (s % 2 == 0) ? TQ_Q_KMEANS : TQ_Q_DCT;
    return q.kind;
}

void *Ctx::dev_alloc(size_t bytes) {
    void *p = nullptr;
    TQ_CHECK_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    TQ_CHECK_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
    owned.push_back(p);
    return p;
}

void Ctx::create(const tq_geometry &g, const tq_graph &gr, int n_slices, int rank_, int world_,
                 const uint8_t *nccl_id, int precision, int device_) {
    N = g.image_side; n_ang = g.n_angles; n_det = g.n_det;
    if (const char *e = getenv("TQ_AX_MAXAGE")) ax_maxage = std::max(0, atoi(e));
    TQ_REQUIRE(N >= 8 && N % 8 == 0, "image_side must be a positive multiple of 8");
    TQ_REQUIRE(N <= 16384, "image_side too large");
    TQ_REQUIRE(n_ang >= 1, "n_angles must be >= 1");
    TQ_REQUIRE((long long)n_det * n_det >= 2LL * N * N, "n_det must be >= ceil(N sqrt 2)");
    TQ_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (fp32) or 1 (fp64)");
    TQ_REQUIRE(n_slices >= 1, "n_slices must be >= 1");
    TQ_REQUIRE(world_ >= 1 && rank_ >= 0 && rank_ < world_, "bad rank/world");
    M = gr.n_nodes;
    TQ_REQUIRE(M >= 1 && M <= n_ang, "n_nodes must be in [1, n_angles]");
    TQ_REQUIRE(gr.rule == TQ_RULE_GRAPH || gr.rule == TQ_RULE_PAPER || gr.rule == TQ_RULE_CONSENSUS, "bad rule");
    TQ_REQUIRE(gr.angle_split == TQ_SPLIT_ROUND_ROBIN || gr.angle_split == TQ_SPLIT_CONTIGUOUS, "bad split");
    TQ_REQUIRE(gr.n_edges >= 0 && (gr.n_edges == 0 || gr.edges), "edges missing");
    S = n_slices; rank = rank_; world = world_; prec = precision; device = device_;
    rule = gr.rule; split = gr.angle_split;
    n = (long long)N * N;
    edges.assign(gr.edges, gr.edges + 2 * (size_t)gr.n_edges);
    adj.assign(M, {});
    std::set<std::pair<int, int>> seen;
    for (int e = 0; e < gr.n_edges; e++) {
        const int i = edges[2 * e], j = edges[2 * e + 1];
        TQ_REQUIRE(i >= 0 && i < M && j >= 0 && j < M && i != j, "edge endpoints out of range or self loop");
        TQ_REQUIRE(seen.insert({std::min(i, j), std::max(i, j)}).second, "duplicate edge");
        adj[i].push_back(j);
        adj[j].push_back(i);
    }
    for (int i = 0; i < M; i++)
        TQ_REQUIRE((int)adj[i].size() <= TQ_MAX_DEGREE, "graph rule: node degree must be <= 64");
    if (rule == TQ_RULE_GRAPH && M > 1) {  // connected graph (consensus reaches every node)
        std::vector<int> stack{0}, vis(M, 0);
        vis[0] = 1;
        while (!stack.empty()) {
            const int u = stack.back();
            stack.pop_back();
            for (int v : adj[u]) if (!vis[v]) { vis[v] = 1; stack.push_back(v); }
        }
        for (int i = 0; i < M; i++) TQ_REQUIRE(vis[i], "graph rule needs a connected graph");
    }
    node_rank.resize(M);
    for (int i = 0; i < M; i++) {
        node_rank[i] = gr.node_rank ? gr.node_rank[i] : i % world;
        TQ_REQUIRE(node_rank[i] >= 0 && node_rank[i] < world, "node_rank out of range");
    }
    partition_angles(n_ang, M, split, aoff, aidx);
    partition_rows(N, M, row_off);
    loc_of.assign((size_t)S * M, -1);
    std::vector<std::vector<int>> angles;
    for (int s = 0; s < S; s++)
        for (int m = 0; m < M; m++)
            if (node_rank[m] == rank) {
                loc_of[(size_t)s * M + m] = (int)loc.size();
                loc.push_back({s, m});
                angles.push_back(std::vector<int>(aidx.begin() + aoff[m], aidx.begin() + aoff[m + 1]));
            }
    L = (int)loc.size();
    TQ_CHECK_CUDA(cudaSetDevice(device));
    TQ_CHECK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    TQ_CHECK_CUDA(cudaStreamCreateWithFlags(&up_stream, cudaStreamNonBlocking));
    TQ_CHECK_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    for (int g = 1; g < MAXG; g++) {
        TQ_CHECK_CUDA(cudaStreamCreateWithFlags(&sg[g], cudaStreamNonBlocking));
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&ev_join[g], cudaEventDisableTiming));
    }
    TQ_CHECK_CUDA(cudaEventCreate(&ev0));
    TQ_CHECK_CUDA(cudaEventCreate(&ev1));
    TQ_CHECK_CUDA(cudaEventCreateWithFlags(&run_done, cudaEventDisableTiming));
    TQ_CHECK_CUDA(cudaEventCreateWithFlags(&gathers_done, cudaEventDisableTiming));
    TQ_CHECK_CUDA(cudaEventCreateWithFlags(&src_ready, cudaEventDisableTiming));
    for (int b = 0; b < NSTAGE; b++) {
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&stage_copied[b], cudaEventDisableTiming));
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&stage_free[b], cudaEventDisableTiming));
    }
    TQ_REQUIRE(g.projector == TQ_PROJ_JOSEPH || g.projector == TQ_PROJ_SIDDON, "bad projector");
    check_angles(g.angles_rad, n_ang);
    geo.init(N, n_ang, n_det, g.projector, g.angles_rad);
    in.init(prec, geo, angles);
    const size_t es = prec ? 8 : 4;
    TQ_CHECK_CUDA(cudaMalloc(&ALPHA, std::max<size_t>(16, es * n * L)));
    TQ_CHECK_CUDA(cudaMemset(ALPHA, 0, std::max<size_t>(16, es * n * L)));
    if (segmented()) {
        TQ_CHECK_CUDA(cudaMalloc(&XG, es * n * S));
        TQ_CHECK_CUDA(cudaMemset(XG, 0, es * n * S));
    }
    if (rule == TQ_RULE_CONSENSUS) {  // every rank joins the segment reductions, even without nodes
        TQ_CHECK_CUDA(cudaMalloc(&CSUM, sizeof(double) * n * S));
        TQ_CHECK_CUDA(cudaMemset(CSUM, 0, sizeof(double) * n * S));
    }
    if (world > 1) tr = make_transport(nccl_id, rank, world, device);
    sino_set.assign(L, 0);
    st.local_nodes = L;
    st.world = world;
}

void Ctx::invalidate() {
    for (auto &g : segs) cudaGraphExecDestroy(g.exec);
    segs.clear();
    for (auto &g : psegs) cudaGraphExecDestroy(g.exec);
    psegs.clear();
    free_stop_test();
    if (seg2.exec) cudaGraphExecDestroy(seg2.exec);
    seg2 = Seg{nullptr, 0, COMM_NONE};
}

void Ctx::free_exchange() {
    invalidate();
    for (void *p : owned) cudaFree(p);
    owned.clear();
    kmw.release();
    for (auto &w : kmw_g) w.release();
    for (auto &w : dctw_g) w.release();
    for (auto &w : jenc_g) w.release();
    ngroups = 1;
    dctw.release();
    jenc.release();
    jdec.release();
    jmult.clear();
    logical_fixed = 0;
    pays.clear();
    pay_of.clear();
    for (auto &b : enc) b = Batch();
    for (auto &b : dec) b = Batch();
    sends.clear(); recvs.clear(); sum_segs.clear();
    label_row.clear();
    fstage = nullptr; labels_buf = nullptr; xh_tab = nullptr; own_slot = nbr_off = nbr_slot = nullptr;
    own_ptr = nbr_ptr = nullptr;
    xg_tab = nullptr; seg_lo = nullptr; seg_len = nullptr; seg_tab = nullptr;
    cs_slice = cs_first = cs_cnt = node_slice = nullptr;
    xready = false;
}

void Ctx::destroy() {
    if (run_done) cudaEventSynchronize(run_done);
    pending = false;
    pend_gathers.clear();
    if (stream) cudaStreamSynchronize(stream);
    if (up_stream) cudaStreamSynchronize(up_stream);
    free_exchange();
    in.release();
    geo.release();
    if (ALPHA) cudaFree(ALPHA);
    if (XG) cudaFree(XG);
    if (CSUM) cudaFree(CSUM);
    ALPHA = XG = nullptr;
    CSUM = nullptr;
    for (int b = 0; b < NSTAGE; b++) {
        if (sino_stage[b]) cudaFree(sino_stage[b]);
        sino_stage[b] = nullptr;
        sino_stage_len[b] = 0;
    }
    for (auto &g : gather_maps)
        if (g.second.pairs) cudaFree(g.second.pairs);
    gather_maps.clear();
    if (img_stage) cudaFree(img_stage);
    for (int b = 0; b < 2; b++) {
        if (img_done[b]) cudaEventSynchronize(img_done[b]);
        if (img_async[b]) cudaFree(img_async[b]);
        if (img_ready[b]) cudaEventDestroy(img_ready[b]);
        if (img_done[b]) cudaEventDestroy(img_done[b]);
        img_async[b] = nullptr; img_ready[b] = img_done[b] = nullptr;
    }
    img_stage = nullptr;
    tr.reset();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (cudaEvent_t e : pev) cudaEventDestroy(e);
    pev.clear();
    if (run_done) cudaEventDestroy(run_done);
    run_done = nullptr;
    if (gathers_done) cudaEventDestroy(gathers_done);
    gathers_done = nullptr;
    if (src_ready) cudaEventDestroy(src_ready);
    src_ready = nullptr;
    for (int b = 0; b < NSTAGE; b++) {
        if (stage_copied[b]) cudaEventDestroy(stage_copied[b]);
        if (stage_free[b]) cudaEventDestroy(stage_free[b]);
        stage_copied[b] = stage_free[b] = nullptr;
    }
    if (norm_host) cudaFreeHost(norm_host);
    norm_host = nullptr;
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    if (up_stream) cudaStreamDestroy(up_stream);
    up_stream = nullptr;
    for (int g = 1; g < MAXG; g++) {
        if (sg[g]) cudaStreamDestroy(sg[g]);
        if (ev_join[g]) cudaEventDestroy(ev_join[g]);
        sg[g] = nullptr;
        ev_join[g] = nullptr;
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    ev_fork = nullptr;
}

void Ctx::set_params(const tq_params &p) {
    finish();
    ax_valid = false;  // e.g. GD steps may have moved x without the kept A x
    TQ_REQUIRE(p.rho > 0.0 && std::isfinite(p.rho), "rho must be > 0");
    TQ_REQUIRE(p.inner == TQ_INNER_GD || p.inner == TQ_INNER_CG, "inner must be GD or CG");
    TQ_REQUIRE(p.e1 >= 0 && p.e1 <= 100000, "e1 out of range");
    TQ_REQUIRE(p.stop_tol >= 0.0 && std::isfinite(p.stop_tol), "stop_tol must be finite and >= 0");
    if (rule == TQ_RULE_PAPER) {
        TQ_REQUIRE(p.e2 >= 0, "e2 must be >= 0");
        TQ_REQUIRE(p.eta2 * p.rho > 0.0 && p.eta2 * p.rho < 2.0, "need 0 < eta2 rho < 2 (Alg. 3 contraction)");
    }
    prm = p;
    eta1.clear();
    if (p.eta1) eta1.assign(p.eta1, p.eta1 + M);
    prm.eta1 = nullptr;
    std::vector<double> c(L), eta(L);
    for (int i = 0; i < L; i++) {
        const int m = loc[i].second;
        c[i] = rule == TQ_RULE_GRAPH ? 2.0 * p.rho * (double)adj[m].size() : p.rho;
        const int a = aoff[m + 1] - aoff[m];
        eta[i] = eta1.empty() ? 1.0 / (2.0 * a * N + c[i]) : eta1[m];  // R-8
    }
    if (L) {
        TQ_CHECK_CUDA(cudaMemcpy(in.cnode, c.data(), sizeof(double) * L, cudaMemcpyHostToDevice));
        TQ_CHECK_CUDA(cudaMemcpy(in.eta, eta.data(), sizeof(double) * L, cudaMemcpyHostToDevice));
    }
    // a change of rho (or of c_i) after iterations ran: b' of the current state is rebuilt with
    // the new values before the next iteration (as tq_import_state does)
    if (have_params) need_rhs = true;
    have_params = true;
    invalidate();
}

void Ctx::set_quant(const tq_quant &qq) {
    finish();
    TQ_REQUIRE(qq.kind >= TQ_Q_NONE && qq.kind <= TQ_Q_ALTERNATE, "bad quantizer kind");
    const bool km = qq.kind == TQ_Q_KMEANS || qq.kind == TQ_Q_ALTERNATE;
    const bool dc = qq.kind == TQ_Q_DCT || qq.kind == TQ_Q_ALTERNATE;
    if (km) TQ_REQUIRE(qq.k >= 1 && qq.k <= 256 && qq.lloyd_iters >= 0, "kmeans: k in [1,256], lloyd >= 0");
    if (dc) TQ_REQUIRE(qq.quality >= 1 && qq.quality <= 100, "dct: quality in [1,100]");
    TQ_REQUIRE(qq.jpeg_restart >= 0 && qq.jpeg_restart <= (1 << 20), "jpeg_restart must be in [0, 2^20]");
    if (segmented() && qq.kind != TQ_Q_NONE) {
        TQ_REQUIRE(N % M == 0, "paper/consensus rule with a quantizer needs equal segments (M | N)");
        if (dc) TQ_REQUIRE((N / M) % 8 == 0, "paper/consensus rule with DCT needs 8 | N/M");
    }
    free_exchange();
    q = qq;
}

void Ctx::set_sinogram(int slice, int node, const float *d, long long len, bool on_device, cudaStream_t src_s,
                       bool has_src_s) {
    Nvtx nv("tq:set_sinogram");
    TQ_REQUIRE(slice >= 0 && slice < S, "slice out of range");
    TQ_REQUIRE(node >= -1 && node < M, "node out of range");
    TQ_REQUIRE(d != nullptr, "null sinogram");
    const long long rows = node < 0 ? n_ang : (aoff[node + 1] - aoff[node]);
    TQ_REQUIRE(len == rows * n_det, "sinogram length mismatch");
    // staging copy on the device (upload stream, double-buffered), then a gather of the rows
    // of every local node, deferred to the stream of the next run (flush_gathers)
    TQ_CHECK_CUDA(cudaSetDevice(device));
    const int b = stage_buf;
    for (const PendGather &pg : pend_gathers)  // this buffer still queued: place the older gathers now
        if (pg.buf == b) {
            flush_gathers(pending ? run_s : stream);
            break;
        }
    if (sino_stage_len[b] < len) {
        TQ_CHECK_CUDA(cudaStreamSynchronize(up_stream));
        if (sino_stage[b]) {
            TQ_CHECK_CUDA(cudaEventSynchronize(stage_free[b]));
            cudaFree(sino_stage[b]);
        }
        sino_stage[b] = nullptr;
        TQ_CHECK_CUDA(cudaMalloc(&sino_stage[b], sizeof(float) * len));
        sino_stage_len[b] = len;
    }
    // the buffer is free once the last gather that read it ran; the caller's buffer is free
    // once this copy completed (waited for below)
    TQ_CHECK_CUDA(cudaStreamWaitEvent(up_stream, stage_free[b], 0));
    if (has_src_s) {  // the caller's device buffer is read after the work already on its stream
        TQ_CHECK_CUDA(cudaEventRecord(src_ready, src_s));
        TQ_CHECK_CUDA(cudaStreamWaitEvent(up_stream, src_ready, 0));
    }
    TQ_CHECK_CUDA(cudaMemcpyAsync(sino_stage[b], d, sizeof(float) * len,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, up_stream));
    TQ_CHECK_CUDA(cudaEventRecord(stage_copied[b], up_stream));
    stage_buf = (stage_buf + 1) % NSTAGE;
    // (source row, destination row) pairs of the local nodes, built once per (slice, node)
    auto it = gather_maps.find({slice, node});
    if (it == gather_maps.end()) {
        std::vector<int> pr;
        for (int i = 0; i < L; i++) {
            if (loc[i].first != slice) continue;
            const int m = loc[i].second;
            if (node >= 0 && m != node) continue;
            for (int k = 0; k < aoff[m + 1] - aoff[m]; k++) {
                pr.push_back(node < 0 ? aidx[aoff[m] + k] : k);
                pr.push_back(in.row0_h[i] + k);
            }
        }
        GatherMap gm{nullptr, (int)pr.size() / 2};
        if (gm.count) {
            TQ_CHECK_CUDA(cudaMalloc(&gm.pairs, sizeof(int) * pr.size()));
            TQ_CHECK_CUDA(cudaMemcpy(gm.pairs, pr.data(), sizeof(int) * pr.size(), cudaMemcpyHostToDevice));
        }
        it = gather_maps.emplace(std::make_pair(slice, node), gm).first;
    }
    for (int i = 0; i < L; i++)
        if (loc[i].first == slice && (node < 0 || loc[i].second == node)) sino_set[i] = 1;
    pend_gathers.push_back(PendGather{b, it->second.pairs, it->second.count});
    TQ_CHECK_CUDA(cudaEventSynchronize(stage_copied[b]));
}

// A stream wait on an event that has already completed is left out: no dependency node in
// front of the next graph launch.
static void wait_unless_done(cudaStream_t s, cudaEvent_t e) {
    const cudaError_t q = cudaEventQuery(e);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) TQ_CHECK_CUDA(q);
    TQ_CHECK_CUDA(cudaStreamWaitEvent(s, e, 0));
}

// The deferred sinogram gathers, in call order, on s: behind every run enqueued before them
// (s is the stream of the last run, or the next run's), ahead of the next.
void Ctx::flush_gathers(cudaStream_t s) {
    if (pend_gathers.empty()) return;
    if (pending && s != run_s) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, run_done, 0));
    for (const PendGather &pg : pend_gathers) {
        wait_unless_done(s, stage_copied[pg.buf]);
        if (pg.count) {
            const dim3 grid(ceil_div(n_det, 256), pg.count);
            if (prec == 0) gather_rows<float><<<grid, 256, 0, s>>>(sino_stage[pg.buf], pg.pairs, (float *)in.D, n_det);
            else gather_rows<double><<<grid, 256, 0, s>>>(sino_stage[pg.buf], pg.pairs, (double *)in.D, n_det);
            TQ_CHECK_CUDA(cudaGetLastError());
        }
        TQ_CHECK_CUDA(cudaEventRecord(stage_free[pg.buf], s));
    }
    pend_gathers.clear();
    // a run or component launched later on another stream orders itself after these gathers
    TQ_CHECK_CUDA(cudaEventRecord(gathers_done, s));
    gathers_s = s;
    gathers_live = true;
}

// the gathers placed by flush_gathers on another stream than s complete before s reads D
void Ctx::order_after_gathers(cudaStream_t s) {
    if (gathers_live && gathers_s != s) wait_unless_done(s, gathers_done);
}

long long Ctx::launch_component(int component, int reps, cudaStream_t s) {
    TQ_REQUIRE(reps >= 0, "reps must be >= 0");
    finish();
    flush_gathers(s ? s : stream);
    order_after_gathers(s ? s : stream);
    if (!have_params) fail(TQ_ESTATE, "tq_set_params must be called first");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    if (!xready) setup_exchange();
    long long vu = 0;
    for (int i = 0; i < L; i++) vu += (long long)in.nang_h[i] * n;
    switch (component) {
        case 0: for (int r = 0; r < reps; r++) in.project(geo, in.P, false, s); return vu;
        case 1: for (int r = 0; r < reps; r++) in.backproject(geo, EPI_CGR, in.Q, nullptr, in.P, s, in.R); return vu;
        case 2: for (int r = 0; r < reps; r++) in.project(geo, in.X, true, s); return vu;
        case 3:
        case 4: {
            const int kd = component == 3 ? TQ_Q_KMEANS : TQ_Q_DCT;
            Batch &E = enc[kd];
            TQ_REQUIRE(E.P > 0, "no local payloads of that quantizer kind");
            for (int r = 0; r < reps; r++) {
                if (E.need_conv) launch_to_float(prec, E.conv_src_d, E.conv_dst_d, n, (int)E.conv_src.size(), s);
                if (kd == TQ_Q_KMEANS) kmeans_encode(E.vin, kmw, q.lloyd_iters, E.pay, E.labels, s, E.dec_out, prec);
                else dct_encode(E.vin, E.P, segmented() ? N / M : N, N, q.quality, dctw, E.pay, s, jw_enc());
            }
            return (long long)E.P * payload_len;
        }
        case 5: for (int r = 0; r < reps; r++) prepare_rhs(s); return (long long)L * n;
        default: fail(TQ_EINVAL, "unknown component");
    }
}

void Ctx::setup_exchange() {
    free_exchange();
    const size_t es = prec ? 8 : 4;
    const bool paper = segmented();  // segment payloads + all-gather (paper and consensus rules)
    payload_len = paper ? n / M : n;
    std::vector<std::pair<int, int>> sp, rp;
    exchange_plan(M, edges, node_rank, rule, rank, world, sp, rp);
    // ---- payload list
    auto add_pay = [&](int s, int m, bool local) {
        if (pay_of.count({s, m})) return;
        Pay p{s, m, nullptr, local, kind_of_slice(s)};
        pay_of[{s, m}] = (int)pays.size();
        pays.push_back(p);
    };
    std::vector<int> slices_here;
    for (int s = 0; s < S; s++) {
        bool any = false;
        for (int m = 0; m < M; m++) any |= local(s, m) >= 0;
        if (any) slices_here.push_back(s);
    }
    for (int i = 0; i < L; i++) add_pay(loc[i].first, loc[i].second, true);
    for (int s : slices_here) {
        if (paper) {
            for (int m = 0; m < M; m++) add_pay(s, m, local(s, m) >= 0);
        } else {
            for (auto &r : rp) add_pay(s, r.first, false);
        }
    }
    // ---- buffers: payload (wire) and decoded public value
    std::vector<void *> xh(pays.size(), nullptr), outp(pays.size(), nullptr);
    std::vector<long long> pbytes(pays.size(), 0);
    for (size_t k = 0; k < pays.size(); k++) {
        Pay &p = pays[k];
        const int li = local(p.slice, p.node);
        if (p.kind == TQ_Q_NONE) {
            if (paper) {
                const long long lo = (long long)row_off[p.node] * N, len = (long long)(row_off[p.node + 1] - row_off[p.node]) * N;
                p.buf = (uint8_t *)XG + es * ((long long)p.slice * n + lo);
                pbytes[k] = es * len;
            } else {
                p.buf = li >= 0 ? (uint8_t *)in.xrow(in.X, li) : (uint8_t *)dev_alloc(es * n);
                pbytes[k] = es * n;
                xh[k] = p.buf;
            }
        } else {
            pbytes[k] = p.kind == TQ_Q_KMEANS ? kmeans_payload_bytes(q.k, payload_len) : dct_bytes(payload_len);
            p.buf = (uint8_t *)dev_alloc(pbytes[k]);
            if (paper) {
                outp[k] = (uint8_t *)XG + es * ((long long)p.slice * n + (long long)row_off[p.node] * N);
            } else {
                xh[k] = dev_alloc(es * n);
                outp[k] = xh[k];
            }
        }
    }
    auto upload = [&](const void *src, size_t bytes) {
        void *d = dev_alloc(bytes);
        TQ_CHECK_CUDA(cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice));
        return d;
    };
    // ---- float staging for quantizer inputs
    std::vector<int> stage_row(L, -1);
    int nstage = 0;
    for (int i = 0; i < L; i++) {
        const int kd = kind_of_slice(loc[i].first);
        if (kd == TQ_Q_NONE) continue;
        if (paper || prec == 1) stage_row[i] = nstage++;
    }
    if (nstage) fstage = (float *)dev_alloc(sizeof(float) * payload_len * nstage);
    label_row.assign(L, -1);
    int nlab = 0;
    if (q.keep_labels)
        for (int i = 0; i < L; i++)
            if (kind_of_slice(loc[i].first) == TQ_Q_KMEANS) label_row[i] = nlab++;
    if (nlab) labels_buf = (int32_t *)dev_alloc(sizeof(int32_t) * payload_len * nlab);
    // ---- encode / decode batches
    for (int kd = 1; kd <= 2; kd++) {
        Batch &E = enc[kd], &D = dec[kd];
        E.kind = D.kind = kd;
        std::vector<const float *> vin;
        std::vector<uint8_t *> pe, pd;
        std::vector<int32_t *> lab;
        std::vector<const void *> csrc;
        std::vector<float *> cdst;
        std::vector<void *> out, eout;
        for (size_t k = 0; k < pays.size(); k++) {
            if (pays[k].kind != kd) continue;
            // K-means payloads produced here are decoded by the encoder's final pass
            if (!(kd == TQ_Q_KMEANS && pays[k].local)) {
                pd.push_back(pays[k].buf);
                out.push_back(outp[k]);
                D.members.push_back((int)k);
            }
            if (!pays[k].local) continue;
            eout.push_back(outp[k]);
            const int li = local(pays[k].slice, pays[k].node);
            E.members.push_back((int)k);
            pe.push_back(pays[k].buf);
            const float *v;
            if (stage_row[li] >= 0) {
                v = fstage + (long long)stage_row[li] * payload_len;
                if (!paper) { csrc.push_back(in.xrow(in.X, li)); cdst.push_back((float *)v); }
            } else {
                v = (const float *)in.xrow(in.X, li);
            }
            vin.push_back(v);
            lab.push_back(label_row[li] >= 0 ? labels_buf + (long long)label_row[li] * payload_len : nullptr);
        }
        E.P = (int)pe.size();
        D.P = (int)pd.size();
        if (E.P) {
            E.vin = (const float **)upload(vin.data(), sizeof(void *) * E.P);
            E.pay = (uint8_t **)upload(pe.data(), sizeof(void *) * E.P);
            if (kd == TQ_Q_KMEANS && nlab) E.labels = (int32_t **)upload(lab.data(), sizeof(void *) * E.P);
            if (kd == TQ_Q_KMEANS) E.dec_out = (void **)upload(eout.data(), sizeof(void *) * E.P);
            if (!csrc.empty()) {
                E.need_conv = true;
                E.conv_src.assign(csrc.begin(), csrc.end());
                E.conv_src_d = (const void **)upload(csrc.data(), sizeof(void *) * csrc.size());
                E.conv_dst_d = (float **)upload(cdst.data(), sizeof(void *) * cdst.size());
            }
            if (kd == TQ_Q_KMEANS) kmw.alloc(E.P, q.k, payload_len);
            else {
                dctw.alloc(E.P, payload_len);
                if (q.jpeg_restart > 0) jenc.alloc(E.P, payload_len, q.jpeg_restart);
            }
        }
        if (kd == TQ_Q_DCT && D.P && q.jpeg_restart > 0) jdec.alloc(D.P, payload_len, q.jpeg_restart);
        if (D.P) {
            D.pay = (uint8_t **)upload(pd.data(), sizeof(void *) * D.P);
            D.out = (void **)upload(out.data(), sizeof(void *) * D.P);
        }
    }
    // ---- node groups (TQ_GROUPS; 1 = one launch sequence over all nodes): the graph rule's fp32
    // path; each encode batch (K-means, DCT with or without JPEG coding) must hold local payloads
    // in local-node order, so a group's payloads are one contiguous subrange of each batch
    {
        const char *env = getenv("TQ_GROUPS");
        // default: one group per node (up to MAXG) for images of 512^2 and more; below that the
        // kernels are short and the extra launches cost more than the overlap gains (C1, C2)
        const int dflt = geo.N >= 512 ? (int)MAXG : 1;
        const int want = std::min(std::min(env ? atoi(env) : dflt, (int)MAXG), L);
        bool ok = want >= 2 && prec == 0 && rule == TQ_RULE_GRAPH && geo.N % 4 == 0;
        std::vector<int> li_of[3];
        for (int kd = 1; ok && kd <= 2; kd++) {
            if (!enc[kd].P) continue;
            ok = !enc[kd].need_conv;
            for (int b = 0; ok && b < enc[kd].P; b++) {
                const Pay &p = pays[enc[kd].members[b]];
                const int li = local(p.slice, p.node);
                ok = li >= 0 && (li_of[kd].empty() || li > li_of[kd].back());
                li_of[kd].push_back(li);
            }
        }
        if (ok) {
            ngroups = want;
            for (int g = 0; g < want; g++) {
                grp_n0[g] = g * L / want;
                grp_cnt[g] = (g + 1) * L / want - grp_n0[g];
                for (int kd = 1; kd <= 2; kd++) {
                    int b0 = 0, bc = 0;
                    for (int li : li_of[kd]) {
                        if (li < grp_n0[g]) b0++;
                        else if (li < grp_n0[g] + grp_cnt[g]) bc++;
                    }
                    grp_b0[kd][g] = b0;
                    grp_bc[kd][g] = bc;
                }
                if (grp_bc[TQ_Q_KMEANS][g]) kmw_g[g].alloc(grp_bc[TQ_Q_KMEANS][g], q.k, payload_len);
                if (grp_bc[TQ_Q_DCT][g]) {
                    dctw_g[g].alloc(grp_bc[TQ_Q_DCT][g], payload_len);
                    if (q.jpeg_restart > 0) jenc_g[g].alloc(grp_bc[TQ_Q_DCT][g], payload_len, q.jpeg_restart);
                }
            }
        }
    }
    // ---- consensus tables
    if (!paper) {
        xh_tab = (const void **)upload(xh.data(), sizeof(void *) * xh.size());
        std::vector<int> own(L), off(L + 1, 0), nb;
        for (int i = 0; i < L; i++) {
            own[i] = pay_of.at(loc[i]);
            for (int j : adj[loc[i].second]) nb.push_back(pay_of.at({loc[i].first, j}));
            off[i + 1] = (int)nb.size();
        }
        own_slot = (int *)upload(own.data(), sizeof(int) * std::max(1, L));
        nbr_off = (int *)upload(off.data(), sizeof(int) * (L + 1));
        if (nb.empty()) nb.push_back(0);
        nbr_slot = (int *)upload(nb.data(), sizeof(int) * nb.size());
        // the same tables resolved to pointers (the dual kernel's prologue: one load level)
        std::vector<const void *> ownp(std::max(1, L), nullptr), nbp(nb.size());
        for (int i = 0; i < L; i++) ownp[i] = xh[own[i]];
        for (size_t k = 0; k < nb.size(); k++) nbp[k] = xh[nb[k]];
        own_ptr = (const void **)upload(ownp.data(), sizeof(void *) * ownp.size());
        nbr_ptr = (const void **)upload(nbp.data(), sizeof(void *) * nbp.size());
    } else {
        std::vector<void *> xg(L);
        std::vector<long long> lo(L), len(L);
        std::vector<float *> seg(L, nullptr);
        for (int i = 0; i < L; i++) {
            const int s = loc[i].first, m = loc[i].second;
            xg[i] = (uint8_t *)XG + es * (long long)s * n;
            lo[i] = (long long)row_off[m] * N;
            len[i] = (long long)(row_off[m + 1] - row_off[m]) * N;
            if (stage_row[i] >= 0) seg[i] = fstage + (long long)stage_row[i] * payload_len;
        }
        xg_tab = (void **)upload(xg.data(), sizeof(void *) * std::max(1, L));
        seg_lo = (long long *)upload(lo.data(), sizeof(long long) * std::max(1, L));
        seg_len = (long long *)upload(len.data(), sizeof(long long) * std::max(1, L));
        seg_max = 0;
        for (int m = 0; m < M; m++) seg_max = std::max(seg_max, (long long)(row_off[m + 1] - row_off[m]) * N);
        seg_tab = (float **)upload(seg.data(), sizeof(void *) * std::max(1, L));
        if (rule == TQ_RULE_CONSENSUS) {
            // partial-sum tables over ALL slices (slices without local nodes write zeros, so
            // the reduction never re-adds a stale sum); local nodes of a slice are contiguous
            std::vector<int> sl(S), fi(S, 0), cn(S, 0), ns(L);
            for (int t = 0; t < S; t++) sl[t] = t;
            for (int i = L - 1; i >= 0; i--) { fi[loc[i].first] = i; cn[loc[i].first]++; }
            for (int i = 0; i < L; i++) ns[i] = loc[i].first;
            cs_slice = (int *)upload(sl.data(), sizeof(int) * S);
            cs_first = (int *)upload(fi.data(), sizeof(int) * S);
            cs_cnt = (int *)upload(cn.data(), sizeof(int) * S);
            node_slice = (int *)upload(ns.data(), sizeof(int) * std::max(1, L));
        }
    }
    // ---- NCCL transfers (per slice, same plan)
    for (int s : slices_here) {
        for (auto &x : sp) {
            const int k = pay_of.at({s, x.first});
            sends.push_back(XferDesc{s, x.first, x.second, pays[k].buf, pbytes[k]});
        }
        for (auto &x : rp) {
            const int k = pay_of.at({s, x.first});
            recvs.push_back(XferDesc{s, x.first, x.second, pays[k].buf, pbytes[k]});
        }
    }
    // ---- logical bytes (what the method sends, independent of placement)
    // (entropy-coded DCT payloads: capacity until a run reports their actual sizes)
    long long logical = 0;
    for (int i = 0; i < L; i++) {
        const int kd = kind_of_slice(loc[i].first), m = loc[i].second;
        const long long len = paper ? (long long)(row_off[m + 1] - row_off[m]) * N : n;
        const long long pb = kd == TQ_Q_NONE ? (long long)es * len
                             : kd == TQ_Q_KMEANS ? kmeans_payload_bytes(q.k, payload_len)
                                                 : dct_bytes(payload_len);
        const long long mult = paper ? (M - 1) : (long long)adj[m].size();
        logical += pb * mult;
        if (rule == TQ_RULE_CONSENSUS) logical += 8LL * (n - len);  // fp64 sums of the other segments
        if (kd == TQ_Q_DCT && q.jpeg_restart > 0) logical_fixed -= pb * mult;
    }
    logical_fixed += logical;
    if (jenc.P) {
        Batch &E = enc[TQ_Q_DCT];
        for (int k : E.members) {
            const int m = pays[k].node;
            jmult.push_back(paper ? (M - 1) : (long long)adj[m].size());
        }
    }
    st.payload_bytes_logical = logical;
    st.nccl_bytes_sent = 0;
    for (auto &x : sends) st.nccl_bytes_sent += x.bytes;
    st.nccl_bytes_recv = 0;
    for (auto &x : recvs) st.nccl_bytes_recv += x.bytes;
    if (rule == TQ_RULE_CONSENSUS)
        for (int t = 0; t < S; t++)
            for (int m = 0; m < M; m++)
                sum_segs.push_back(SumSeg{(long long)t * n + (long long)row_off[m] * N,
                                          (long long)(row_off[m + 1] - row_off[m]) * N, node_rank[m]});
    xready = true;
}

// Bytes node (slice, node) sent / received per iteration as the method moves them
// (tq_get_node_bytes).  Entropy-coded DCT payloads: the coded sizes in their headers.
void Ctx::node_bytes(int slice, int node, long long &sent, long long &recv) {
    finish();
    const int i = local(slice, node);
    TQ_REQUIRE(i >= 0, "node is not local to this rank");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    if (!xready) setup_exchange();
    const size_t es = prec ? 8 : 4;
    const bool seg = segmented();
    auto seglen = [&](int m) { return (long long)(row_off[m + 1] - row_off[m]) * N; };
    auto pay_bytes = [&](int m) -> long long {
        const int kd = kind_of_slice(slice);
        if (kd == TQ_Q_NONE) return (long long)es * (seg ? seglen(m) : n);
        if (kd == TQ_Q_KMEANS) return kmeans_payload_bytes(q.k, payload_len);
        if (q.jpeg_restart <= 0) return dct_payload_bytes(payload_len);
        const Pay &p = pays[pay_of.at({slice, m})];  // [mn][mx][u32 bytes | raw bit 31][u32 blocks]
        uint32_t w = 0;
        TQ_CHECK_CUDA(cudaMemcpy(&w, p.buf + 8, sizeof w, cudaMemcpyDeviceToHost));
        return 16 + ((w & 0x80000000u) ? 2 * payload_len : (long long)w);
    };
    sent = recv = 0;
    if (!seg) {
        const long long own = pay_bytes(node);
        sent = own * (long long)adj[node].size();
        for (int j : adj[node]) recv += pay_bytes(j);
    } else {
        sent = pay_bytes(node) * (M - 1);
        for (int m = 0; m < M; m++)
            if (m != node) recv += pay_bytes(m);
        if (rule == TQ_RULE_CONSENSUS) {  // fp64 partial sums of the other segments / of its own
            sent += 8LL * (n - seglen(node));
            recv += 8LL * (M - 1) * seglen(node);
        }
    }
}

bool Ctx::use_ax() const { return ax_maxage > 0 && prm.inner == TQ_INNER_CG && rule == TQ_RULE_GRAPH; }

// before graph launches covering `iters` iterations: refresh the kept A x (outside the graphs)
// when it is stale or would age past ax_maxage iterations (its fp rounding then stays at the
// level of a few direct projections)
void Ctx::ax_before(int iters, cudaStream_t s) {
    if (!use_ax() || iters <= 0) return;
    if (!ax_valid || ax_age + iters > std::max(ax_maxage, MULTI)) {
        in.project(geo, in.X, false, s, in.AX, n_det, 0);
        ax_valid = true;
        ax_age = 0;
    }
    ax_age += iters;
}

bool Ctx::grouped() const {
    return ngroups >= 2 && rule == TQ_RULE_GRAPH && prm.inner == TQ_INNER_CG && prec == 0;
}

int Ctx::stage01_grouped(cudaStream_t s) {
    TQ_CHECK_CUDA(cudaEventRecord(ev_fork, s));
    for (int g = 1; g < ngroups; g++) TQ_CHECK_CUDA(cudaStreamWaitEvent(sg[g], ev_fork, 0));
    int k = 0;
    for (int g = 0; g < ngroups; g++) {
        cudaStream_t st = g ? sg[g] : s;
        k += in.cg(geo, prm.e1, st, use_ax() ? AX_CACHED : AX_OFF, grp_n0[g], grp_cnt[g]);
        if (grp_bc[TQ_Q_KMEANS][g]) {
            Batch &E = enc[TQ_Q_KMEANS];
            const int b0 = grp_b0[TQ_Q_KMEANS][g];
            k += kmeans_encode(E.vin + b0, kmw_g[g], q.lloyd_iters, E.pay + b0, E.labels ? E.labels + b0 : nullptr,
                               st, E.dec_out ? E.dec_out + b0 : nullptr, prec);
        }
        if (grp_bc[TQ_Q_DCT][g]) {
            Batch &E = enc[TQ_Q_DCT];
            const int b0 = grp_b0[TQ_Q_DCT][g];
            k += dct_encode(E.vin + b0, grp_bc[TQ_Q_DCT][g], N, N, q.quality, dctw_g[g], E.pay + b0, st,
                            q.jpeg_restart > 0 ? &jenc_g[g] : nullptr);
        }
    }
    for (int g = 1; g < ngroups; g++) {
        TQ_CHECK_CUDA(cudaEventRecord(ev_join[g], sg[g]));
        TQ_CHECK_CUDA(cudaStreamWaitEvent(s, ev_join[g], 0));
    }
    return k;
}

int Ctx::stages(const std::vector<int> &ids, cudaStream_t s) {
    int c = 0;
    for (size_t i = 0; i < ids.size(); i++) {
        if (ids[i] == 0 && i + 1 < ids.size() && ids[i + 1] == 1 && grouped()) {
            c += stage01_grouped(s);
            i++;
        } else {
            c += stage(ids[i], s);
        }
    }
    return c;
}

int Ctx::stage(int id, cudaStream_t s) {
    if (id == 2) return phase_b(s);
    int k = 0;
    if (id == 0) {
        k += prm.inner == TQ_INNER_CG ? in.cg(geo, prm.e1, s, use_ax() ? AX_CACHED : AX_OFF) : in.gd(geo, prm.e1, s);
        if (rule == TQ_RULE_PAPER)
            k += launch_paper_alg3(prec, in.X, ALPHA, xg_tab, seg_lo, seg_len, seg_max, seg_tab, n, L,
                                   prm.rho, prm.eta2, prm.e2, s);
        if (rule == TQ_RULE_CONSENSUS)
            k += launch_consensus_partial(prec, in.X, ALPHA, CSUM, cs_slice, cs_first, cs_cnt, S, n, prm.rho, s);
        return k;
    }
    if (rule == TQ_RULE_CONSENSUS)
        k += launch_consensus_segment(prec, CSUM, node_slice, xg_tab, seg_lo, seg_len, seg_max, seg_tab, n, L, M, s);
    for (int kd = 1; kd <= 2; kd++) {
        Batch &E = enc[kd];
        if (!E.P) continue;
        if (E.need_conv) k += launch_to_float(prec, E.conv_src_d, E.conv_dst_d, n, (int)E.conv_src.size(), s);
        if (kd == TQ_Q_KMEANS) k += kmeans_encode(E.vin, kmw, q.lloyd_iters, E.pay, E.labels, s, E.dec_out, prec);
        else {
            const int rows = segmented() ? N / M : N;
            k += dct_encode(E.vin, E.P, rows, N, q.quality, dctw, E.pay, s, jw_enc());
        }
    }
    return k;
}

// consensus rule, world > 1: segment m of every slice's partial sum is summed onto the
// rank owning node m (one grouped ncclReduce per (slice, segment) -- a reduce-scatter in
// the paper's segment layout), which then forms x[m] locally.
void Ctx::reduce_sums(cudaStream_t s) { tr->reduce_sum(s, CSUM, sum_segs); }

void Ctx::exchange(cudaStream_t s) {
    if (!has_exchange()) return;
    tr->exchange(s, sends, recvs);
}

bool Ctx::has_exchange() const {
    return world > 1 && (tr->collective_exchange() || !(sends.empty() && recvs.empty()));
}

int Ctx::phase_b(cudaStream_t s) {
    int k = 0;
    for (int kd = 1; kd <= 2; kd++) {
        Batch &D = dec[kd];
        if (!D.P) continue;
        if (kd == TQ_Q_KMEANS) k += kmeans_decode(D.pay, D.P, payload_len, q.k, prec, D.out, s);
        else {
            const int rows = segmented() ? N / M : N;
            k += dct_decode(D.pay, D.P, rows, N, q.quality, prec, D.out, s, jdec.P ? &jdec : nullptr);
        }
    }
    if (rule == TQ_RULE_GRAPH)
        k += launch_graph_dual(prec, own_ptr, nbr_ptr, nbr_off, ALPHA, in.BP, n, L, prm.rho, 1, s);
    else
        k += launch_paper_dual(prec, in.X, ALPHA, in.BP, (const void *const *)xg_tab, n, L, prm.rho, 1, s);
    return k;
}

int Ctx::prepare_rhs(cudaStream_t s) {
    if (rule == TQ_RULE_GRAPH)
        return launch_graph_dual(prec, own_ptr, nbr_ptr, nbr_off, ALPHA, in.BP, n, L, prm.rho, 0, s);
    return launch_paper_dual(prec, in.X, ALPHA, in.BP, (const void *const *)xg_tab, n, L, prm.rho, 0, s);
}

void Ctx::run(int iters, cudaStream_t user) {
    enqueue(iters, user);
    finish();
}

void Ctx::run_async(int iters, cudaStream_t user) { enqueue(iters, user); }

void Ctx::enqueue(int iters, cudaStream_t user) {
    Nvtx nv("tq:run");
    TQ_REQUIRE(iters >= 0, "iters must be >= 0");
    if (!have_params) fail(TQ_ESTATE, "tq_set_params must be called before tq_run");
    for (int i = 0; i < L; i++)
        if (!sino_set[i]) fail(TQ_ESTATE, "sinogram of a local node was never set");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    if (!xready) {
        finish();  // the exchange state is (re)built: nothing may be in flight
        setup_exchange();
    }
    cudaStream_t s = user ? user : stream;
    if (pending && s != run_s) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, run_done, 0));  // previous run
    flush_gathers(s);  // a new sinogram: its gather, in-stream
    order_after_gathers(s);  // gathers flushed earlier onto another stream (set_sinogram reuse)
    for (int b = 0; b < 2; b++)  // an enqueued tq_get_image_async snapshot reads X first
        if (img_used[b] && img_s[b] != s) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, img_ready[b], 0));
    run_s = s;
    if (need_rhs) {
        prepare_rhs(s);
        need_rhs = false;
    }
    auto capture = [&](std::vector<Seg> &into, const std::vector<int> &ids, int comm_after) {
        Nvtx nc("tq:capture");
        cudaGraph_t g;
        TQ_CHECK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int c = 0;
        try {
            c += stages(ids, s);
        } catch (...) {
            if (cudaStreamEndCapture(s, &g) == cudaSuccess && g) cudaGraphDestroy(g);
            (void)cudaGetLastError();  // do not leave the capture failure as the sticky last error
            throw;
        }
        TQ_CHECK_CUDA(cudaStreamEndCapture(s, &g));
        Seg sg{nullptr, c, comm_after};
        const cudaError_t e = cudaGraphInstantiate(&sg.exec, g, 0);
        cudaGraphDestroy(g);
        TQ_CHECK_CUDA(e);
        TQ_CHECK_CUDA(cudaGraphUpload(sg.exec, s));  // the first launch does not pay the upload
        into.push_back(sg);
    };
    const bool red = rule == TQ_RULE_CONSENSUS && world > 1;
    const bool exch = has_exchange();
    const bool stop = prm.stop_tol > 0.0;
    if (stop) setup_stop_test(s);  // allocations before any capture of this call
    // ranks sharing a process (loopback) capture between two host fences: a thread's device
    // allocation or graph instantiation must not overlap another rank's capture
    const bool capturing = segs.empty() || (profiling && psegs.empty());
    if (capturing && world > 1) tr->host_fence();
    if (segs.empty()) {
        // stages 0 | reduce | 1 | exchange | 2, merged where no communication separates them
        std::vector<int> cur{0};
        if (red) { capture(segs, cur, COMM_REDUCE); cur.clear(); }
        cur.push_back(1);
        if (exch) { capture(segs, cur, COMM_EXCHANGE); cur.clear(); }
        cur.push_back(2);
        capture(segs, cur, COMM_NONE);
    }
    if (profiling && psegs.empty()) {  // one graph per phase, timing events in between
        capture(psegs, {0}, red ? COMM_REDUCE : COMM_NONE);
        capture(psegs, {1}, exch ? COMM_EXCHANGE : COMM_NONE);
        capture(psegs, {2}, COMM_NONE);
    }
    if (capturing && world > 1) tr->host_fence();
    // one rank without communication steps: a second graph holding MULTI iterations (built
    // with the first, i.e. during warm-up) cuts the graph-to-graph boundaries of long runs
    if (!stop && !profiling && segs.size() == 1 && segs[0].comm == COMM_NONE && !seg2.exec) {
        cudaGraph_t g;
        TQ_CHECK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int c = 0;
        try {
            for (int rep = 0; rep < MULTI; rep++) c += stages({0, 1, 2}, s);
        } catch (...) {
            if (cudaStreamEndCapture(s, &g) == cudaSuccess && g) cudaGraphDestroy(g);
            (void)cudaGetLastError();
            throw;
        }
        TQ_CHECK_CUDA(cudaStreamEndCapture(s, &g));
        const cudaError_t e = cudaGraphInstantiate(&seg2.exec, g, 0);
        cudaGraphDestroy(g);
        TQ_CHECK_CUDA(e);
        TQ_CHECK_CUDA(cudaGraphUpload(seg2.exec, s));
        seg2.launches = c;
    }
    int per_iter = 0;
    for (auto &g : segs) per_iter += g.launches;
    if (profiling && (int)pev.size() < 5 * iters) {
        const size_t old = pev.size();
        pev.resize(5 * (size_t)iters);
        for (size_t k = old; k < pev.size(); k++) TQ_CHECK_CUDA(cudaEventCreate(&pev[k]));
    }
    auto comm_step = [&](int comm) {
        if (comm == COMM_REDUCE) { Nvtx nc("tq:reduce"); reduce_sums(s); }
        else if (comm == COMM_EXCHANGE) { Nvtx nc("tq:exchange"); exchange(s); }
    };
    // phase of the stage graphs (psegs / a segment starting at stage 0, 1 or 2)
    static const char *const kPhase[3] = {"tq:inner_solve", "tq:encode", "tq:decode_dual"};
    TQ_CHECK_CUDA(cudaEventRecord(ev0, s));
    int it0 = 0, done = 0;
    st.rel_change_last = -1.0;
    if (seg2.exec && !stop && !profiling)
        for (; it0 + MULTI <= iters; it0 += MULTI) {
            Nvtx ni("tq:iterations");
            ax_before(MULTI, s);
            TQ_CHECK_CUDA(cudaGraphLaunch(seg2.exec, s));
        }
    done = it0;
    for (int it = it0; it < iters; it++) {
        Nvtx ni("tq:iteration");
        ax_before(1, s);
        if (profiling) {
            cudaEvent_t *e = &pev[5 * (size_t)it];
            TQ_CHECK_CUDA(cudaEventRecord(e[0], s));
            { Nvtx np(kPhase[0]); TQ_CHECK_CUDA(cudaGraphLaunch(psegs[0].exec, s)); }
            comm_step(psegs[0].comm);
            TQ_CHECK_CUDA(cudaEventRecord(e[1], s));
            { Nvtx np(kPhase[1]); TQ_CHECK_CUDA(cudaGraphLaunch(psegs[1].exec, s)); }
            TQ_CHECK_CUDA(cudaEventRecord(e[2], s));
            comm_step(psegs[1].comm);
            TQ_CHECK_CUDA(cudaEventRecord(e[3], s));
            { Nvtx np(kPhase[2]); TQ_CHECK_CUDA(cudaGraphLaunch(psegs[2].exec, s)); }
            TQ_CHECK_CUDA(cudaEventRecord(e[4], s));
        } else {
            for (auto &g : segs) {
                TQ_CHECK_CUDA(cudaGraphLaunch(g.exec, s));
                comm_step(g.comm);
            }
        }
        done = it + 1;
        if (stop) {
            double r = stop_test(s);
            if (world > 1) r = tr->allreduce_max(r, s);
            st.rel_change_last = r;
            if (r <= prm.stop_tol) break;
        }
    }
    TQ_CHECK_CUDA(cudaEventRecord(ev1, s));
    // CG with E1 >= 1 leaves ||x||^2 in the scalar table (its last step); otherwise compute it
    if (!(done > 0 && prm.inner == TQ_INNER_CG && prm.e1 >= 1)) in.norm2(s);
    TQ_CHECK_CUDA(cudaEventRecord(run_done, s));
    st.iters += done;
    st.iters_last_run = done;
    st.kernel_launches = (long long)done * per_iter + (stop ? done : 0);
    st.phase_valid = 0;
    st.node_groups = (!profiling && grouped()) ? ngroups : 1;
    pending = true;
    pending_iters = done;
    prof_iters = profiling ? done : 0;
}

// tq_params.stop_tol: the iterates whose relative change is tested (graph rule: every local
// node's private x_i; paper / consensus rules: the consensus x of every slice held here),
// snapshotted at the start of each run
void Ctx::setup_stop_test(cudaStream_t s) {
    const bool seg = segmented();
    const int V = seg ? S : L;
    if (chg_V != V) {
        const size_t es = prec ? 8 : 4;
        auto A = [&](void **p, size_t bytes) {
            TQ_CHECK_CUDA(cudaMalloc(p, std::max<size_t>(bytes, 16)));
            TQ_CHECK_CUDA(cudaMemset(*p, 0, std::max<size_t>(bytes, 16)));
            chg_owned.push_back(*p);
        };
        A(&XPREV, es * n * std::max(1, V));
        A((void **)&chg_out, sizeof(double) * 2 * std::max(1, V));
        A((void **)&chg_part, sizeof(double) * 2 * (size_t)vec_blocks(n) * std::max(1, V));
        A((void **)&chg_cnt, sizeof(unsigned) * std::max(1, V));
        std::vector<const void *> tab(std::max(1, V), nullptr);
        for (int v = 0; v < V; v++) tab[v] = seg ? (const void *)((const uint8_t *)XG + es * n * v) : in.xrow(in.X, v);
        A((void **)&chg_tab, sizeof(void *) * tab.size());
        TQ_CHECK_CUDA(cudaMemcpy(chg_tab, tab.data(), sizeof(void *) * tab.size(), cudaMemcpyHostToDevice));
        TQ_CHECK_CUDA(cudaMallocHost(&chg_host, sizeof(double) * 2 * std::max(1, V)));
        chg_V = V;
    }
    const size_t es = prec ? 8 : 4;
    if (seg) TQ_CHECK_CUDA(cudaMemcpyAsync(XPREV, XG, es * n * V, cudaMemcpyDeviceToDevice, s));
    else if (V) TQ_CHECK_CUDA(cudaMemcpyAsync(XPREV, in.X, es * n * V, cudaMemcpyDeviceToDevice, s));
}

// r_k = max over the tested iterates of ||x^{k+1} - x^k|| / ||x^{k+1}|| (0/0 := 0); blocking
double Ctx::stop_test(cudaStream_t s) {
    launch_rel_change(prec, chg_tab, XPREV, n, chg_V, chg_out, chg_part, vec_blocks(n), chg_cnt, s);
    if (chg_V) TQ_CHECK_CUDA(cudaMemcpyAsync(chg_host, chg_out, sizeof(double) * 2 * chg_V, cudaMemcpyDeviceToHost, s));
    TQ_CHECK_CUDA(cudaStreamSynchronize(s));
    double r = 0.0;
    for (int v = 0; v < chg_V; v++) {
        const double dd = chg_host[2 * v], xx = chg_host[2 * v + 1];
        const double q = dd == 0.0 ? 0.0 : (xx > 0.0 ? sqrt(dd / xx) : INFINITY);
        r = std::max(r, q);
    }
    return r;
}

void Ctx::free_stop_test() {
    for (void *p : chg_owned) cudaFree(p);
    chg_owned.clear();
    if (chg_host) cudaFreeHost(chg_host);
    chg_host = nullptr;
    XPREV = nullptr; chg_out = chg_part = nullptr; chg_cnt = nullptr; chg_tab = nullptr;
    chg_V = -1;
}

void Ctx::set_profiling(bool on) {
    finish();
    profiling = on;
}

// The host side of an enqueued run: wait for it, then its statistics and the divergence
// guard (SPEC "divergence guard"; the norms of its last iteration).
void Ctx::finish() {
    if (!pending) return;
    Nvtx nv("tq:wait");
    pending = false;
    TQ_CHECK_CUDA(cudaEventSynchronize(run_done));
    if (guards_enabled()) {  // TQ_GUARD=1: the run wrote nothing outside its allocations
        std::string where;
        if (!guards_intact(where)) fail(TQ_ECUDA, "TQ_GUARD: guard band corrupted: " + where);
    }
    // the scalar table of the last enqueued run (nothing else writes it before this call)
    if (!norm_host) TQ_CHECK_CUDA(cudaMallocHost(&norm_host, sizeof(double) * S_NSLOT * std::max(1, L)));
    if (L) TQ_CHECK_CUDA(cudaMemcpy(norm_host, in.scal, sizeof(double) * S_NSLOT * L, cudaMemcpyDeviceToHost));
    const int iters = pending_iters;
    float ms = 0.f;
    TQ_CHECK_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    st.ms_last_run = ms;
    if (prof_iters > 0) {  // per-phase device time of the profiled run
        double ph[4] = {0, 0, 0, 0};
        for (int it = 0; it < prof_iters; it++)
            for (int k = 0; k < 4; k++) {
                float t = 0.f;
                TQ_CHECK_CUDA(cudaEventElapsedTime(&t, pev[5 * (size_t)it + k], pev[5 * (size_t)it + k + 1]));
                ph[k] += t;
            }
        for (int k = 0; k < 4; k++) st.phase_ms[k] = ph[k];
        st.phase_valid = 1;
        prof_iters = 0;
    }
    for (int i = 0; i < L; i++) {
        const double nrm = sqrt(norm_host[(size_t)i * S_NSLOT + S_NORM]);
        if (!(nrm <= 1e12)) fail(TQ_EDIVERGED, "node iterate norm exceeded 1e12 (diverged)");
    }
    if (iters > 0 && (jenc.P || jdec.P)) {  // entropy-coded DCT payloads: actual sizes, stream checks
        std::vector<long long> eb(std::max(1, jenc.P));
        std::vector<unsigned> sd(2 * std::max(1, jdec.P), 0u);
        if (jenc.P && st.node_groups > 1) {  // the last run's coders were the groups' (their subranges)
            for (int g = 0; g < ngroups; g++)
                if (jenc_g[g].P)
                    TQ_CHECK_CUDA(cudaMemcpy(eb.data() + grp_b0[TQ_Q_DCT][g], jenc_g[g].enc_bytes,
                                             sizeof(long long) * jenc_g[g].P, cudaMemcpyDeviceToHost));
        } else if (jenc.P) {
            TQ_CHECK_CUDA(cudaMemcpy(eb.data(), jenc.enc_bytes, sizeof(long long) * jenc.P, cudaMemcpyDeviceToHost));
        }
        if (jdec.P) TQ_CHECK_CUDA(cudaMemcpy(sd.data(), jdec.status, sizeof(unsigned) * 2 * jdec.P, cudaMemcpyDeviceToHost));
        long long logical = logical_fixed;
        for (int b = 0; b < jenc.P; b++) logical += eb[b] * jmult[b];
        st.payload_bytes_logical = logical;
        for (int b = 0; b < jdec.P; b++)
            if (sd[2 * b + 1]) fail(TQ_ECUDA, "malformed JPEG entropy stream in a received DCT payload");
    }
}

void Ctx::snapshot_image(int slice, int node, float *d, cudaStream_t stream) {
    const int blocks = (int)std::min<long long>(2048, (n + 255) / 256);
    if (node >= 0) {
        const int i = local(slice, node);
        if (i < 0) fail(TQ_EINVAL, "node is not local to this rank");
        if (prec == 0) TQ_CHECK_CUDA(cudaMemcpyAsync(d, in.xrow(in.X, i), sizeof(float) * n, cudaMemcpyDeviceToDevice, stream));
        else launch_convert(prec, in.xrow(in.X, i), 0, d, n, stream);
    } else if (segmented()) {
        TQ_REQUIRE(slice >= 0 && slice < S, "slice out of range");
        launch_convert(prec, (uint8_t *)XG + (prec ? 8 : 4) * (long long)slice * n, 0, d, n, stream);
    } else {
        const int i0 = local(slice, 0);
        bool all = i0 >= 0;
        for (int m = 0; m < M && all; m++) all = local(slice, m) == i0 + m;
        if (!all) fail(TQ_EINVAL, "node=-1 (mean image) needs every node of the slice on this rank");
        if (prec == 0) mean_rows<float><<<blocks, 256, 0, stream>>>((const float *)in.xrow(in.X, i0), M, n, d);
        else mean_rows<double><<<blocks, 256, 0, stream>>>((const double *)in.xrow(in.X, i0), M, n, d);
        TQ_CHECK_CUDA(cudaGetLastError());
    }
}

void Ctx::get_image(int slice, int node, float *out, long long len, bool on_device) {
    Nvtx nv("tq:get_image");
    TQ_REQUIRE(len == n, "image length must be N*N");
    finish();
    TQ_CHECK_CUDA(cudaSetDevice(device));
    const float *src = nullptr;
    if (prec == 0 && node >= 0) {  // fp32 state: copied out directly
        const int i = local(slice, node);
        if (i < 0) fail(TQ_EINVAL, "node is not local to this rank");
        src = (const float *)in.xrow(in.X, i);
    } else if (prec == 0 && segmented()) {
        TQ_REQUIRE(slice >= 0 && slice < S, "slice out of range");
        src = (const float *)((uint8_t *)XG + 4 * (long long)slice * n);
    } else {
        if (!img_stage) TQ_CHECK_CUDA(cudaMalloc(&img_stage, sizeof(float) * n));
        snapshot_image(slice, node, img_stage, stream);
        src = img_stage;
    }
    TQ_CHECK_CUDA(cudaMemcpyAsync(out, src, sizeof(float) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream));
    TQ_CHECK_CUDA(cudaStreamSynchronize(stream));
}

void Ctx::get_image_async(int slice, int node, float *out, long long len, bool on_device, cudaStream_t s) {
    Nvtx nv("tq:get_image_async");
    TQ_REQUIRE(len == n, "image length must be N*N");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    const int b = img_buf;
    if (!img_async[b]) {
        TQ_CHECK_CUDA(cudaMalloc(&img_async[b], sizeof(float) * n));
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&img_ready[b], cudaEventDisableTiming));
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&img_done[b], cudaEventDisableTiming));
    }
    // the snapshot goes behind the last enqueued run on its stream (or on the context's own
    // stream when none is pending), once this buffer's previous copy has left
    cudaStream_t ss = pending ? run_s : stream;
    if (img_used[b]) wait_unless_done(ss, img_done[b]);
    snapshot_image(slice, node, img_async[b], ss);
    TQ_CHECK_CUDA(cudaEventRecord(img_ready[b], ss));
    img_s[b] = ss;
    TQ_CHECK_CUDA(cudaStreamWaitEvent(s, img_ready[b], 0));
    TQ_CHECK_CUDA(cudaMemcpyAsync(out, img_async[b], sizeof(float) * n,
                                  on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    TQ_CHECK_CUDA(cudaEventRecord(img_done[b], s));
    img_used[b] = true;
    img_buf ^= 1;
}

static void to_host_double(int prec, const void *src, double *dst, long long n, cudaStream_t s) {
    double *d = nullptr;
    TQ_CHECK_CUDA(cudaMalloc(&d, sizeof(double) * n));
    launch_convert(prec, src, 1, d, n, s);
    TQ_CHECK_CUDA(cudaMemcpyAsync(dst, d, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    TQ_CHECK_CUDA(cudaStreamSynchronize(s));
    cudaFree(d);
}

static void from_host_double(int prec, const double *src, void *dst, long long n, cudaStream_t s) {
    double *d = nullptr;
    TQ_CHECK_CUDA(cudaMalloc(&d, sizeof(double) * n));
    TQ_CHECK_CUDA(cudaMemcpyAsync(d, src, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    launch_convert(1, d, prec, dst, n, s);
    TQ_CHECK_CUDA(cudaStreamSynchronize(s));
    cudaFree(d);
}

void Ctx::export_state(int slice, int node, double *buf, long long len) {
    TQ_REQUIRE(len == 3 * n, "state length must be 3*N*N");
    finish();
    const int i = local(slice, node);
    TQ_REQUIRE(i >= 0, "node is not local to this rank");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    if (!xready) setup_exchange();
    const size_t es = prec ? 8 : 4;
    to_host_double(prec, in.xrow(in.X, i), buf, n, stream);
    to_host_double(prec, (uint8_t *)ALPHA + es * n * i, buf + n, n, stream);
    if (segmented()) {
        to_host_double(prec, (uint8_t *)XG + es * n * slice, buf + 2 * n, n, stream);
    } else {
        const int k = pay_of.at({slice, node});
        const void *xh = pays[k].kind == TQ_Q_NONE ? pays[k].buf : nullptr;
        if (!xh) {  // decoded buffer of the own payload
            std::vector<const void *> tab((size_t)pays.size());
            TQ_CHECK_CUDA(cudaMemcpy(tab.data(), xh_tab, sizeof(void *) * pays.size(), cudaMemcpyDeviceToHost));
            xh = tab[k];
        }
        to_host_double(prec, xh, buf + 2 * n, n, stream);
    }
}

void Ctx::import_state(int slice, int node, const double *buf, long long len) {
    TQ_REQUIRE(len == 3 * n, "state length must be 3*N*N");
    finish();
    const int i = local(slice, node);
    TQ_REQUIRE(i >= 0, "node is not local to this rank");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    if (!xready) setup_exchange();
    const size_t es = prec ? 8 : 4;
    from_host_double(prec, buf, in.xrow(in.X, i), n, stream);
    ax_valid = false;  // x changed outside a solve
    from_host_double(prec, buf + n, (uint8_t *)ALPHA + es * n * i, n, stream);
    if (segmented()) {
        from_host_double(prec, buf + 2 * n, (uint8_t *)XG + es * n * slice, n, stream);
    } else {
        const int k = pay_of.at({slice, node});
        if (pays[k].kind != TQ_Q_NONE) {
            std::vector<void *> tab((size_t)pays.size());
            TQ_CHECK_CUDA(cudaMemcpy(tab.data(), xh_tab, sizeof(void *) * pays.size(), cudaMemcpyDeviceToHost));
            from_host_double(prec, buf + 2 * n, tab[k], n, stream);
        }
    }
    need_rhs = true;
}

void Ctx::export_labels(int slice, int node, int32_t *buf, long long len) {
    finish();
    const int i = local(slice, node);
    TQ_REQUIRE(i >= 0, "node is not local to this rank");
    TQ_REQUIRE(xready && (int)label_row.size() == L && label_row[i] >= 0,
               "labels not kept (set keep_labels and a K-means quantizer, then run)");
    TQ_REQUIRE(len == payload_len, "labels length must equal the payload length");
    TQ_CHECK_CUDA(cudaMemcpy(buf, labels_buf + (long long)label_row[i] * payload_len, sizeof(int32_t) * len,
                             cudaMemcpyDeviceToHost));
}

}  // namespace tq
