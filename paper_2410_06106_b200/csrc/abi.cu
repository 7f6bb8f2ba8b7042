// abi.cu -- the extern "C" boundary of libtomoq.so (include/tomoq.h).  Every entry
// point converts internal errors (tq::Error, std::bad_alloc) into a tq_status and a
// message; nothing throws across the boundary.
#include <cstring>
#include <new>

#include "engine.cuh"

using namespace tq;

struct tq_ctx {
    Ctx c;
};

namespace {
thread_local std::string g_err;

template <typename F>
tq_status guard(tq_ctx *ctx, F &&f) {
    try {
        f();
        if (ctx) ctx->c.err.clear();
        return TQ_OK;
    } catch (const Error &e) {
        (ctx ? ctx->c.err : g_err) = e.msg;
        if (ctx) g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc &) {
        (ctx ? ctx->c.err : g_err) = "host allocation failed";
        return TQ_ENOMEM;
    } catch (const std::exception &e) {
        (ctx ? ctx->c.err : g_err) = e.what();
        return TQ_EINVAL;
    }
}

void check_geom(const tq_geometry *g) {
    TQ_REQUIRE(g != nullptr, "null geometry");
    TQ_REQUIRE(g->image_side >= 1 && g->n_angles >= 1, "bad geometry");
    TQ_REQUIRE(g->projector == TQ_PROJ_JOSEPH || g->projector == TQ_PROJ_SIDDON, "bad projector");
    TQ_REQUIRE((long long)g->n_det * g->n_det >= 2LL * g->image_side * g->image_side,
               "n_det must be >= ceil(N sqrt 2)");
    check_angles(g->angles_rad, g->n_angles);
}

// device scratch released at scope exit
struct DevTmp {
    std::vector<void *> p;
    void *get(size_t bytes) {
        void *q = nullptr;
        TQ_CHECK_CUDA(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
        p.push_back(q);
        return q;
    }
    template <typename T>
    T *up(const T *src, size_t count) {
        T *d = (T *)get(sizeof(T) * count);
        TQ_CHECK_CUDA(cudaMemcpy(d, src, sizeof(T) * count, cudaMemcpyHostToDevice));
        return d;
    }
    ~DevTmp() {
        for (void *q : p) cudaFree(q);
    }
};

std::vector<int> check_sel(const tq_geometry *g, const int32_t *sel, int n_sel) {
    TQ_REQUIRE(n_sel >= 1 && sel != nullptr, "need at least one angle");
    std::vector<int> s(sel, sel + n_sel);
    for (int a : s) TQ_REQUIRE(a >= 0 && a < g->n_angles, "angle id out of range");
    return s;
}

}  // namespace

extern "C" {

tq_status tq_nccl_unique_id(uint8_t id[128]) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(id != nullptr, "null id");
        ncclUniqueId u;
        ncclResult_t r = nccl().GetUniqueId(&u);
        if (r != ncclSuccess) fail(TQ_ENCCL, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
        memcpy(id, &u, 128);
    });
}

tq_status tq_loopback_id(uint8_t id[128]) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(id != nullptr, "null id");
        new_loopback_id(id);
    });
}

tq_status tq_create(const tq_geometry *geom, const tq_graph *graph, int32_t n_slices, int32_t rank,
                    int32_t world, const uint8_t *nccl_id, int32_t precision, int32_t device,
                    tq_ctx **out) {
    if (out) *out = nullptr;
    tq_ctx *c = nullptr;
    tq_status s = guard(nullptr, [&] {
        TQ_REQUIRE(geom && graph && out, "null argument");
        c = new tq_ctx();
        c->c.create(*geom, *graph, n_slices, rank, world, nccl_id, precision, device);
    });
    if (s != TQ_OK) {
        if (c) {
            try { c->c.destroy(); } catch (...) {}
            delete c;
        }
        return s;
    }
    *out = c;
    return TQ_OK;
}

tq_status tq_set_params(tq_ctx *ctx, const tq_params *p) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(p != nullptr, "null params");
        ctx->c.set_params(*p);
    });
}

tq_status tq_set_quantizer(tq_ctx *ctx, const tq_quant *q) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(q != nullptr, "null quantizer");
        ctx->c.set_quant(*q);
    });
}

tq_status tq_set_sinogram(tq_ctx *ctx, int32_t slice, int32_t node, const float *d, int64_t len,
                          int32_t on_device) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.set_sinogram(slice, node, d, len, on_device != 0); });
}

tq_status tq_set_sinogram_stream(tq_ctx *ctx, int32_t slice, int32_t node, const float *d, int64_t len,
                                 void *stream) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.set_sinogram(slice, node, d, len, true, (cudaStream_t)stream, true); });
}

tq_status tq_run(tq_ctx *ctx, int32_t iters, void *stream) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.run(iters, (cudaStream_t)stream); });
}

tq_status tq_run_async(tq_ctx *ctx, int32_t iters, void *stream) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.run_async(iters, (cudaStream_t)stream); });
}

tq_status tq_wait(tq_ctx *ctx) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.finish(); });
}

tq_status tq_get_image(tq_ctx *ctx, int32_t slice, int32_t node, float *out, int64_t len,
                       int32_t on_device) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(out != nullptr, "null output");
        ctx->c.get_image(slice, node, out, len, on_device != 0);
    });
}

tq_status tq_get_image_async(tq_ctx *ctx, int32_t slice, int32_t node, float *out, int64_t len,
                             int32_t on_device, void *stream) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(out != nullptr, "null output");
        ctx->c.get_image_async(slice, node, out, len, on_device != 0, (cudaStream_t)stream);
    });
}

tq_status tq_export_state(tq_ctx *ctx, int32_t slice, int32_t node, double *buf, int64_t len) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(buf != nullptr, "null buffer");
        ctx->c.export_state(slice, node, buf, len);
    });
}

tq_status tq_import_state(tq_ctx *ctx, int32_t slice, int32_t node, const double *buf, int64_t len) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(buf != nullptr, "null buffer");
        TQ_REQUIRE(ctx->c.world == 1 || ctx->c.rule != TQ_RULE_GRAPH,
                   "import_state with the graph rule needs world == 1 (neighbour values)");
        ctx->c.import_state(slice, node, buf, len);
    });
}

tq_status tq_export_labels(tq_ctx *ctx, int32_t slice, int32_t node, int32_t *buf, int64_t len) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(buf != nullptr, "null buffer");
        ctx->c.export_labels(slice, node, buf, len);
    });
}

tq_status tq_launch_component(tq_ctx *ctx, int32_t component, int32_t reps, void *stream,
                              int64_t *units) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        const long long u = ctx->c.launch_component(component, reps, stream ? (cudaStream_t)stream : ctx->c.stream);
        if (units) *units = u;
    });
}

tq_status tq_get_stats(const tq_ctx *ctx, tq_stats *out) {
    if (!ctx || !out) return TQ_EINVAL;
    tq_ctx *c = const_cast<tq_ctx *>(ctx);  // the handle is never a const object
    const tq_status r = guard(c, [&] { c->c.finish(); });
    *out = ctx->c.st;
    return r;
}

tq_status tq_set_profiling(tq_ctx *ctx, int32_t on) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] { ctx->c.set_profiling(on != 0); });
}

tq_status tq_get_node_bytes(tq_ctx *ctx, int32_t slice, int32_t node, int64_t *sent, int64_t *recv) {
    if (!ctx) return TQ_EINVAL;
    return guard(ctx, [&] {
        TQ_REQUIRE(sent && recv, "null output");
        long long s = 0, r = 0;
        ctx->c.node_bytes(slice, node, s, r);
        *sent = s;
        *recv = r;
    });
}

tq_status tq_debug_guard_check(void) {
    return guard(nullptr, [&] {
        std::string where;
        if (!guards_intact(where)) fail(TQ_ECUDA, "TQ_GUARD: guard band corrupted: " + where);
    });
}

tq_status tq_debug_transport_check(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                                   int64_t bytes, int64_t n_doubles, int32_t rounds) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(id != nullptr, "null transport id");
        transport_check(id, rank, world, device, bytes, n_doubles, rounds);
    });
}

const char *tq_last_error(const tq_ctx *ctx) { return ctx ? ctx->c.err.c_str() : g_err.c_str(); }
const char *tq_last_error_global(void) { return g_err.c_str(); }

void tq_destroy(tq_ctx *ctx) {
    if (!ctx) return;
    try { ctx->c.destroy(); } catch (...) {}
    delete ctx;
}

// ---------------------------------------------------------------- host-side plans
tq_status tq_partition_angles(int32_t n_angles, int32_t n_nodes, int32_t split, int32_t *offsets,
                              int32_t *idx) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(n_nodes >= 1 && n_nodes <= n_angles && offsets && idx, "bad partition arguments");
        std::vector<int> off, ix;
        partition_angles(n_angles, n_nodes, split, off, ix);
        std::copy(off.begin(), off.end(), offsets);
        std::copy(ix.begin(), ix.end(), idx);
    });
}

tq_status tq_exchange_plan(const tq_graph *graph, int32_t rank, int32_t world, int32_t *sends,
                           int32_t cap_sends, int32_t *n_sends, int32_t *recvs, int32_t cap_recvs,
                           int32_t *n_recvs) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(graph && n_sends && n_recvs, "null argument");
        TQ_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        const int M = graph->n_nodes;
        std::vector<int> edges(graph->edges, graph->edges + 2 * (size_t)graph->n_edges), nr(M);
        for (int i = 0; i < M; i++) nr[i] = graph->node_rank ? graph->node_rank[i] : i % world;
        std::vector<std::pair<int, int>> s, r;
        exchange_plan(M, edges, nr, graph->rule, rank, world, s, r);
        *n_sends = (int32_t)s.size();
        *n_recvs = (int32_t)r.size();
        TQ_REQUIRE((int)s.size() <= cap_sends && (int)r.size() <= cap_recvs, "plan capacity too small");
        for (size_t i = 0; i < s.size(); i++) { sends[2 * i] = s[i].first; sends[2 * i + 1] = s[i].second; }
        for (size_t i = 0; i < r.size(); i++) { recvs[2 * i] = r[i].first; recvs[2 * i + 1] = r[i].second; }
    });
}

int64_t tq_payload_bytes(int32_t kind, int32_t k, int64_t n, int32_t precision) {
    if (kind == TQ_Q_KMEANS) return kmeans_payload_bytes(k, n);
    if (kind == TQ_Q_DCT) return dct_payload_bytes(n);
    return (precision ? 8 : 4) * n;
}

// ---------------------------------------------------------------- stateless kernels
tq_status tq_project(const tq_geometry *g, const int32_t *sel, int32_t n_sel, const void *img,
                     void *sino, int32_t precision, void *stream) {
    return guard(nullptr, [&] {
        check_geom(g);
        TQ_REQUIRE(img && sino && (precision == 0 || precision == 1), "bad arguments");
        std::vector<int> s = check_sel(g, sel, n_sel);
        DevGeom geo;
        geo.init(g->image_side, g->n_angles, g->n_det, g->projector, g->angles_rad);
        Inner in;
        in.init(precision, geo, {s});
        cudaStream_t st = (cudaStream_t)stream;
        in.project(geo, img, false, st, sino, g->n_det, 0);
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        in.release();
        geo.release();
    });
}

tq_status tq_backproject(const tq_geometry *g, const int32_t *sel, int32_t n_sel, const void *sino,
                         void *img, int32_t precision, void *stream) {
    return guard(nullptr, [&] {
        check_geom(g);
        TQ_REQUIRE(img && sino && (precision == 0 || precision == 1), "bad arguments");
        std::vector<int> s = check_sel(g, sel, n_sel);
        DevGeom geo;
        geo.init(g->image_side, g->n_angles, g->n_det, g->projector, g->angles_rad);
        DevTmp t;
        std::vector<RayRow> rows;
        for (int k = 0; k < n_sel; k++) rows.push_back(RayRow{0, s[k], k, 0});
        RayRow *rd = t.up(rows.data(), rows.size());
        const int zero = 0;
        int *row0 = t.up(&zero, 1), *nang = t.up(&n_sel, 1);
        cudaStream_t st = (cudaStream_t)stream;
        // guarded copy: zero bins at 0 and n_det + 1 of every row, SPAD zeros around (BpArgs::s)
        const size_t es = precision ? 8 : 4;
        const long long sp = g->n_det + 2;
        uint8_t *gs = (uint8_t *)t.get(es * ((size_t)n_sel * sp + 2 * SPAD));
        TQ_CHECK_CUDA(cudaMemsetAsync(gs, 0, es * ((size_t)n_sel * sp + 2 * SPAD), st));
        TQ_CHECK_CUDA(cudaMemcpy2DAsync(gs + es * (SPAD + 1), es * sp, sino, es * g->n_det, es * g->n_det, n_sel,
                                        cudaMemcpyDeviceToDevice, st));
        const void *sg = gs + es * SPAD;
        if (precision == 0) {
            BpArgs<float> a{};
            a.s = (const float *)sg; a.s_stride = (int)sp; a.s_off = 1;
            a.node_row0 = row0; a.node_nang = nang; a.rows = rd; a.trig = geo.trig; a.xmaj = geo.xmaj;
            a.N = g->image_side; a.n_det = g->n_det; a.n = geo.n; a.out = (float *)img; a.magic = kMagicBits4;
            a.siddon = geo.proj;
            launch_bp(0, EPI_PLAIN, &a, 1, g->image_side, st);
        } else {
            BpArgs<double> a{};
            a.s = (const double *)sg; a.s_stride = (int)sp; a.s_off = 1;
            a.node_row0 = row0; a.node_nang = nang; a.rows = rd; a.trig = geo.trig; a.xmaj = geo.xmaj;
            a.N = g->image_side; a.n_det = g->n_det; a.n = geo.n; a.out = (double *)img; a.magic = kMagicBits4;
            a.siddon = geo.proj;
            launch_bp(1, EPI_PLAIN, &a, 1, g->image_side, st);
        }
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        geo.release();
    });
}

tq_status tq_local_solve(const tq_geometry *g, const int32_t *sel, int32_t n_sel, const void *d,
                         const void *bprime, double c, int32_t inner, int32_t e1, double eta, void *x,
                         int32_t precision, void *stream) {
    return guard(nullptr, [&] {
        check_geom(g);
        TQ_REQUIRE(d && bprime && x && (precision == 0 || precision == 1), "bad arguments");
        TQ_REQUIRE(inner == TQ_INNER_GD || inner == TQ_INNER_CG, "bad inner solver");
        TQ_REQUIRE(e1 >= 0 && c >= 0.0, "bad e1 / c");
        std::vector<int> s = check_sel(g, sel, n_sel);
        DevGeom geo;
        geo.init(g->image_side, g->n_angles, g->n_det, g->projector, g->angles_rad);
        Inner in;
        in.init(precision, geo, {s});
        cudaStream_t st = (cudaStream_t)stream;
        const size_t es = precision ? 8 : 4;
        TQ_CHECK_CUDA(cudaMemcpyAsync(in.D, d, es * n_sel * g->n_det, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(in.BP, bprime, es * geo.n, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(in.X, x, es * geo.n, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(in.cnode, &c, sizeof(double), cudaMemcpyHostToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(in.eta, &eta, sizeof(double), cudaMemcpyHostToDevice, st));
        if (inner == TQ_INNER_CG) in.cg(geo, e1, st);
        else in.gd(geo, e1, st);
        TQ_CHECK_CUDA(cudaMemcpyAsync(x, in.X, es * geo.n, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        in.release();
        geo.release();
    });
}

tq_status tq_kmeans_encode(const float *v, int64_t n, int32_t k, int32_t iters, float *centers,
                           uint32_t *planes, int32_t *labels, void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(v && centers && (planes || k == 1) && n >= 1 && k >= 1 && k <= 256 && iters >= 0,
                   "bad kmeans arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long pb = kmeans_payload_bytes(k, n);
        uint8_t *pay = (uint8_t *)t.get(pb);
        const float **vt = t.up(&v, 1);
        uint8_t **pt = t.up(&pay, 1);
        int32_t **lt = labels ? t.up(&labels, 1) : nullptr;
        KmeansWork w;
        w.alloc(1, k, n);
        kmeans_encode(vt, w, iters, pt, lt, st);
        TQ_CHECK_CUDA(cudaMemcpyAsync(centers, pay, 4LL * k, cudaMemcpyDeviceToDevice, st));
        if (pb > 4LL * k)
            TQ_CHECK_CUDA(cudaMemcpyAsync(planes, pay + 4LL * k, pb - 4LL * k, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        w.release();
    });
}

tq_status tq_kmeans_decode(const float *centers, const uint32_t *planes, int64_t n, int32_t k,
                           float *out, void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(centers && out && (planes || k == 1) && n >= 1 && k >= 1 && k <= 256, "bad kmeans arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long pb = kmeans_payload_bytes(k, n);
        uint8_t *pay = (uint8_t *)t.get(pb);
        TQ_CHECK_CUDA(cudaMemcpyAsync(pay, centers, 4LL * k, cudaMemcpyDeviceToDevice, st));
        if (pb > 4LL * k)
            TQ_CHECK_CUDA(cudaMemcpyAsync(pay + 4LL * k, planes, pb - 4LL * k, cudaMemcpyDeviceToDevice, st));
        const uint8_t **pt = (const uint8_t **)t.up(&pay, 1);
        void **ot = t.up((void **)&out, 1);
        kmeans_decode(pt, 1, n, k, 0, ot, st);
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
    });
}

tq_status tq_dct_encode(const float *v, int32_t rows, int32_t cols, int32_t quality, int16_t *coef,
                        float *minmax, void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(v && coef && minmax && rows > 0 && cols > 0 && rows % 8 == 0 && cols % 8 == 0 &&
                       quality >= 1 && quality <= 100,
                   "bad dct arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long nv = (long long)rows * cols;
        uint8_t *pay = (uint8_t *)t.get(dct_payload_bytes(nv));
        const float **vt = t.up(&v, 1);
        uint8_t **pt = t.up(&pay, 1);
        DctWork w;
        w.alloc(1, nv);
        dct_encode(vt, 1, rows, cols, quality, w, pt, st);
        TQ_CHECK_CUDA(cudaMemcpyAsync(minmax, pay, 8, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(coef, pay + 8, 2 * nv, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        w.release();
    });
}

tq_status tq_dct_decode(const int16_t *coef, const float *minmax, int32_t rows, int32_t cols,
                        int32_t quality, float *out, void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(coef && minmax && out && rows > 0 && cols > 0 && rows % 8 == 0 && cols % 8 == 0 &&
                       quality >= 1 && quality <= 100,
                   "bad dct arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long nv = (long long)rows * cols;
        uint8_t *pay = (uint8_t *)t.get(dct_payload_bytes(nv));
        TQ_CHECK_CUDA(cudaMemcpyAsync(pay, minmax, 8, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(pay + 8, coef, 2 * nv, cudaMemcpyDeviceToDevice, st));
        const uint8_t **pt = (const uint8_t **)t.up(&pay, 1);
        void **ot = t.up((void **)&out, 1);
        dct_decode(pt, 1, rows, cols, quality, 0, ot, st);
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
    });
}

tq_status tq_jpeg_encode(const int16_t *coef, int64_t n_blocks, int32_t restart, uint8_t *out, int64_t cap,
                         int64_t *nbytes, void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(coef && out && nbytes && n_blocks >= 1 && restart >= 1 && cap >= 0, "bad jpeg arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long nv = 64LL * n_blocks;
        uint8_t *pay = (uint8_t *)t.get(jpeg_payload_bytes(nv));
        TQ_CHECK_CUDA(cudaMemsetAsync(pay, 0, 8, st));
        uint8_t **pt = t.up(&pay, 1);
        JpegWork w;
        w.alloc(1, nv, restart);
        TQ_CHECK_CUDA(cudaMemcpyAsync(w.coef, coef, 2 * nv, cudaMemcpyDeviceToDevice, st));
        jpeg_encode(pt, w, st);
        unsigned stat[2];
        TQ_CHECK_CUDA(cudaMemcpyAsync(stat, w.status, sizeof stat, cudaMemcpyDeviceToHost, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        w.release();
        TQ_REQUIRE(!(stat[1] & 1u), "jpeg: a coefficient lies outside the baseline categories");
        TQ_REQUIRE(!(stat[0] & 0x80000000u), "jpeg: stream would exceed 2 bytes per coefficient");
        const long long n = stat[0];
        TQ_REQUIRE(n <= cap, "jpeg: output capacity too small");
        *nbytes = n;
        TQ_CHECK_CUDA(cudaMemcpyAsync(out, pay + 16, n, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
    });
}

tq_status tq_jpeg_decode(const uint8_t *in, int64_t nbytes, int64_t n_blocks, int32_t restart, int16_t *coef,
                         void *stream) {
    return guard(nullptr, [&] {
        TQ_REQUIRE(in && coef && n_blocks >= 1 && restart >= 1 && nbytes >= 0 && nbytes < (1LL << 31),
                   "bad jpeg arguments");
        cudaStream_t st = (cudaStream_t)stream;
        DevTmp t;
        const long long nv = 64LL * n_blocks;
        uint8_t *pay = (uint8_t *)t.get(16 + std::max<long long>(nbytes, 2 * nv));
        const uint32_t hdr[4] = {0u, 0u, (uint32_t)nbytes, (uint32_t)n_blocks};
        TQ_CHECK_CUDA(cudaMemcpyAsync(pay, hdr, sizeof hdr, cudaMemcpyHostToDevice, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(pay + 16, in, nbytes, cudaMemcpyDeviceToDevice, st));
        uint8_t **pt = t.up(&pay, 1);
        JpegWork w;
        w.alloc(1, nv, restart);
        jpeg_decode(pt, w, st);
        unsigned stat[2];
        TQ_CHECK_CUDA(cudaMemcpyAsync(stat, w.status, sizeof stat, cudaMemcpyDeviceToHost, st));
        TQ_CHECK_CUDA(cudaMemcpyAsync(coef, w.coef, 2 * nv, cudaMemcpyDeviceToDevice, st));
        TQ_CHECK_CUDA(cudaStreamSynchronize(st));
        w.release();
        TQ_REQUIRE(stat[1] == 0, "jpeg: malformed entropy-coded stream");
    });
}

}  // extern "C"
