// transport.cu -- see transport.cuh.
#include <dlfcn.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>

#include "transport.cuh"

namespace tq {

// ---------------------------------------------------------------- NCCL (dlopen'd)
NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        bool ok = true;
        auto sym = [&](const char *name) {
            void *p = dlsym(h, name);
            if (!p) ok = false;
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.Reduce = (decltype(api.Reduce))sym("ncclReduce");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        if (ok) api.h = h;
    });
    if (!api.h) fail(TQ_ENCCL, "libnccl.so.2 could not be loaded");
    return api;
}

#define TQ_CHECK_NCCL(call)                                                                       \
    do {                                                                                          \
        ncclResult_t _r = (call);                                                                 \
        if (_r != ncclSuccess)                                                                    \
            ::tq::fail(TQ_ENCCL, std::string(#call) + ": " + ::tq::nccl().GetErrorString(_r));    \
    } while (0)

namespace {

// ---------------------------------------------------------------- NCCL transport
struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    double *dscal = nullptr;
    const char *name() const override { return "nccl"; }
    bool collective_exchange() const override { return false; }
    NcclTransport(const uint8_t id[128], int r, int w, int dev) {
        rank = r; world = w; device = dev;
        ncclUniqueId u;
        static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
        memcpy(&u, id, sizeof(u));
        TQ_CHECK_CUDA(cudaSetDevice(device));
        TQ_CHECK_NCCL(nccl().CommInitRank(&comm, world, u, rank));
        TQ_CHECK_CUDA(cudaMalloc(&dscal, sizeof(double)));
    }
    ~NcclTransport() override {
        if (comm) nccl().CommDestroy(comm);
        if (dscal) cudaFree(dscal);
    }
    void exchange(cudaStream_t s, const std::vector<XferDesc> &sends, const std::vector<XferDesc> &recvs) override {
        if (sends.empty() && recvs.empty()) return;
        NcclApi &api = nccl();
        TQ_CHECK_NCCL(api.GroupStart());
        for (const XferDesc &x : sends)
            TQ_CHECK_NCCL(api.Send(x.buf, (size_t)x.bytes, ncclUint8, x.peer, comm, s));
        for (const XferDesc &x : recvs)
            TQ_CHECK_NCCL(api.Recv(x.buf, (size_t)x.bytes, ncclUint8, x.peer, comm, s));
        TQ_CHECK_NCCL(api.GroupEnd());
    }
    void reduce_sum(cudaStream_t s, double *base, const std::vector<SumSeg> &segs) override {
        NcclApi &api = nccl();
        TQ_CHECK_NCCL(api.GroupStart());
        for (const SumSeg &g : segs)
            TQ_CHECK_NCCL(api.Reduce(base + g.off, base + g.off, (size_t)g.count, ncclFloat64, ncclSum, g.root, comm, s));
        TQ_CHECK_NCCL(api.GroupEnd());
    }
    double allreduce_max(double v, cudaStream_t s) override {
        TQ_CHECK_CUDA(cudaMemcpyAsync(dscal, &v, sizeof(double), cudaMemcpyHostToDevice, s));
        TQ_CHECK_NCCL(nccl().AllReduce(dscal, dscal, 1, ncclFloat64, ncclMax, comm, s));
        TQ_CHECK_CUDA(cudaMemcpyAsync(&v, dscal, sizeof(double), cudaMemcpyDeviceToHost, s));
        TQ_CHECK_CUDA(cudaStreamSynchronize(s));
        return v;
    }
};

// ---------------------------------------------------------------- in-process loopback
constexpr char kLoopMagic[8] = {'T', 'Q', 'L', 'O', 'O', 'P', 'B', 'K'};
constexpr int kLoopMaxWorld = 64;

struct LoopWorld {
    int size = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    bool broken = false;
    struct Slot {
        bool joined = false;
        int device = 0;
        cudaEvent_t ready = nullptr, done = nullptr;
        const std::vector<XferDesc> *sends = nullptr;
        double *sum_base = nullptr;
        double hv = 0.0;
    };
    std::vector<Slot> slot;

    // all `size` ranks meet (generation counting, reusable); a rank that does not arrive
    // within the timeout breaks the world for everyone (no rank hangs forever)
    void barrier() {
        const char *env = getenv("TQ_LOOPBACK_TIMEOUT_S");
        const double tmo = env && atof(env) > 0 ? atof(env) : 120.0;
        std::unique_lock<std::mutex> lk(m);
        if (broken) fail(TQ_ENCCL, "loopback world broken (a peer failed or timed out)");
        const unsigned long long g = gen;
        if (++arrived == size) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(tmo), [&] { return gen != g || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            fail(TQ_ENCCL, "loopback rendezvous timed out (a peer never reached the same call)");
        }
    }
};

std::mutex g_reg_m;
std::map<unsigned long long, std::weak_ptr<LoopWorld>> g_reg;

// out[i] = src_0[i] + src_1[i] + ... in rank order (fixed order: deterministic)
struct SumSrc {
    const double *p[kLoopMaxWorld];
};
__global__ void sum_ranks(double *out, SumSrc src, int nsrc, long long count) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        double acc = src.p[0][i];
        for (int q = 1; q < nsrc; q++) acc += src.p[q][i];
        out[i] = acc;
    }
}

struct LoopTransport : Transport {
    std::shared_ptr<LoopWorld> W;
    double *scratch = nullptr;
    long long scratch_len = 0;
    const char *name() const override { return "loopback"; }
    bool collective_exchange() const override { return true; }

    LoopTransport(const uint8_t id[128], int r, int w, int dev) {
        rank = r; world = w; device = dev;
        TQ_REQUIRE(w <= kLoopMaxWorld, "loopback world size must be <= 64");
        unsigned long long key;
        memcpy(&key, id + 8, sizeof key);
        {
            std::lock_guard<std::mutex> lk(g_reg_m);
            auto it = g_reg.find(key);
            if (it != g_reg.end()) W = it->second.lock();
            if (!W) {
                W = std::make_shared<LoopWorld>();
                W->size = w;
                W->slot.resize(w);
                g_reg[key] = W;
            }
        }
        std::lock_guard<std::mutex> lk(W->m);
        TQ_REQUIRE(W->size == w, "loopback id used with a different world size");
        TQ_REQUIRE(!W->slot[r].joined, "loopback rank joined twice");
        TQ_CHECK_CUDA(cudaSetDevice(device));
        LoopWorld::Slot &sl = W->slot[r];
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
        TQ_CHECK_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
        sl.device = device;
        sl.joined = true;
        // ranks on other GPUs: direct peer copies over NVLink where the driver allows it
        for (int q = 0; q < w; q++) {
            if (q == r || !W->slot[q].joined || W->slot[q].device == device) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, device, W->slot[q].device);
            if (can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(W->slot[q].device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TQ_CHECK_CUDA(e);
                (void)cudaGetLastError();
            }
        }
    }
    ~LoopTransport() override {
        if (scratch) cudaFree(scratch);
        std::lock_guard<std::mutex> lk(W->m);
        LoopWorld::Slot &sl = W->slot[rank];
        if (sl.ready) cudaEventDestroy(sl.ready);
        if (sl.done) cudaEventDestroy(sl.done);
        sl = LoopWorld::Slot();
    }

    void wait_peers_done(cudaStream_t s) {
        for (int q = 0; q < world; q++)
            if (q != rank) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, W->slot[q].done, 0));
    }

    void exchange(cudaStream_t s, const std::vector<XferDesc> &sends, const std::vector<XferDesc> &recvs) override {
        LoopWorld::Slot &me = W->slot[rank];
        me.sends = &sends;
        TQ_CHECK_CUDA(cudaEventRecord(me.ready, s));
        W->barrier();  // every rank's payloads are enqueued (ready recorded) and published
        std::set<int> waited;
        for (const XferDesc &r : recvs) {
            const LoopWorld::Slot &ps = W->slot[r.peer];
            const XferDesc *src = nullptr;
            for (const XferDesc &x : *ps.sends)
                if (x.peer == rank && x.slice == r.slice && x.node == r.node) { src = &x; break; }
            TQ_REQUIRE(src != nullptr, "loopback: no matching send for a planned receive");
            TQ_REQUIRE(src->bytes == r.bytes, "loopback: send/receive sizes differ");
            if (waited.insert(r.peer).second) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, ps.ready, 0));
            TQ_CHECK_CUDA(cudaMemcpyAsync(r.buf, src->buf, (size_t)r.bytes, cudaMemcpyDefault, s));
        }
        TQ_CHECK_CUDA(cudaEventRecord(me.done, s));
        W->barrier();  // every receive is enqueued (done recorded)
        wait_peers_done(s);  // senders keep their payloads until every receiver has its copy
    }

    void reduce_sum(cudaStream_t s, double *base, const std::vector<SumSeg> &segs) override {
        LoopWorld::Slot &me = W->slot[rank];
        me.sum_base = base;
        TQ_CHECK_CUDA(cudaEventRecord(me.ready, s));
        W->barrier();
        long long need = 0;
        for (const SumSeg &g : segs)
            if (g.root == rank) need += g.count * (world - 1);
        if (need > scratch_len) {
            TQ_CHECK_CUDA(cudaStreamSynchronize(s));
            if (scratch) cudaFree(scratch);
            scratch = nullptr;
            TQ_CHECK_CUDA(cudaMalloc(&scratch, sizeof(double) * need));
            scratch_len = need;
        }
        bool waited = false;
        long long at = 0;
        for (const SumSeg &g : segs) {
            if (g.root != rank) continue;
            if (!waited) {
                for (int q = 0; q < world; q++)
                    if (q != rank) TQ_CHECK_CUDA(cudaStreamWaitEvent(s, W->slot[q].ready, 0));
                waited = true;
            }
            SumSrc src{};
            for (int q = 0; q < world; q++) {
                if (q == rank) { src.p[q] = base + g.off; continue; }
                double *dst = scratch + at;
                at += g.count;
                TQ_CHECK_CUDA(cudaMemcpyAsync(dst, W->slot[q].sum_base + g.off, sizeof(double) * g.count,
                                              cudaMemcpyDefault, s));
                src.p[q] = dst;
            }
            const int blocks = (int)std::min<long long>(1184, (g.count + 255) / 256);
            if (g.count > 0) sum_ranks<<<std::max(1, blocks), 256, 0, s>>>(base + g.off, src, world, g.count);
            TQ_CHECK_CUDA(cudaGetLastError());
        }
        TQ_CHECK_CUDA(cudaEventRecord(me.done, s));
        W->barrier();
        wait_peers_done(s);  // partial sums stay until every owner has read them
    }

    void host_fence() override { W->barrier(); }

    double allreduce_max(double v, cudaStream_t s) override {
        (void)s;
        W->slot[rank].hv = v;
        W->barrier();
        double m = v;
        for (int q = 0; q < world; q++) m = std::max(m, W->slot[q].hv);
        W->barrier();  // nobody overwrites hv before every rank has read it
        return m;
    }
};

}  // namespace

bool is_loopback_id(const uint8_t id[128]) { return id && memcmp(id, kLoopMagic, 8) == 0; }

void new_loopback_id(uint8_t id[128]) {
    static std::atomic<unsigned long long> counter{1};
    memset(id, 0, 128);
    memcpy(id, kLoopMagic, 8);
    const unsigned long long key = ((unsigned long long)getpid() << 32) ^ counter.fetch_add(1);
    memcpy(id + 8, &key, sizeof key);
}

std::unique_ptr<Transport> make_transport(const uint8_t id[128], int rank, int world, int device) {
    TQ_REQUIRE(id != nullptr, "world > 1 needs a transport id (tq_nccl_unique_id or tq_loopback_id)");
    if (is_loopback_id(id)) return std::unique_ptr<Transport>(new LoopTransport(id, rank, world, device));
    return std::unique_ptr<Transport>(new NcclTransport(id, rank, world, device));
}


// ---------------------------------------------------------------- transport self-check
// Every operation of the Transport interface on a synthetic plan (tq_debug_transport_check):
// each rank sends `bytes` bytes to every rank including itself (a self send / receive is an
// ordinary NCCL point-to-point pair), then sums `n_doubles` doubles over the ranks onto
// segment owners (segment g of `world`, owner g), then takes the maximum of the rank ids.
// Byte k sent from rank a to rank b is pattern(a, b, k); element i of rank a's sum buffer is
// a + 1 + i / 2, so every expected value is exact and known on the host.
namespace {
inline uint8_t xcheck_byte(int a, int b, long long k) {
    return (uint8_t)(a * 37 + b * 11 + k * 7 + (k >> 8));
}
}  // namespace

void transport_check(const uint8_t id[128], int rank, int world, int device, long long bytes, long long n_doubles,
                     int rounds) {
    TQ_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
    TQ_REQUIRE(bytes >= 1 && n_doubles >= 1 && rounds >= 1, "bytes, n_doubles and rounds must be >= 1");
    TQ_CHECK_CUDA(cudaSetDevice(device));
    std::unique_ptr<Transport> tr = make_transport(id, rank, world, device);
    cudaStream_t s = nullptr;
    TQ_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint8_t *sbuf = nullptr, *rbuf = nullptr;
    double *sum = nullptr;
    std::string bad;
    try {
        TQ_CHECK_CUDA(cudaMalloc(&sbuf, (size_t)bytes * world));
        TQ_CHECK_CUDA(cudaMalloc(&rbuf, (size_t)bytes * world));
        TQ_CHECK_CUDA(cudaMalloc(&sum, sizeof(double) * (size_t)n_doubles));
        std::vector<uint8_t> hs((size_t)bytes * world), hr((size_t)bytes * world);
        for (int q = 0; q < world; q++)
            for (long long k = 0; k < bytes; k++) hs[(size_t)q * bytes + k] = xcheck_byte(rank, q, k);
        std::vector<double> hsum((size_t)n_doubles);
        // segment g = [g * per, ...) owned by rank g (the last one takes the remainder)
        std::vector<SumSeg> segs;
        const long long per = n_doubles / world;
        for (int g = 0; g < world; g++) {
            const long long off = g * per, cnt = g + 1 < world ? per : n_doubles - off;
            if (cnt > 0) segs.push_back({off, cnt, g});
        }
        std::vector<XferDesc> sends, recvs;  // sorted by (peer, node) as the engine's plan
        for (int q = 0; q < world; q++) {
            sends.push_back({0, rank, q, sbuf + (size_t)q * bytes, bytes});
            recvs.push_back({0, q, q, rbuf + (size_t)q * bytes, bytes});
        }
        for (int round = 0; round < rounds && bad.empty(); round++) {
            for (long long i = 0; i < n_doubles; i++) hsum[(size_t)i] = rank + 1 + 0.5 * (double)i + round;
            TQ_CHECK_CUDA(cudaMemcpyAsync(sbuf, hs.data(), hs.size(), cudaMemcpyHostToDevice, s));
            TQ_CHECK_CUDA(cudaMemsetAsync(rbuf, 0, hr.size(), s));
            TQ_CHECK_CUDA(cudaMemcpyAsync(sum, hsum.data(), sizeof(double) * hsum.size(), cudaMemcpyHostToDevice, s));
            tr->exchange(s, sends, recvs);
            tr->reduce_sum(s, sum, segs);
            TQ_CHECK_CUDA(cudaMemcpyAsync(hr.data(), rbuf, hr.size(), cudaMemcpyDeviceToHost, s));
            TQ_CHECK_CUDA(cudaMemcpyAsync(hsum.data(), sum, sizeof(double) * hsum.size(), cudaMemcpyDeviceToHost, s));
            TQ_CHECK_CUDA(cudaStreamSynchronize(s));
            const double mx = tr->allreduce_max((double)rank + round, s);
            for (int q = 0; q < world && bad.empty(); q++)
                for (long long k = 0; k < bytes; k++)
                    if (hr[(size_t)q * bytes + k] != xcheck_byte(q, rank, k)) {
                        bad = "exchange: byte " + std::to_string(k) + " from rank " + std::to_string(q) + " differs";
                        break;
                    }
            const double rs = 0.5 * world * (world + 1) + (double)world * round;  // sum of (a + 1 + round)
            for (const SumSeg &g : segs) {
                if (g.root != rank || !bad.empty()) continue;
                for (long long i = g.off; i < g.off + g.count; i++)
                    if (hsum[(size_t)i] != rs + 0.5 * (double)world * (double)i) {
                        bad = "reduce_sum: element " + std::to_string(i) + " differs";
                        break;
                    }
            }
            if (bad.empty() && mx != (double)(world - 1 + round)) bad = "allreduce_max differs";
        }
    } catch (...) {
        if (sbuf) cudaFree(sbuf);
        if (rbuf) cudaFree(rbuf);
        if (sum) cudaFree(sum);
        cudaStreamDestroy(s);
        throw;
    }
    cudaFree(sbuf);
    cudaFree(rbuf);
    cudaFree(sum);
    cudaStreamDestroy(s);
    if (!bad.empty()) fail(TQ_ENCCL, std::string(tr->name()) + " transport check failed: " + bad);
}

}  // namespace tq
