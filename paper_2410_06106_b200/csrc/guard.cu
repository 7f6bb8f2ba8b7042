// guard.cu -- guarded device allocations (see common.cuh "guarded allocations").
#define TQ_NO_GUARD_MACROS
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"

namespace tq {

namespace {
constexpr size_t GB = 256;  // guard band bytes (keeps the 256-byte alignment of cudaMalloc)
constexpr unsigned char PATTERN = 0xA5;
std::mutex g_m;
std::map<void *, size_t> g_live;  // user pointer -> user bytes
}  // namespace

bool guards_enabled() {
    static const bool on = [] {
        const char *e = getenv("TQ_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}

cudaError_t guarded_malloc(void **p, size_t bytes) {
    if (!guards_enabled()) return cudaMalloc(p, bytes);
    void *base = nullptr;
    cudaError_t e = cudaMalloc(&base, bytes + 2 * GB);
    if (e != cudaSuccess) return e;
    unsigned char *b = static_cast<unsigned char *>(base);
    if ((e = cudaMemset(b, PATTERN, GB)) != cudaSuccess) return e;
    if ((e = cudaMemset(b + GB + bytes, PATTERN, GB)) != cudaSuccess) return e;
    if ((e = cudaMemset(b + GB, 0xff, bytes)) != cudaSuccess) return e;  // poison
    *p = b + GB;
    std::lock_guard<std::mutex> lk(g_m);
    g_live[*p] = bytes;
    return cudaSuccess;
}

cudaError_t guarded_free(void *p) {
    if (!guards_enabled() || p == nullptr) return cudaFree(p);
    {
        std::lock_guard<std::mutex> lk(g_m);
        auto it = g_live.find(p);
        if (it == g_live.end()) return cudaFree(p);  // not ours
        g_live.erase(it);
    }
    return cudaFree(static_cast<unsigned char *>(p) - GB);
}

// every live allocation's guard bands still hold the pattern (synchronises the device)
bool guards_intact(std::string &where) {
    if (!guards_enabled()) return true;
    if (cudaDeviceSynchronize() != cudaSuccess) { where = "device error"; return false; }
    std::lock_guard<std::mutex> lk(g_m);
    unsigned char h[2 * GB];
    for (auto &kv : g_live) {
        unsigned char *u = static_cast<unsigned char *>(kv.first);
        if (cudaMemcpy(h, u - GB, GB, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(h + GB, u + kv.second, GB, cudaMemcpyDeviceToHost) != cudaSuccess) {
            where = "guard read failed";
            return false;
        }
        for (size_t i = 0; i < 2 * GB; i++)
            if (h[i] != PATTERN) {
                where = "allocation of " + std::to_string(kv.second) + " bytes: " +
                        (i < GB ? "underrun" : "overrun") + " at byte " +
                        std::to_string(i < GB ? (long long)i - (long long)GB : (long long)(i - GB));
                return false;
            }
    }
    return true;
}


bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("TQ_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

}  // namespace tq
