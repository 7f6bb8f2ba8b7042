// common.cuh -- internal helpers of libtomoq (sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/tomoq.h"

namespace tq {

struct Error {
    tq_status code;
    std::string msg;
};

[[noreturn]] void fail(tq_status code, const std::string &msg);

#define TQ_CHECK_CUDA(call)                                                              \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess)                                                           \
            ::tq::fail(TQ_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));    \
    } while (0)

#define TQ_REQUIRE(cond, msg)                                                            \
    do {                                                                                 \
        if (!(cond)) ::tq::fail(TQ_EINVAL, msg);                                         \
    } while (0)

// ---------------------------------------------------------------- guarded allocations
// Debug aid standing in for compute-sanitizer (closed on the GPU pool): with TQ_GUARD=1 in the
// environment every device allocation of the library gets 256-byte guard bands filled with a
// pattern on both sides (checked after every run and at tq_destroy: an out-of-bounds write
// fails with TQ_ECUDA) and its contents poisoned with 0xff bytes (NaN / -1) instead of left
// undefined, so a read of memory nobody wrote changes the results (tests compare bitwise
// against an unguarded run).  Without TQ_GUARD these are plain cudaMalloc / cudaFree.
cudaError_t guarded_malloc(void **p, size_t bytes);
cudaError_t guarded_free(void *p);
bool guards_enabled();
bool guards_intact(std::string &where);
#ifndef TQ_NO_GUARD_MACROS
#define cudaMalloc(p, b) ::tq::guarded_malloc(reinterpret_cast<void **>(p), (b))
#define cudaFree(p) ::tq::guarded_free((void *)(p))
#endif

// ---------------------------------------------------------------- geometry (host)
// DESIGN.md R-1..R-3: theta_a = pi a / n_ang; x-major iff 4a in [n_ang, 3 n_ang];
// m_a = |sin| (x-major) or |cos| (y-major).  Explicit angle lists: x-major iff |sin| >= |cos|.
struct AngleHost {
    double cs, sn, m;
    int xmajor;
};
std::vector<AngleHost> make_angles(int n_ang, const double *angles_rad = nullptr);
// explicit angle lists: every angle in [0, pi) (the half turn of P:315; a parallel ray set repeats after pi)
void check_angles(const double *angles_rad, int n_ang);
void partition_angles(int n_ang, int M, int split, std::vector<int> &off, std::vector<int> &idx);
void partition_rows(int N, int M, std::vector<int> &row_off);

// Per-angle record used by the projector kernels (one per (local node, angle)).
struct RayRow {
    int node;      // local node index
    int angle;     // global angle id
    int k;         // index of the angle within the node
    int pad;
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block sum (deterministic): warp butterflies then warp 0 over the
// per-warp results.  All threads of the block must call it.  Result valid in
// every thread.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *sh /* >= NT/32 + 1 */) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        double t = (l < NT / 32) ? sh[l] : 0.0;
        t = warp_sum(t);
        if (l == 0) sh[NT / 32] = t;
    }
    __syncthreads();
    return sh[NT / 32];
}

// "Last block finalises": every block of a group has thread 0 write its partial, then
// the last block to arrive sums all partials in index order (deterministic) and resets
// the counter.  Only thread 0 fences (release before the arrival count, acquire after
// it); readers of the partials use __ldcg.  Returns true in every thread of the last block.
__device__ __forceinline__ bool last_block_of_group(unsigned *counter, unsigned nblocks,
                                                    bool *sh_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(counter, 1u);
        const bool last = (prev == nblocks - 1);
        if (last) {
            *counter = 0u;
            __threadfence();
        }
        *sh_flag = last;
    }
    __syncthreads();
    return *sh_flag;
}

// floor for 0 <= x < 2^22 without a conversion instruction: the round-down add
// puts floor(x) in the mantissa of 2^23 + floor(x).
__device__ __forceinline__ float floor_pos(float x, int &i) {
    float m = __fadd_rd(x, 8388608.0f);
    i = __float_as_int(m) - 0x4B000000;
    return m - 8388608.0f;
}

// 4 consecutive elements through 16-byte accesses (p must be 4-element aligned)
template <typename T>
struct Q4 {
    T v[4];
};
__device__ __forceinline__ Q4<float> ld4(const float *__restrict__ p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    return Q4<float>{{a.x, a.y, a.z, a.w}};
}
__device__ __forceinline__ Q4<double> ld4(const double *__restrict__ p) {
    const double2 a = reinterpret_cast<const double2 *>(p)[0], b = reinterpret_cast<const double2 *>(p)[1];
    return Q4<double>{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ void st4(float *__restrict__ p, const Q4<float> &q) {
    *reinterpret_cast<float4 *>(p) = make_float4(q.v[0], q.v[1], q.v[2], q.v[3]);
}
__device__ __forceinline__ void st4(double *__restrict__ p, const Q4<double> &q) {
    reinterpret_cast<double2 *>(p)[0] = make_double2(q.v[0], q.v[1]);
    reinterpret_cast<double2 *>(p)[1] = make_double2(q.v[2], q.v[3]);
}

template <typename T>
struct Vec;  // storage helpers
template <>
struct Vec<float> {
    static constexpr int id = 0;
};
template <>
struct Vec<double> {
    static constexpr int id = 1;
};

constexpr int TQ_MAX_DEGREE = 64;  // graph rule: neighbours per node (tq_create validates)

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Programmatic dependent launch (sm_90+): the hot-loop kernels are launched with the
// programmatic-serialization attribute so a kernel's launch overlaps the end of the one
// before it on the stream; each such kernel calls pdl_wait() before it touches memory the
// previous kernel wrote (griddepcontrol.wait returns once that grid has completed and its
// writes are visible; a no-op for a normal launch).  TQ_PDL=0 launches them normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KP, typename... A>
inline void launch_pdl(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TQ_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...));
}

}  // namespace tq
