// common.cuh — shared device/host helpers for the eeb kernels (sm_100a).
#pragma once

#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

namespace eeb {

// ---------------------------------------------------------------------------
// Status plumbing.  Host code throws eeb::Error; the C ABI catches and maps it
// to the eeb_status code (errors.hpp:9-30 ↔ EEB_E_*).
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define EEB_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw ::eeb::Error(5, std::string(#call) + ": " + cudaGetErrorString(_e) +  \
                                      " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define EEB_CHECK_LAUNCH() EEB_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// Element types.  Weights, GEMM activations and KV share the model dtype
// (f32 for the parity configuration, bf16 for speed); the residual stream and
// every accumulator are f32.
// ---------------------------------------------------------------------------
template <typename T> struct TypeTag;
template <> struct TypeTag<float> { static constexpr int kDtype = 0; };
template <> struct TypeTag<__nv_bfloat16> { static constexpr int kDtype = 1; };

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

// 16-byte vector of T: 8 bf16 or 4 f32.
template <typename T> struct Vec16 { static constexpr int N = 16 / sizeof(T); };

__device__ __forceinline__ void unpack16(const uint4& u, float* f, const float*) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack16(const uint4& u, float* f, const __nv_bfloat16*) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        f[2 * j] = __uint_as_float(w[j] << 16);
        f[2 * j + 1] = __uint_as_float(w[j] & 0xffff0000u);
    }
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Programmatic dependent launch (PDL).  Every kernel of the step lets its
// successor launch at once (launch_dependents) and waits for its predecessor
// (wait) before touching data the predecessor produced; work on constant
// data (weights, older KV) can run before the wait.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch of this CTA's share of [p, p + bytes): the weights of the GEMM
// that follows a latency-bound kernel (norm, attention), pulled into L2 while
// that kernel runs so the GEMM streams them from L2.  One warp (the caller's
// lanes) issues 16 KB bulk prefetches; no completion to wait for.
__device__ __forceinline__ void l2_prefetch_share(const void* p, size_t bytes, int lane) {
    if (!p || !bytes) return;
    const size_t nct = (size_t)gridDim.x * gridDim.y;
    const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
    const size_t share = ((bytes + nct - 1) / nct + 255) & ~(size_t)255;
    const size_t b0 = cta * share, b1 = b0 + share < bytes ? b0 + share : bytes;
    constexpr size_t kPiece = 16384;
    for (size_t o = b0 + (size_t)lane * kPiece; o < b1; o += 32 * kPiece) {
        const uint32_t n = (uint32_t)((b1 - o < kPiece ? b1 - o : kPiece) & ~(size_t)15);
        if (n)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(p) + o), "r"(n)
                         : "memory");
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// In-graph launch timeline (eeb_debug_stamps).  Every step kernel takes a Stamp
// as its first argument and opens a StampScope: with stamping on, thread 0 of
// each CTA records the CTA's start and lane 0 of every warp its exit
// (%globaltimer, fire-and-forget red.min / red.max into [slot][cta] cells, no
// contention), so the host gets each launch's first-start / last-exit inside
// the captured, PDL-chained graph — the execution that is timed.  Off (buf
// null): one predicated branch per CTA.
// ---------------------------------------------------------------------------
struct Stamp {
    unsigned long long* buf = nullptr;  // starts [slots][kStampCtas], ends at + end_off, waits at + 2 end_off
    int slot = 0;
    int64_t end_off = 0;
};
constexpr int kStampCtas = 2048;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    return t;
}
__device__ __forceinline__ unsigned long long* stamp_cell(const Stamp& s) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    return s.buf + (size_t)s.slot * kStampCtas + min(cta, (unsigned)kStampCtas - 1);
}
struct StampScope {
    const Stamp& s;
    __device__ __forceinline__ explicit StampScope(const Stamp& st) : s(st) {
        if (s.buf && threadIdx.x == 0)
            asm volatile("red.global.min.u64 [%0], %1;" ::"l"(stamp_cell(s)), "l"(gtimer()) : "memory");
    }
    __device__ __forceinline__ ~StampScope() {
        if (s.buf && (threadIdx.x & 31) == 0)
            asm volatile("red.global.max.u64 [%0], %1;" ::"l"(stamp_cell(s) + s.end_off), "l"(gtimer()) : "memory");
    }
};
// After the kernel's griddepcontrol.wait returned (first CTA): the predecessor
// finished; wait - previous end = launch/flush latency, end - wait = work.
__device__ __forceinline__ void stamp_waited(const Stamp& s) {
    if (s.buf && threadIdx.x == 0)
        asm volatile("red.global.min.u64 [%0], %1;" ::"l"(stamp_cell(s) + 2 * s.end_off), "l"(gtimer()) : "memory");
}
// A kernel-specific midpoint (GEMM: accumulator complete), the latest over
// CTAs: wait -> mark is the main loop, mark -> end the epilogue tail.
__device__ __forceinline__ void stamp_mark(const Stamp& s) {
    if (s.buf)
        asm volatile("red.global.max.u64 [%0], %1;" ::"l"(stamp_cell(s) + 3 * s.end_off), "l"(gtimer()) : "memory");
}
// Host: the stamp for the next launch (defined in eeb_api.cu; buf null unless
// the calling thread is recording a timeline).
Stamp stamp_next(const void* kernel);

// Host: launch with the programmatic-stream-serialization attribute so the
// kernel may start while its predecessor drains (captured into graphs as a
// programmatic edge).  The kernel's first parameter is its Stamp.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(Stamp, KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("EEB_NO_PDL") != nullptr;  // debugging: plain stream order
    static const char* no_pdl_k = std::getenv("EEB_NO_PDL_K");          // ... for kernels named like these
    bool off = no_pdl;
    if (!off && no_pdl_k) {
        const char* name = nullptr;
        if (cudaFuncGetName(&name, reinterpret_cast<const void*>(kern)) == cudaSuccess && name) {
            std::string list(no_pdl_k), nm(name);
            size_t a = 0;
            while (a <= list.size()) {
                size_t b = list.find(',', a);
                if (b == std::string::npos) b = list.size();
                if (b > a && nm.find(list.substr(a, b - a)) != std::string::npos) off = true;
                a = b + 1;
            }
        }
    }
    cfg.numAttrs = off ? 0 : 1;
    EEB_CUDA(cudaLaunchKernelEx(&cfg, kern, stamp_next(reinterpret_cast<const void*>(kern)),
                                std::forward<Args>(args)...));
}

}  // namespace eeb
