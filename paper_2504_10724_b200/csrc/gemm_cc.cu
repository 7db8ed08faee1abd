// gemm_cc.cu — tier-1 decode GEMM on CUDA cores: y[B, N] = x[B, K] · W[N, K]^T.
//
// Weight-streaming: every weight element is read exactly once per launch with
// 16-byte non-allocating loads; the activation slice [B, KS] is staged in
// shared memory and reused across the CTA's output rows.  Split-K fills the
// 148 SMs when N is small; partials are summed in a fixed order by the
// epilogue kernel (deterministic — no atomics feed the logits, SURVEY §7
// hard part 2).  This tier serves small batches and the f32 parity model; the
// tcgen05 tier (gemm_tc.cu) takes over for bf16 once B >= 16.
#include "kernels.h"

namespace eeb {

namespace {

constexpr int kWarps = 8;
constexpr int kRowsPerWarp = 2;
constexpr int kRowsPerCta = kWarps * kRowsPerWarp;

template <typename T, int MAXB>
__global__ void __launch_bounds__(kWarps * 32)
    gemm_cc_kernel(Stamp stamp, const T* __restrict__ W, const T* X, const int* n_active,
                   float* part, int N, int K, int KS, int64_t split_stride) {
    StampScope stamp_scope(stamp);
    constexpr int VEC = Vec16<T>::N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* xs = reinterpret_cast<T*>(smem_raw);  // [MAXB][KS]

    pdl_launch_dependents();
    const int k0 = blockIdx.y * KS;
    const int kn = min(KS, K - k0);
    // The weights do not depend on the predecessor: pull this CTA's slice
    // (one K-span per weight row) into L2 while the predecessor drains, so
    // the stream after the wait runs out of L2 — at 1-2 rows the GEMV's
    // weight stream is otherwise fully exposed after every kernel boundary.
    // Skipped when no row is live (every row exited early): the count is read
    // before the wait, so it may be stale — that costs only a useless or a
    // missed prefetch; the count after the wait decides what is computed.
    static constexpr bool kL2Prefetch = false;  // measured: B=1 C2 0.78 -> 0.85 ms/step with it
    if (kL2Prefetch && threadIdx.x < kRowsPerCta && *reinterpret_cast<const volatile int*>(n_active) > 0) {
        const int n = blockIdx.x * kRowsPerCta + threadIdx.x;
        if (n < N) {
            const char* src = reinterpret_cast<const char*>(W + (int64_t)n * K + k0);
            const uint32_t bytes = (uint32_t)(kn * (int)sizeof(T)) & ~15u;
            for (uint32_t o = 0; o < bytes; o += 16384u) {
                const uint32_t len = min(16384u, bytes - o);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + o), "r"(len) : "memory");
            }
        }
    }
    pdl_wait();
    const int nb = min(*n_active, MAXB);
    if (nb <= 0) return;

    // Stage the activation slice.
    const int vec_per_row = kn / VEC;
    for (int idx = threadIdx.x; idx < nb * vec_per_row; idx += blockDim.x) {
        const int b = idx / vec_per_row, v = idx % vec_per_row;
        reinterpret_cast<uint4*>(xs + b * KS)[v] =
            *reinterpret_cast<const uint4*>(X + (int64_t)b * K + k0 + v * VEC);
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * kRowsPerCta + warp * kRowsPerWarp;
    float acc[kRowsPerWarp][MAXB];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
        for (int b = 0; b < MAXB; ++b) acc[r][b] = 0.f;

    const T* wrow[kRowsPerWarp];
    bool rvalid[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
        rvalid[r] = (n0 + r) < N;
        wrow[r] = W + (int64_t)(rvalid[r] ? n0 + r : 0) * K + k0;
    }

    for (int kk = lane * VEC; kk < kn; kk += 32 * VEC) {
        float w[kRowsPerWarp][VEC];
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r) {
            const uint4 u = ldg_stream(wrow[r] + kk);
            unpack16(u, w[r], (const T*)nullptr);
        }
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
            if (b < nb) {
                float xv[VEC];
                unpack16(*reinterpret_cast<const uint4*>(xs + b * KS + kk), xv, (const T*)nullptr);
#pragma unroll
                for (int r = 0; r < kRowsPerWarp; ++r) {
                    float a = acc[r][b];
#pragma unroll
                    for (int j = 0; j < VEC; ++j) a = fmaf(w[r][j], xv[j], a);
                    acc[r][b] = a;
                }
            }
        }
    }

    float* out = part + blockIdx.y * split_stride;
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
            if (b < nb) {
                const float v = warp_sum(acc[r][b]);
                if (lane == 0 && rvalid[r]) out[(int64_t)b * N + n0 + r] = v;
            }
        }
    }
}

template <typename T, int MAXB>
int run_cc(const GemmArgs& a, cudaStream_t s) {
    constexpr int VEC = Vec16<T>::N;
    const int tiles = (a.N + kRowsPerCta - 1) / kRowsPerCta;
    // Split K until the grid covers ~2 waves, keeping KS a multiple of 32*VEC
    // and the staged slice within 96 KB of shared memory.
    int splits = 1;
    const int kmin = 32 * VEC;
    auto ks_of = [&](int sp) {
        int ks = (a.K + sp - 1) / sp;
        return (ks + kmin - 1) / kmin * kmin;
    };
    while (true) {
        const int ks = ks_of(splits);
        const bool smem_ok = (int64_t)ks * MAXB * (int)sizeof(T) <= 96 * 1024;
        const bool occ_ok = (int64_t)tiles * splits >= 2LL * a.num_sms;
        if (smem_ok && (occ_ok || ks <= kmin)) break;
        if (ks <= kmin) break;
        ++splits;
    }
    const int KS = ks_of(splits);
    splits = (a.K + KS - 1) / KS;
    const int64_t split_stride = a.plane_stride;
    if (splits > a.max_planes) throw Error(2, "gemm_cc: split-K workspace too small");
    const size_t smem = (size_t)KS * MAXB * sizeof(T);
    auto kern = gemm_cc_kernel<T, MAXB>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(tiles, splits);
    launch_pdl(kern, grid, dim3(kWarps * 32), smem, s, static_cast<const T*>(a.W), static_cast<const T*>(a.X),
               a.n_active, a.out, a.N, a.K, KS, split_stride);
    EEB_CHECK_LAUNCH();
    return splits;
}

template <typename T>
int dispatch_cc(const GemmArgs& a, cudaStream_t s) {
    if (a.K % (32 * Vec16<T>::N) != 0) throw Error(1, "gemm_cc: K must be a multiple of 32 vectors");
    const int b = a.max_rows;
    if (b <= 1) return run_cc<T, 1>(a, s);
    if (b <= 2) return run_cc<T, 2>(a, s);
    if (b <= 4) return run_cc<T, 4>(a, s);
    if (b <= 8) return run_cc<T, 8>(a, s);
    if (b <= 16) return run_cc<T, 16>(a, s);
    if (b <= 32) return run_cc<T, 32>(a, s);
    if (b <= 64) return run_cc<T, 64>(a, s);
    throw Error(1, "gemm_cc: batch > 64 needs the tensor-core tier");
}

}  // namespace

int gemm_cc(const GemmArgs& a, cudaStream_t s) {
    return a.dtype == 0 ? dispatch_cc<float>(a, s) : dispatch_cc<__nv_bfloat16>(a, s);
}

}  // namespace eeb
