// Micro-benchmark of the per-row kernels between the GEMMs (C2 shape: 64 rows,
// d 2048, 16 split-K planes): back-to-back launches timed with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/micro/rows_bench.cu -o tools/micro/rows_bench
#include "../../paper_2504_10724_b200/csrc/rows.cu"

#include <cstdio>

namespace eeb {
namespace {
__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 1234567) *p = 1;
}
__global__ void empty_pdl_kernel(int* p) {
    pdl_launch_dependents();
    pdl_wait();
    if (p && threadIdx.x == 1234567) *p = 1;
}
// one CTA per row, no cluster: the planes of a row summed by 512 threads
template <int kV>
__global__ void __launch_bounds__(512) norm_row_kernel(const float* part, int splits, int64_t split_stride,
                                                       const int* n_active, float* x, int d, float eps,
                                                       const float* g1, __nv_bfloat16* out1) {
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= *n_active) return;
    __shared__ float red[32];
    float* row = x + (int64_t)i * d;
    float4 v[kV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < d) {
            float4 xv = *reinterpret_cast<const float4*>(row + c);
            const float* src = part + (int64_t)i * d + c;
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s0 = 0; s0 < splits; s0 += 8) {
                float4 t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (s0 + j < splits) t[j] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + j) * split_stride));
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (s0 + j < splits) add4(y, t[j]);
            }
            add4(xv, y);
            *reinterpret_cast<float4*>(row + c) = xv;
            v[k] = xv;
            ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        }
    }
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)d + eps);
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) {
            const float4 gg = *reinterpret_cast<const float4*>(g1 + c);
            store4<__nv_bfloat16>(out1 + (int64_t)i * d + c,
                                  make_float4(v[k].x * inv * gg.x, v[k].y * inv * gg.y, v[k].z * inv * gg.z, v[k].w * inv * gg.w));
        }
    }
}
}  // namespace
}  // namespace eeb

using namespace eeb;

template <typename F>
static float time_it(F f, int reps, cudaStream_t s) {
    for (int i = 0; i < 10; ++i) f();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps;
}

int main() {
    const int B = 64, D = 2048, S = 16;
    float *part, *x, *g;
    __nv_bfloat16* out;
    int* na;
    int* src;
    cudaMalloc(&src, 256 * 4);
    cudaMemset(src, 0, 256 * 4);
    cudaMalloc(&part, (size_t)S * B * D * 4);
    cudaMalloc(&x, (size_t)B * D * 4);
    cudaMalloc(&g, D * 4);
    cudaMalloc(&out, (size_t)B * D * 2);
    cudaMalloc(&na, 4);
    cudaMemset(part, 0, (size_t)S * B * D * 4);
    cudaMemset(x, 0, (size_t)B * D * 4);
    cudaMemset(g, 0, D * 4);
    cudaMemcpy(na, &B, 4, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int R = 200;
    printf("empty 1 CTA          %.2f us\n", time_it([&] { empty_kernel<<<1, 32, 0, s>>>(nullptr); }, R, s));
    printf("empty 1 CTA pdl      %.2f us\n", time_it([&] { launch_pdl(empty_pdl_kernel, dim3(1), dim3(32), 0, s, (int*)nullptr); }, R, s));
    printf("empty 512 CTA pdl    %.2f us\n", time_it([&] { launch_pdl(empty_pdl_kernel, dim3(512), dim3(64), 0, s, (int*)nullptr); }, R, s));
    for (int sp : {1, 6, 16}) {
        printf("norm cluster  S=%2d   %.2f us\n", sp, time_it([&] {
            launch_residual_norm(1, part, sp, (int64_t)B * D, na, B, x, D, 1e-5f, g, out, nullptr, nullptr, s);
        }, R, s));
        printf("norm row512   S=%2d   %.2f us\n", sp, time_it([&] {
            launch_pdl(norm_row_kernel<1>, dim3(B), dim3(512), 0, s, (const float*)part, sp, (int64_t)B * D,
                       (const int*)na, x, D, 1e-5f, (const float*)g, out);
        }, R, s));
        printf("norm row256   S=%2d   %.2f us\n", sp, time_it([&] {
            launch_pdl(norm_row_kernel<2>, dim3(B), dim3(256), 0, s, (const float*)part, sp, (int64_t)B * D,
                       (const int*)na, x, D, 1e-5f, (const float*)g, out);
        }, R, s));
    }
    printf("gather 64 rows       %.2f us\n", time_it([&] {
        launch_gather_rows(x, part, out, out + B * D / 2, D * 2, src, na, B, D, s);
    }, R, s));
    // the same launches captured into one graph (as the step is)
    auto graph_of = [&](auto body, int n) {
        cudaGraph_t gr;
        cudaGraphExec_t ex;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < n; ++i) body();
        cudaStreamEndCapture(s, &gr);
        cudaGraphInstantiate(&ex, gr, 0);
        return ex;
    };
    const int N = 182;
    cudaGraphExec_t ge = graph_of([&] { launch_pdl(empty_pdl_kernel, dim3(1), dim3(32), 0, s, (int*)nullptr); }, N);
    printf("graph %d empty pdl    %.2f us per kernel\n", N, time_it([&] { cudaGraphLaunch(ge, s); }, 20, s) / N);
    cudaGraphExec_t ge2 = graph_of([&] { empty_kernel<<<1, 32, 0, s>>>(nullptr); }, N);
    printf("graph %d empty plain  %.2f us per kernel\n", N, time_it([&] { cudaGraphLaunch(ge2, s); }, 20, s) / N);
    cudaGraphExec_t ge3 = graph_of([&] { launch_pdl(empty_pdl_kernel, dim3(296), dim3(192), 0, s, (int*)nullptr); }, N);
    printf("graph %d 296x192 pdl  %.2f us per kernel\n", N, time_it([&] { cudaGraphLaunch(ge3, s); }, 20, s) / N);
    cudaGraphExec_t ge4 = graph_of([&] {
        launch_residual_norm(1, part, 16, (int64_t)B * D, na, B, x, D, 1e-5f, g, out, nullptr, nullptr, s); }, N);
    printf("graph %d norm cluster %.2f us per kernel\n", N, time_it([&] { cudaGraphLaunch(ge4, s); }, 20, s) / N);
    cudaGraphExec_t ge5 = graph_of([&] {
        launch_pdl(norm_row_kernel<1>, dim3(B), dim3(512), 0, s, (const float*)part, 16, (int64_t)B * D,
                   (const int*)na, x, D, 1e-5f, (const float*)g, out); }, N);
    printf("graph %d norm row512  %.2f us per kernel\n", N, time_it([&] { cudaGraphLaunch(ge5, s); }, 20, s) / N);
    auto launch_cl = [&](int cl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(296);
        cfg.blockDim = dim3(192);
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = cl;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = cl ? 2 : 1;
        cudaLaunchKernelEx(&cfg, empty_pdl_kernel, (int*)nullptr);
    };
    for (int cl : {0, 1, 2, 4, 8}) {
        cudaGraphExec_t gc = graph_of([&] { launch_cl(cl); }, N);
        printf("graph %d 296x192 pdl cluster %d  %.2f us per kernel\n", N, cl, time_it([&] { cudaGraphLaunch(gc, s); }, 20, s) / N);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
