// Latency / throughput of warp-level mma.sync m16n8k16 bf16 (legacy HMMA path)
// and of MUFU.EX2 / SHFL on this GPU: one warp, dependent chains vs independent.
#include <cstdio>
#include <cuda_bf16.h>
__device__ __forceinline__ void mma(float* c, const unsigned* a, unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k_mma(long long* out, float* sink, int iters) {
    unsigned a[4] = {0x3f803f80u ^ threadIdx.x, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u};
    float c[CH][4] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) mma(c[j], a, 0x3f803f80u, 0x3f803f80u);
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += c[j][0];
    sink[threadIdx.x] = s;
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
__global__ void k_shfl(long long* out, float* sink, int iters) {
    float v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.f;
    long long t1 = clock64();
    sink[threadIdx.x] = v;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_ex2(long long* out, float* sink, int iters) {
    float v = threadIdx.x * 1e-3f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) v = __expf(v) * 0.5f;
    long long t1 = clock64();
    sink[threadIdx.x] = v;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    long long* d; float* s; long long h[8];
    cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 4096 * 4);
    const int it = 4096;
    k_mma<1><<<1, 32>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("HMMA dependent chain: %.1f cycles/mma\n", (double)h[0] / it);
    k_mma<4><<<1, 32>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("HMMA 4 chains, 1 warp: %.1f cycles/mma\n", (double)h[0] / it / 4);
    k_mma<8><<<1, 32>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("HMMA 8 chains, 1 warp: %.1f cycles/mma\n", (double)h[0] / it / 8);
    k_mma<8><<<1, 128>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("HMMA 8 chains, 4 warps (1/SMSP): %.1f cycles/mma per warp\n", (double)h[0] / it / 8);
    k_mma<8><<<1, 256>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("HMMA 8 chains, 8 warps (2/SMSP): %.1f cycles/mma per warp\n", (double)h[0] / it / 8);
    k_shfl<<<1, 32>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("SHFL+FADD dependent: %.1f cycles\n", (double)h[0] / it);
    k_ex2<<<1, 32>>>(d, s, it); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("EX2+FMUL dependent: %.1f cycles\n", (double)h[0] / it);
    return 0;
}
