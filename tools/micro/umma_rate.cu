// Microbenchmark: tcgen05.mma (kind::f16, M=128, N=n, K=16, SW128 K-major smem
// operands) issue rate from one thread, with and without a commit per k-block.
#include <cstdio>
#include <cuda.h>
#include "../../paper_2504_10724_b200/csrc/ptx.cuh"
using namespace eeb::ptx;

__global__ void k(int n, int iters, int commit_every, int nacc, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint64_t bar2[4];
    __shared__ uint32_t slot;
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); for (int c = 0; c < 4; ++c) mbar_init(smem_u32(&bar2[c]), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, n);
        const uint64_t da = smem_desc_sw128(base), db = smem_desc_sw128(base + 16384);
        unsigned long long t0 = clock64();
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem + (uint32_t)((kk % nacc) * n), da + 2 * kk, db + 2 * kk, idesc, 1);
            if (commit_every > 0 && (i % commit_every) == commit_every - 1) {
                umma_commit(smem_u32(&bar));
                mbar_wait(smem_u32(&bar), ph); ph ^= 1;
            }
            if (commit_every < 0)  // commits without waiting (two per k-block, like the step kernel)
                for (int c = 0; c < -commit_every; ++c) umma_commit(smem_u32(&bar2[c]));
        }
        umma_commit(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), ph);
        out[0] = clock64() - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 1000;
    for (int n : {16, 64, 128, 256})
        for (int ce : {0, 1, 4, -1, -2})
            for (int na : {1, 4}) {
                if (na * n > 512) continue;
                k<<<1, 128, 64 * 1024>>>(n, iters, ce, na, d);
                unsigned long long c = 0;
                cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
                printf("N=%3d commit_every=%d nacc=%d: %.1f clk per MMA (%.1f per k-block of 4)  err=%s\n", n, ce, na,
                       (double)c / (iters * 4), (double)c / iters, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
