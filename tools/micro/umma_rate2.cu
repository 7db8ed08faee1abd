// tcgen05.mma issue rate: single-lane loop vs whole-warp loop (elect.sync per op).
#include <cstdio>
#include <cuda.h>
#include "../../paper_2504_10724_b200/csrc/ptx.cuh"
using namespace eeb::ptx;

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

template <int MODE, int N>
__global__ void k(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[3];
    __shared__ uint32_t slot;
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) mbar_init(smem_u32(&bar[i]), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x < 32) tmem_alloc(smem_u32(&slot), 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t idesc = idesc_bf16(128, N);
    const uint64_t da = smem_desc_sw128(base), db = smem_desc_sw128(base + 16384);
    unsigned long long t0 = clock64();
    if (MODE == 0) {  // one lane
        if (threadIdx.x == 0) {
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, 1);
                umma_commit(smem_u32(&bar[1]));
                umma_commit(smem_u32(&bar[2]));
            }
            umma_commit(smem_u32(&bar[0]));
            mbar_wait(smem_u32(&bar[0]), 0);
        }
    } else {  // whole warp, elect per op
        if (threadIdx.x < 32) {
            for (int i = 0; i < iters; ++i) {
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, 1);
                    umma_commit(smem_u32(&bar[1]));
                    umma_commit(smem_u32(&bar[2]));
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(smem_u32(&bar[0]));
            __syncwarp();
            mbar_wait(smem_u32(&bar[0]), 0);
        }
    }
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE, int N> void run(unsigned long long* d) {
    cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 2000;
    k<MODE, N><<<1, 128, 64 * 1024>>>(iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("mode=%d N=%3d: %.1f clk per k-block (4 MMA + 2 commits)  %s\n", MODE, N, (double)c / iters,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    run<0, 64>(d); run<1, 64>(d); run<0, 128>(d); run<1, 128>(d); run<0, 256>(d); run<1, 256>(d);
    run<0, 64>(d); run<1, 64>(d);
    return 0;
}
