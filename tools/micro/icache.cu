// icache.cu — cost of executing straight-line code the SM has not run
// recently (instruction-cache fill) vs the same code hot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu && ./icache
// Kernel `line` runs N straight-line independent ops per thread; `other` is a
// different large kernel run in between to evict `line` from the SM's
// instruction caches.  Thread 0 of each CTA records clock64 around the code.
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void line(long long* out, int seed) {
    int a = threadIdx.x + seed, b = seed * 3, c = seed ^ 7, d = seed + 11;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < N; ++i) {
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a) : "r"(seed), "r"(i));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(b) : "r"(seed), "r"(i));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(c) : "r"(seed), "r"(i));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(d) : "r"(seed), "r"(i));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (a + b + c + d == 0x12345) out[blockIdx.x] = 0;
}

int main() {
    long long *d, h[148];
    cudaMalloc(&d, sizeof h);
    auto run = [&](auto kern, const char* what) {
        kern<<<148, 128>>>(d, 1);
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0, mn = 1LL << 62;
        for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
        printf("%-28s cycles min %lld max %lld\n", what, mn, mx);
    };
    for (int rep = 0; rep < 3; ++rep) {
        run(line<1024>, "A (4096 ops) after B");
        run(line<1024>, "A again (hot)");
        run(line<2048>, "B (8192 ops) evicts A");
    }
    return 0;
}
