#include <cuda_runtime.h>
#include <cstdio>
__global__ void setk(cudaGraphConditionalHandle h, const int* v) { if (threadIdx.x == 0) cudaGraphSetConditional(h, *v > 0 ? 1u : 0u); }
__global__ void body(int* x) { atomicAdd(x, 1); }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  int *d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  int one = 0; cudaMemcpy(d, &one, 4, cudaMemcpyHostToDevice);
  cudaGraph_t g; cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
  cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
  cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault);
  setk<<<1,32,0,s>>>(h, d);
  cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
  cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeIf; p.conditional.size = 1;
  cudaGraphNode_t node; cudaError_t e = cudaGraphAddNode(&node, cg, deps, nd, &p);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
  cudaStream_t s2; cudaStreamCreate(&s2);
  e = cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  printf("cap2 %s\n", cudaGetErrorString(e));
  body<<<1,1,0,s2>>>(d + 1);
  cudaStreamEndCapture(s2, nullptr);
  body<<<1,1,0,s>>>(d + 1);  // after the conditional: always
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int r[2]; cudaMemcpy(r, d, 8, cudaMemcpyDeviceToHost); printf("cond=0: count %d (want 1)\n", r[1]);
  one = 1; cudaMemcpy(d, &one, 4, cudaMemcpyHostToDevice);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  cudaMemcpy(r, d, 8, cudaMemcpyDeviceToHost); printf("cond=1: count %d (want 3)\n", r[1]);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
