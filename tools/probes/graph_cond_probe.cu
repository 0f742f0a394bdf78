// Probe: can kernel nodes inside a conditional WHILE body be updated with
// cudaGraphExecKernelNodeSetParams after instantiation?  (CUDA 12.9)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_add(int* ctr, int v) { atomicAdd(ctr, v); }
__global__ void k_cond(cudaGraphConditionalHandle h, int* it, int n) {
  int i = ++(*it);
  cudaGraphSetConditional(h, i < n ? 1u : 0u);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s -> %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int *ctr, *it;
  CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&it, 4));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  // body: k_add(ctr, 1) -> k_cond
  cudaKernelNodeParams kp = {};
  int one = 1;
  void* a1[] = {&ctr, &one};
  kp.func = (void*)k_add; kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = a1;
  cudaGraphNode_t kadd, kc;
  CK(cudaGraphAddKernelNode(&kadd, body, nullptr, 0, &kp));
  int n = 5;
  void* a2[] = {&h, &it, &n};
  cudaKernelNodeParams kq = {};
  kq.func = (void*)k_cond; kq.gridDim = dim3(1); kq.blockDim = dim3(1); kq.kernelParams = a2;
  CK(cudaGraphAddKernelNode(&kc, body, &kadd, 1, &kq));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  CK(cudaMemsetAsync(ctr, 0, 4, st)); CK(cudaMemsetAsync(it, 0, 4, st));
  CK(cudaGraphLaunch(ex, st));
  int hc = 0; CK(cudaMemcpyAsync(&hc, ctr, 4, cudaMemcpyDeviceToHost, st)); CK(cudaStreamSynchronize(st));
  printf("first launch: ctr = %d (expect 5)\n", hc);
  int seven = 7;
  void* a3[] = {&ctr, &seven};
  kp.kernelParams = a3;
  cudaError_t e = cudaGraphExecKernelNodeSetParams(ex, kadd, &kp);
  printf("SetParams on body node: %s\n", cudaGetErrorString(e));
  CK(cudaMemsetAsync(ctr, 0, 4, st)); CK(cudaMemsetAsync(it, 0, 4, st));
  CK(cudaGraphLaunch(ex, st));
  CK(cudaMemcpyAsync(&hc, ctr, 4, cudaMemcpyDeviceToHost, st)); CK(cudaStreamSynchronize(st));
  printf("second launch: ctr = %d (expect 35 if updated)\n", hc);
  // timing: launch overhead of a 1000-iteration while loop with 2 tiny kernels
  n = 1000;
  void* a4[] = {&h, &it, &n};
  kq.kernelParams = a4;
  e = cudaGraphExecKernelNodeSetParams(ex, kc, &kq);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaMemsetAsync(it, 0, 4, st));
  cudaEventRecord(e0, st);
  CK(cudaGraphLaunch(ex, st));
  cudaEventRecord(e1, st);
  CK(cudaStreamSynchronize(st));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("1000 loop iterations (2 kernels each): %.3f ms -> %.2f us/iteration\n", ms, ms);
  return 0;
}
