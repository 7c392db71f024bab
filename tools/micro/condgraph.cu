// Per-iteration cost of the stand-alone loop's graph structure with empty
// kernels: WHILE { child(A) ; check ; IF { child(B) } } vs a plain WHILE { A ; check ; B }.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_check(cudaGraphConditionalHandle a, cudaGraphConditionalHandle b, int* it, int n) {
  const int i = ++*it;
  const unsigned go = i < n;
  cudaGraphSetConditional(a, go);
  if (b) cudaGraphSetConditional(b, go);
}
__global__ void k_check1(cudaGraphConditionalHandle a, int* it, int n) {
  const int i = ++*it;
  cudaGraphSetConditional(a, i < n);
}

static cudaGraph_t chain(int k) {  // k dependent empty kernels
  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaGraphNode_t prev = nullptr, nd;
  for (int i = 0; i < k; ++i) {
    cudaKernelNodeParams kp{};
    kp.func = (void*)k_empty; kp.gridDim = dim3(1); kp.blockDim = dim3(32); kp.kernelParams = nullptr;
    cudaGraphAddKernelNode(&nd, g, prev ? &prev : nullptr, prev ? 1 : 0, &kp);
    prev = nd;
  }
  return g;
}

int main() {
  int* d_it;
  cudaMalloc(&d_it, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const int N = 1000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int kb : {1, 12}) {
      cudaGraph_t cg;
      cudaGraphCreate(&cg, 0);
      cudaGraphConditionalHandle hw, hi = 0;
      cudaGraphConditionalHandleCreate(&hw, cg, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams wp{};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = hw; wp.conditional.type = cudaGraphCondTypeWhile; wp.conditional.size = 1;
      cudaGraphNode_t wn;
      cudaGraphAddNode(&wn, cg, nullptr, 0, &wp);
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      cudaGraphNode_t a, c, b;
      cudaGraphAddChildGraphNode(&a, body, nullptr, 0, chain(1));
      if (mode == 2) cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault);
      void* args[] = {&hw, &hi, &d_it, (void*)&N};
      int n = N;
      args[3] = &n;
      cudaKernelNodeParams kp{};
      kp.func = (void*)k_check; kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = args;
      cudaGraphAddKernelNode(&c, body, &a, 1, &kp);
      if (mode == 1) {
        cudaGraphAddChildGraphNode(&b, body, &c, 1, chain(kb));
      } else if (mode == 2) {
        cudaGraphNodeParams ip{};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hi; ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
        cudaGraphNode_t in;
        cudaGraphAddNode(&in, body, &c, 1, &ip);
        cudaGraphAddChildGraphNode(&b, ip.conditional.phGraph_out[0], nullptr, 0, chain(kb));
      }
      cudaGraphExec_t ex;
      cudaError_t e = cudaGraphInstantiate(&ex, cg, 0);
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemsetAsync(d_it, 0, 4, s);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const char* nm[3] = {"WHILE{A;check}", "WHILE{A;check;B(child)}", "WHILE{A;check;IF{B}}"};
      printf("%-26s B=%2d kernels: %.2f us/iter (%s)\n", nm[mode], kb, best * 1e3 / N, cudaGetErrorString(e));
      if (mode == 0) break;
    }
  }
  // reference: plain graph of 14 kernels launched 1000 times
  cudaGraph_t g = chain(14);
  cudaGraphExec_t ex;
  cudaGraphInstantiate(&ex, g, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaGraphLaunch(ex, s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < N; ++i) cudaGraphLaunch(ex, s);
  cudaEventRecord(e1, s);
  cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("plain graph of 14 empty kernels: %.2f us/launch\n", ms * 1e3 / N);
  return 0;
}
