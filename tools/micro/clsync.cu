// cluster barrier latency on B200 for cluster sizes 1..16 (512 threads/CTA),
// with and without one remote (DSMEM) store per thread before each barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int remote, long long* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), cs = cl.num_blocks();
  double* peer = cl.map_shared_rank(sm, (r + 1) % cs);
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (remote) peer[threadIdx.x] = (double)i;
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && r == 0) out[0] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int remote = 0; remote < 2; ++remote) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 160 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, k_sync, &cfg);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_sync, 1000, remote, d);
      e = cudaDeviceSynchronize();
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      e = cudaLaunchKernelEx(&cfg, k_sync, 1000, remote, d);
      cudaEventRecord(e1);
      e = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("cluster %2d remote %d: %6.0f cycles/sync, kernel %.1f us, max active clusters %d (%s)\n", cs, remote,
             c / 1000.0, ms * 1e3, ncl, cudaGetErrorString(e));
    }
  }
  return 0;
}
