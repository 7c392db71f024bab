// Strip-phase synchronisation on a 16-CTA cluster (384 threads/CTA): each
// phase a CTA sends one halo row of NV doubles to each neighbour, then
//   A: generic remote stores + barrier.cluster (the bottom kernel's scheme);
//   B: st.async with complete_tx on the neighbour's mbarrier (one per phase
//      parity), own arrive.expect_tx, try_wait on own mbarrier, __syncthreads.
// cycles per phase (CTA 0, thread 0), plus a check that B delivered the data.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smaddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__global__ void k_phase(int iters, int mode, int nv, long long* out, int* bad) {
  __shared__ double halo[2][2][64];  // [parity][from below / above][value]
  __shared__ alignas(8) unsigned long long bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), cs = cl.num_blocks();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smaddr(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 256; i += blockDim.x) (&halo[0][0][0])[i] = 0.0;
  cl.sync();
  const bool has_up = r > 0, has_dn = r + 1 < cs;
  const int nexp = (has_up ? 1 : 0) + (has_dn ? 1 : 0);
  int errs = 0;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    const int par = k & 1;
    const double val = (double)(k * 100 + (int)r);
    if (mode == 0) {
      if (tid < nv) {
        if (has_up) cl.map_shared_rank(&halo[par][0][0], r - 1)[tid] = val;  // I am below it
        if (has_dn) cl.map_shared_rank(&halo[par][1][0], r + 1)[tid] = val;
      }
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smaddr(&bar[par])),
                     "r"(nexp * nv * 8) : "memory");
      if (tid < nv) {
        if (has_up) {
          const unsigned ra = mapa(smaddr(&halo[par][0][tid]), r - 1), rb = mapa(smaddr(&bar[par]), r - 1);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(val),
                       "r"(rb) : "memory");
        }
        if (has_dn) {
          const unsigned ra = mapa(smaddr(&halo[par][1][tid]), r + 1), rb = mapa(smaddr(&bar[par]), r + 1);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(val),
                       "r"(rb) : "memory");
        }
      }
      const unsigned ph = (k >> 1) & 1;
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "W%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n}" ::"r"(
              smaddr(&bar[par])),
          "r"(ph)
          : "memory");
      __syncthreads();
    }
    // both variants: the halo of this phase must hold the neighbours' values
    if (tid < nv) {
      if (has_dn && halo[par][0][tid] != (double)(k * 100 + (int)r + 1)) ++errs;
      if (has_up && halo[par][1][tid] != (double)(k * 100 + (int)r - 1)) ++errs;
    }
    if (mode == 0) __syncthreads();  // the next phase's stores may not overtake these checks (A has no 3rd buffer)
  }
  long long t1 = clock64();
  if (errs) atomicAdd(bad, errs);
  if (tid == 0 && r == 0) out[0] = t1 - t0;
  cl.sync();
}

int main() {
  long long* d;
  int* bad;
  cudaMalloc(&d, 8);
  cudaMalloc(&bad, 4);
  cudaFuncSetAttribute(k_phase, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int nv : {33, 64}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(bad, 0, 4);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(384);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_phase, 2000, mode, nv, d, bad);
      e = cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      int b; cudaMemcpy(&b, bad, 4, cudaMemcpyDeviceToHost);
      printf("nv %2d %s: %6.0f cycles/phase, %d wrong halo values (%s)\n", nv,
             mode ? "st.async + mbarrier     " : "remote st + cluster bar", c / 2000.0, b, cudaGetErrorString(e));
    }
  }
  return 0;
}
