// Cost of cluster.sync() for a 16-CTA cluster (dev tool).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = iters;
}
__global__ void k_dsmem(int iters, double* out, int csz) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  const int r = int(cl.block_rank());
  if (threadIdx.x < 64) buf[threadIdx.x] = r;
  cl.sync();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    // each CTA reads one value from every peer (a 16-way broadcast/reduce), then syncs
    if (threadIdx.x < csz) acc += *cl.map_shared_rank(&buf[i % 64], threadIdx.x);
    cl.sync();
  }
  if (threadIdx.x == 0) out[r] = acc;
}
int main() {
  int* o; double* od;
  cudaMalloc(&o, 4); cudaMalloc(&od, 16 * 8);
  for (int csz : {2, 8, 16}) {
    for (int threads : {256, 1024}) {
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csz); cfg.blockDim = dim3(threads);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      const int iters = 20000;
      cudaLaunchKernelEx(&cfg, k, 100, o);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k, iters, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k_dsmem, iters, od, csz);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms2; cudaEventElapsedTime(&ms2, a, b);
      printf("cluster %2d x %4d threads: sync %.3f us, dsmem read + sync %.3f us  (%s)\n", csz, threads,
             ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // how many 16-CTA clusters (1024 threads, 1 CTA/SM) can be co-resident
  int ncl = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(1024);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k, &cfg);
  printf("max active 16-CTA clusters (1024 threads): %d\n", ncl);
  return 0;
}
