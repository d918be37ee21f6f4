// Can the executor's cooperative grid (one 256-thread CTA per SM, ~150 KB shared memory) be
// launched as clusters of 2 (DSMEM between the chain CTA and a partner)? Prints the maximum
// number of co-resident 2-clusters and the result of a cooperative + cluster launch.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(256, 1) k(int* out) {
  extern __shared__ double sm[];
  cg::grid_group g = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  cl.sync();
  double* peer = cl.map_shared_rank(sm, cl.block_rank() ^ 1);
  if (threadIdx.x == 0) out[blockIdx.x] = (int)peer[0];
  g.sync();
}
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 150 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsm);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
  printf("SMs %d, max active 2-clusters %d (%s)\n", nsm, nclusters, cudaGetErrorString(e));
  int* out;
  cudaMalloc(&out, nsm * sizeof(int));
  for (int grid : {nsm, 2 * nclusters}) {
    cfg.gridDim = dim3(grid);
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, k, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("cooperative + cluster 2 launch, grid %d: %s / %s\n", grid, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaGetLastError();
  }
  int h[2];
  cudaMemcpy(h, out, 2 * sizeof(int), cudaMemcpyDeviceToHost);
  printf("peer of CTA 0 saw %d, of CTA 1 saw %d\n", h[0], h[1]);
  return 0;
}
