// Cluster barrier / DSMEM latency probe on sm_100a.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_sync(long long* out, int iters, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[4096];
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  const int CS = cl.num_blocks(), rank = cl.block_rank();
  for (int i = 0; i < iters; ++i) {
    if (mode == 1) {  // all-gather 128 doubles to every CTA
      for (int idx = threadIdx.x; idx < CS * 128; idx += blockDim.x) {
        int dst = idx / 128, e = idx % 128;
        double* r = cl.map_shared_rank(buf, dst);
        r[(rank * 128 + e) % 4096] = e + i;
      }
    }
    if (mode == 2) { __syncthreads(); continue; }
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 3; ++mode)
  for (int cs : {1, 2, 4, 8, 16}) {
    for (int thr : {256, 512}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs); cfg.blockDim = dim3(thr);
      cudaLaunchAttribute at; at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
      cfg.attrs = &at; cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, k_sync, d, 2000, mode);
      cudaDeviceSynchronize();
      long long h = -1; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("{\"mode\": \"%s\", \"cs\": %d, \"threads\": %d, \"cycles_per_iter\": %lld, \"err\": \"%s\"}\n",
             mode == 0 ? "cluster.sync" : (mode == 1 ? "allgather128+sync" : "__syncthreads"), cs, thr, h,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
