// One-warp 16 x 16 Cholesky / LU chains of qr_reg.cu's micro-panel fast path, timed alone:
// cycles per call with 1 warp, and with 15 more warps parked at a CTA barrier.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_05782_b200/csrc/small_chains.cuh"

__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ double g[256], rmat[256 + 32], rdinv[16], ud[16];
  __shared__ __align__(16) double scr[96];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 256; e += blockDim.x) g[e] = (e / 16 == e % 16) ? 20.0 : 1.0 / (1 + e % 7);
  __syncthreads();
  for (int mode = 0; mode < 2; ++mode) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (warp == 0) {
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = g[i * 16 + (lane & 15)] * (mode ? 0.01 : 1.0) + ((mode && i == (lane & 15)) ? 1.0 : 0.0);
        bool brk;
        if (mode == 0) {
          double mn, mx;
          brk = rutv::warp_chol16(v, rutv::smem_u32(rmat), rutv::smem_u32(rdinv), rutv::smem_u32(scr), mn, mx, lane);
        } else {
          brk = rutv::warp_lu16(v, rutv::smem_u32(rmat), rutv::smem_u32(rdinv), rutv::smem_u32(ud), rutv::smem_u32(scr), lane);
        }
        if (brk && lane == 0) out[1] = 1.0;
      }
      __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[mode] = (t1 - t0) / reps;
  }
  if (tid < 256) out[2 + tid] = rmat[tid];
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 16);
  for (int threads : {32, 512}) {
    long long h[2];
    for (int rep = 0; rep < 2; ++rep) k<<<1, threads>>>(o, c, 64);
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("{\"threads\": %d, \"chol16_cycles\": %lld, \"lu16_cycles\": %lld}\n", threads, h[0], h[1]);
  }
  return 0;
}
