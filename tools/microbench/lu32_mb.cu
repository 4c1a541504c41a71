// One-warp 32x32 LU (no pivoting) variants, lane = column; cycles per block (clock64).
//   0: multipliers broadcast by shuffles (cqr_lu_kernel's form)
//   1: lane c stores its multiplier column to shared memory with 16-byte
//      stores, every lane reads it back with 16-byte broadcast loads
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned kF = 0xffffffffu;
template <int MODE>
__global__ void k(const double* g, double* out, long long* cyc) {
  __shared__ __align__(16) double A[32 * 36];
  __shared__ __align__(16) double colb[2][32];
  const int lane = threadIdx.x;
  for (int i = 0; i < 32; ++i) A[i + lane * 36] = g[i + lane * 32];
  __syncwarp();
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = A[i + lane * 36];
  bool bad = false;
  double myinv = 1.0;
  __syncwarp();
  long long t0 = clock64();
  double piv = __shfl_sync(kF, v[0], 0);
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    bad |= !(fabs(piv) >= 0.25);
    const double inv = __drcp_rn(piv);
    myinv = lane == c ? inv : myinv;
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i > c && lane == c) v[i] *= inv;
      if (c + 1 < 32) {
        const int n1 = c + 1 < 32 ? c + 1 : c;
        const double l1 = __shfl_sync(kF, v[n1], c);
        if (lane > c) v[n1] = __fma_rn(-l1, v[c], v[n1]);
        piv = __shfl_sync(kF, v[n1], n1);
      }
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i > c + 1) {
          const double li = __shfl_sync(kF, v[i], c);
          if (lane > c) v[i] = __fma_rn(-li, v[c], v[i]);
        }
    } else {
      double* cb = colb[c & 1];
      if (lane == c) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          double2 m;
          m.x = i > c ? v[i] * inv : 0.0;
          m.y = i + 1 > c ? v[i + 1] * inv : 0.0;
          *reinterpret_cast<double2*>(cb + i) = m;
          if (i > c) v[i] = m.x;
          if (i + 1 > c) v[i + 1] = m.y;
        }
      }
      __syncwarp();
      if (c + 1 < 32) {
        const int n1 = c + 1 < 32 ? c + 1 : c;
        if (lane > c) v[n1] = __fma_rn(-cb[n1], v[c], v[n1]);
        piv = __shfl_sync(kF, v[n1], n1);
      }
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const double2 m = *reinterpret_cast<const double2*>(cb + i);
        if (i > c + 1 && lane > c) v[i] = __fma_rn(-m.x, v[c], v[i]);
        if (i + 1 > c + 1 && lane > c) v[i + 1] = __fma_rn(-m.y, v[c], v[i + 1]);
      }
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 32; ++i) out[i + lane * 32] = v[i] + (bad ? 1.0 : 0.0) + myinv * 0.0;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i + j * 32] = (i == j ? 4.0 : 0.0) + 1.0 / (1 + i + 2 * j);
  double *g, *o; long long* c; cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
  double r0[1024], r1[1024];
  const char* names[] = {"shfl", "smem_vec"};
  for (int m = 0; m < 2; ++m) {
    long long hc = 0;
    for (int r = 0; r < 3; ++r) {
      if (m == 0) k<0><<<1, 32>>>(g, o, c);
      if (m == 1) k<1><<<1, 32>>>(g, o, c);
      cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    }
    cudaMemcpy(m ? r1 : r0, o, 8192, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"cycles_per_block\": %lld}\n", names[m], hc);
  }
  double md = 0; for (int i = 0; i < 1024; ++i) md = fmax(md, fabs(r0[i] - r1[i]));
  printf("{\"max_diff\": %g}\n", md);
}
