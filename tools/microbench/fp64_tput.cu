// One-warp issue rate of independent FP64 / LDS / DMMA instructions (cycles per warp instruction).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = a;
  __syncthreads();
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = a + i + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) x[i] = fma(x[i], b, a);
      if (MODE == 1) x[i] = fma(sm[(i + it) & 63], b, x[i]);
      if (MODE == 2) x[i] = x[i] * b;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"16 independent dfma", "16 x (lds broadcast + dfma)", "16 independent dmul"};
  const int n = 2048;
  for (int m = 0; m < 3; ++m) for (int warps : {1, 2, 4, 8}) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<1, 32 * warps>>>(o, c, 1.0000001, 0.9999999, n);
      if (m == 1) k<1><<<1, 32 * warps>>>(o, c, 1.0000001, 0.9999999, n);
      if (m == 2) k<2><<<1, 32 * warps>>>(o, c, 1.0000001, 0.9999999, n);
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("{\"op\": \"%s\", \"warps\": %d, \"cycles_per_warp_instr\": %.2f}\n", names[m], warps, double(h) / n / 16);
  }
  return 0;
}
