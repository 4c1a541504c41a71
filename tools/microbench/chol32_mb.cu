// One-warp 32x32 Cholesky variants (column per lane), cycles per block (clock64).
#include <cstdio>
#include <cuda_runtime.h>
constexpr unsigned kF = 0xffffffffu;
template <int MODE>
__global__ void k(const double* g, double* out, long long* cyc) {
  __shared__ double A[32 * 36];
  __shared__ double rowb[2][32];
  const int lane = threadIdx.x;
  for (int i = 0; i < 32; ++i) A[i + lane * 36] = g[i + lane * 32];
  __syncwarp();
  double v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = A[i + lane * 36];
  bool bad = false;
  long long t0 = clock64();
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const double d = __shfl_sync(kF, v[c], c);
    if (!(d > 0.0)) bad = true;
    double inv, rc;
    if (MODE == 2) { rc = sqrt(d); inv = 1.0 / rc; }
    else { inv = rsqrt(d); rc = d * inv; }
    v[c] = lane == c ? rc : (lane > c ? v[c] * inv : v[c]);
    if (MODE == 1) {
      rowb[c & 1][lane] = v[c];
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i > c) { const double rci = rowb[c & 1][i]; if (lane >= i) v[i] -= rci * v[c]; }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i > c) { const double rci = __shfl_sync(kF, v[c], i); if (lane >= i) v[i] -= rci * v[c]; }
    }
  }
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 32; ++i) out[i + lane * 32] = v[i] + (bad ? 1.0 : 0.0);
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i) for (int j = 0; j < 32; ++j) h[i + j * 32] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *g, *o; long long* c; cudaMalloc(&g, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 8192, cudaMemcpyHostToDevice);
  const char* names[] = {"shfl_rsqrt", "smem_row_rsqrt", "shfl_sqrt_div"};
  for (int m = 0; m < 3; ++m) {
    long long hc = 0;
    for (int r = 0; r < 3; ++r) {
      if (m == 0) k<0><<<1, 32>>>(g, o, c);
      if (m == 1) k<1><<<1, 32>>>(g, o, c);
      if (m == 2) k<2><<<1, 32>>>(g, o, c);
      cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("{\"variant\": \"%s\", \"cycles_per_block\": %lld}\n", names[m], hc);
  }
}
