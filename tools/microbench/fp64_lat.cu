// FP64 latency probe on sm_100a: dependent chains of DFMA / DADD / div / sqrt /
// rcp / shfl, one warp, cycles per op (clock64).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-3;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (MODE == 0) x = fma(x, b, a);
    if (MODE == 1) x = x + b;
    if (MODE == 2) x = a / x;
    if (MODE == 3) x = sqrt(x + a);
    if (MODE == 4) x = __drcp_rn(x + a);
    if (MODE == 5) x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0;
    if (MODE == 6) x = __shfl_xor_sync(0xffffffffu, x, 1);
    if (MODE == 9) x = rsqrt(x + a);
    if (MODE == 7) {  // dependent mma.sync m16n8k4 f64 chain (accumulator dependency)
      double c0 = x, c1 = x, c2 = x, c3 = x;
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a), "d"(b), "d"(a));
      x = c0 + 0.0 * (c1 + c2 + c3);
    }
    if (MODE == 8) {  // same, the accumulator kept in registers (no DADD on the chain)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(x), "+d"(b) : "d"(a), "d"(a));
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"dfma", "dadd", "ddiv", "dsqrt", "drcp_rn", "shfl+dadd", "shfl", "mma16x8x4+dadd", "mma8x8x4", "drsqrt"};
  const int n = 4096;
  for (int m = 0; m < 10; ++m) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (m) {
        case 0: k<0><<<1, 32>>>(o, c, 1.0000001, 0.9999999, n); break;
        case 1: k<1><<<1, 32>>>(o, c, 1.0000001, 1e-9, n); break;
        case 2: k<2><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
        case 3: k<3><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
        case 4: k<4><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
        case 5: k<5><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
        case 6: k<6><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
        case 7: k<7><<<1, 32>>>(o, c, 1e-3, 1e-3, n); break;
        case 8: k<8><<<1, 32>>>(o, c, 1e-3, 1e-3, n); break;
        case 9: k<9><<<1, 32>>>(o, c, 1.5, 1.0, n); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[m], double(h) / n);
  }
  return 0;
}
