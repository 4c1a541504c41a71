// DMMA / DFMA throughput + fragment-layout probe for sm_100a.
// Measures FP64 tensor (mma.sync .f64) issue rate for each legal shape and the
// scalar DFMA rate, and checks our fragment-layout assumptions against a
// host triple loop.  Output: one JSON object per line.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void mma_m8n8k4(double* c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double* c, const double* a, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k8(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

constexpr int CHAINS = 8;

template <int SHAPE>
__global__ void bench_mma(double* out, int iters, double seed) {
  double acc[CHAINS][4];
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = seed * (threadIdx.x - i);
  for (int c = 0; c < CHAINS; ++c) for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (SHAPE == 0) mma_m8n8k4(acc[c], a[0], b[0]);
      if (SHAPE == 1) mma_m16n8k4(acc[c], a, b[0]);
      if (SHAPE == 2) mma_m16n8k8(acc[c], a, b);
      if (SHAPE == 3) mma_m16n8k16(acc[c], a, b);
    }
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
  if (s == 12345.678) out[0] = s;
}

__global__ void bench_dfma(double* out, int iters, double seed) {
  double x[CHAINS];
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + c + threadIdx.x;
  const double m = 0.999999, ad = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], m, ad);
  }
  double s = 0;
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// Fragment-layout probe: one warp, A (M x K) and B (K x N) from global, D out.
template <int SHAPE>
__global__ void probe(const double* A, const double* B, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double c[4] = {0, 0, 0, 0};
  double a[8], b[4];
  if (SHAPE == 0) {  // 8x8x4 ; A row-major MxK, B KxN
    a[0] = A[g * 4 + t];
    b[0] = B[t * 8 + g];
    mma_m8n8k4(c, a[0], b[0]);
    D[g * 8 + 2 * t] = c[0]; D[g * 8 + 2 * t + 1] = c[1];
    return;
  }
  const int K = SHAPE == 1 ? 4 : (SHAPE == 2 ? 8 : 16);
  const int na = K / 2, nb = K / 4;
  for (int i = 0; i < na; ++i) a[i] = A[(g + 8 * (i % 2)) * K + t + 4 * (i / 2)];
  for (int i = 0; i < nb; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  if (SHAPE == 1) mma_m16n8k4(c, a, b[0]);
  if (SHAPE == 2) mma_m16n8k8(c, a, b);
  if (SHAPE == 3) mma_m16n8k16(c, a, b);
  D[g * 8 + 2 * t] = c[0]; D[g * 8 + 2 * t + 1] = c[1];
  D[(g + 8) * 8 + 2 * t] = c[2]; D[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int SHAPE>
void run_probe() {
  const int M = SHAPE == 0 ? 8 : 16, N = 8, K = SHAPE <= 1 ? 4 : (SHAPE == 2 ? 8 : 16);
  std::vector<double> A(M * K), B(K * N), D(M * N), R(M * N, 0.0);
  for (int i = 0; i < M * K; ++i) A[i] = (i * 37 % 11) - 5.0;
  for (int i = 0; i < K * N; ++i) B[i] = (i * 29 % 13) - 6.0;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j)
    for (int k = 0; k < K; ++k) R[i * N + j] += A[i * K + k] * B[k * N + j];
  double *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  probe<SHAPE><<<1, 32>>>(dA, dB, dD);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(D[i] - R[i]));
  printf("{\"probe\": \"shape%d m%dn%dk%d\", \"max_err\": %g}\n", SHAPE, M, N, K, err);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

template <int SHAPE>
void run_bench(int blocks, int threads, int iters) {
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench_mma<SHAPE><<<blocks, threads>>>(out, 10, 1.0);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    bench_mma<SHAPE><<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); best = fminf(best, ms);
  }
  const int M = SHAPE == 0 ? 8 : 16, K = SHAPE <= 1 ? 4 : (SHAPE == 2 ? 8 : 16);
  double flops = 2.0 * M * 8 * K * CHAINS * (double)iters * blocks * (threads / 32);
  printf("{\"bench\": \"mma shape%d m%dn8k%d\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
         SHAPE, M, K, blocks, threads, best, flops / best / 1e9);
  cudaFree(out);
}

void run_dfma(int blocks, int threads, int iters) {
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench_dfma<<<blocks, threads>>>(out, 10, 1.0);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    bench_dfma<<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); best = fminf(best, ms);
  }
  double flops = 2.0 * CHAINS * (double)iters * blocks * threads;
  printf("{\"bench\": \"dfma\", \"blocks\": %d, \"threads\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
         blocks, threads, best, flops / best / 1e9);
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"smem_optin\": %zu}\n", p.name,
         p.multiProcessorCount, p.major, p.minor, p.sharedMemPerBlockOptin);
  run_probe<0>(); run_probe<1>(); run_probe<2>(); run_probe<3>();
  const int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    run_bench<0>(sms * 2, wpb * 32, 20000);
    run_bench<1>(sms * 2, wpb * 32, 20000);
    run_bench<2>(sms * 2, wpb * 32, 10000);
    run_bench<3>(sms * 2, wpb * 32, 5000);
    run_dfma(sms * 2, wpb * 32, 20000);
  }
  return 0;
}
