// Variants of the one-warp 16 x 16 Cholesky chain: which part of a step costs what.
// V bit 0: no rsqrt (cheap stand-in); bit 1: no row broadcast through shared memory (stand-in
// values); bit 2: pivot by lds instead of shfl; bit 3: no trailing updates (i >= 2)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_05782_b200/csrc/small_chains.cuh"
using namespace rutv;

template <int V>
__device__ __forceinline__ double chol_var(double (&v)[16], uint32_t rmat_a, uint32_t piv_a, int lane) {
    double d = __shfl_sync(0xffffffffu, v[0], 0);
    double inv = (V & 1) ? d * 0.01 : chain_rsqrt(d);
    double acc = 0.0;
#pragma unroll 1
    for (int c = 0; c < 16; ++c) {
        const double rcc = d * inv;
        const double rcl = lane == c ? rcc : v[0] * inv;
        const uint32_t row = rmat_a + 8u * (c * 16);
        if (!(V & 2)) {
            if (lane < 16) sts_f64(row + 8u * lane, lane >= c ? rcl : 0.0);
            __syncwarp();
        }
        const uint32_t rb = row + 8u * c;
        const double r1 = (V & 2) ? rcl * 0.5 : lds_f64(rb + 8u);
        const double v0n = __fma_rn(-r1, rcl, v[1]);
        if (V & 4) {
            if (lane == c + 1) sts_f64(piv_a, v0n);
            __syncwarp();
            d = lds_f64(piv_a);
        } else {
            d = __shfl_sync(0xffffffffu, v0n, (c + 1) & 31);
        }
        d = fabs(d) + 1.0;
        inv = (V & 1) ? d * 0.01 : chain_rsqrt(d);
        if (!(V & 8)) {
#pragma unroll
            for (int i = 2; i < 16; ++i) v[i - 1] = __fma_rn(-((V & 2) ? rcl * 0.25 : lds_f64(rb + 8u * i)), rcl, v[i]);
        }
        v[0] = v0n;
        v[15] = 0.0;
        acc += rcc;
    }
    return acc + v[3];
}

template <int V>
__global__ void k(double* out, long long* cyc, int reps) {
    __shared__ double g[256], rmat[256 + 32], pv[2];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int e = tid; e < 256; e += blockDim.x) g[e] = (e / 16 == e % 16) ? 20.0 : 1.0 / (1 + e % 7);
    __syncthreads();
    const uint32_t ra = smem_u32(rmat), pa = smem_u32(pv);
    double s = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = g[i * 16 + (lane & 15)];
        s += chol_var<V>(v, ra, pa, lane);
    }
    long long t1 = clock64();
    out[tid] = s;
    if (tid == 0) cyc[0] = (t1 - t0) / reps;
}

template <int V>
void run(double* o, long long* c) {
    long long h;
    for (int rep = 0; rep < 2; ++rep) k<V><<<1, 32>>>(o, c, 64);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": %d, \"cycles\": %lld, \"per_step\": %.0f}\n", V, h, h / 16.0);
}

int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 16);
    run<0>(o, c); run<1>(o, c); run<2>(o, c); run<3>(o, c); run<4>(o, c); run<8>(o, c); run<9>(o, c); run<11>(o, c); run<15>(o, c);
    return 0;
}
