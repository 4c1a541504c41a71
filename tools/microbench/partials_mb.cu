// Microbenchmark of the QR block-phase partials loop shape (qr_reg.cu):
// 16 warps, `tasks` warps active, each `iters` k4-steps of 2 x m16n8k4 DMMA fed
// by 6 LDS.64 from a shared chunk with leading dimension LD.  Cycles via clock64.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double* c, double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}

__global__ void k(int LD, int tasks, int iters, double* out, long long* cyc) {
    extern __shared__ double chunk[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
    for (int i = tid; i < 96 * LD; i += blockDim.x) chunk[i] = 1e-3 * (i % 97);
    __syncthreads();
    long long t0 = clock64();
    double acc[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0};
    if (warp < tasks) {
        const int q = (warp % 10) * 8 + g;
        const double* pa0 = chunk + g * LD + t4;
        const double* pa1 = pa0 + 8 * LD;
        const double* pb = chunk + (16 + q) * LD + t4;
        for (int k4 = 0; k4 + 1 < iters; k4 += 2) {
            const int o = 4 * k4;
            dmma(acc, pa0[o], pa1[o], pb[o]);
            dmma(acc2, pa0[o + 4], pa1[o + 4], pb[o + 4]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[tid] = acc[0] + acc[1] + acc[2] + acc[3] + acc2[0];
    if (tid == 0) cyc[0] = t1 - t0;
}

int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    int cfgs[][3] = {{251, 10, 63}, {252, 10, 63}, {260, 10, 63}, {251, 16, 63}, {251, 1, 63}, {251, 10, 126}};
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (auto& f : cfgs) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 512, 96 * f[0] * 8>>>(f[0], f[1], f[2], o, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("{\"LD\": %d, \"tasks\": %d, \"iters\": %d, \"cycles\": %lld}\n", f[0], f[1], f[2], h);
    }
    return 0;
}
