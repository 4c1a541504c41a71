// Microbenchmark of the panel-QR per-column message chain (qr_reg.cu column loop),
// one CTA of 512 threads, 8 row-owning warps, 128 "columns".  Variants (mode bits):
//   1: partial sums to smem + named barrier (8 warps)
//   2: warp 0 sums the 8 partials and st.async-sends 32 values to its own CTA,
//      every warp waits on the mbarrier (the DSMEM all-gather with CS = 1)
//   4: 15 w_k shuffles + 16 FMA window update + 16 FMA dots
//   8: 5-level warp butterfly of 16 values
// cycles per column via clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v), "r"(rbar) : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
    uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank)); return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar); uint32_t done = 0;
    while (!done) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(a), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(512, 1) __cluster_dims__(1, 1, 1) k(int mode, double* out, long long* cyc) {
    __shared__ double part[16 * 16];
    __shared__ __align__(16) double msg[2][32];
    __shared__ uint64_t bar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwact = 8;
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncthreads();
    if (tid == 0) { mbar_arm(&bar[0], 256); mbar_arm(&bar[1], 256); }
    __syncthreads();
    double x[16];
    for (int i = 0; i < 16; ++i) x[i] = 1e-3 * (tid + i);
    double acc = 0.0;
    long long t0 = clock64();
    if (warp < nwact) {
        for (int j = 0; j < 128; ++j) {
            const int par = j & 1;
            double vals[16];
            if (mode & 16) {  // shuffles only
                const double wkl = (x[0] + lane) * 1e-9;
                double sacc = 0.0;
#pragma unroll
                for (int kk = 1; kk < 16; ++kk) sacc += __shfl_sync(0xffffffffu, wkl, kk);
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) vals[kk] = x[kk] + sacc;
            } else if (mode & 32) {  // FMAs only (w_k from a register)
                const double wk0 = (x[0] + lane) * 1e-9;
#pragma unroll
                for (int kk = 1; kk < 16; ++kk) x[kk] -= (wk0 + kk) * x[0];
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) vals[kk] = x[1] * x[kk];
            } else if (mode & 64) {  // w_k through shared memory (broadcast LDS.128)
                __shared__ __align__(16) double wks[16][16];
                if (lane < 16) wks[warp][lane] = (x[0] + lane) * 1e-9;
                __syncwarp();
#pragma unroll
                for (int k2 = 0; k2 < 8; ++k2) {
                    const double2 wp = reinterpret_cast<const double2*>(wks[warp])[k2];
                    if (k2) x[2 * k2] -= wp.x * x[0];
                    x[2 * k2 + 1] -= wp.y * x[0];
                }
                __syncwarp();
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) vals[kk] = x[1] * x[kk];
            } else if (mode & 4) {
                const double wkl = (x[0] + lane) * 1e-9;
#pragma unroll
                for (int kk = 1; kk < 16; ++kk) { const double wk = __shfl_sync(0xffffffffu, wkl, kk); x[kk] -= wk * x[0]; }
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) vals[kk] = x[1] * x[kk];
            } else {
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) vals[kk] = x[kk];
            }
            if (mode & 128) {  // transposed shared-memory reduction instead of the butterfly
                __shared__ double tr[8][32 * 17];
                double* tw = tr[warp];
#pragma unroll
                for (int kk = 0; kk < 16; ++kk) tw[lane * 17 + kk] = vals[kk];
                __syncwarp();
                const int col = lane & 15, h = lane >> 4;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                for (int r = 0; r < 16; r += 4) {
                    a0 += tw[(h * 16 + r) * 17 + col];
                    a1 += tw[(h * 16 + r + 1) * 17 + col];
                    a2 += tw[(h * 16 + r + 2) * 17 + col];
                    a3 += tw[(h * 16 + r + 3) * 17 + col];
                }
                double v = (a0 + a1) + (a2 + a3);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                vals[0] = v;
                __syncwarp();
            } else if (mode & 8) {
#pragma unroll
                for (int lvl = 0; lvl < 4; ++lvl) {
                    const int o = 16 >> lvl, n = 8 >> lvl; const bool up = (lane & o) != 0;
#pragma unroll
                    for (int i = 0; i < n; ++i) {
                        const double send = up ? vals[i] : vals[i + n], keep = up ? vals[i + n] : vals[i];
                        vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                vals[0] += __shfl_xor_sync(0xffffffffu, vals[0], 1);
            }
            if (mode & 1) {
                if ((lane & 1) == 0) part[warp * 16 + (lane >> 1)] = vals[0];
                asm volatile("bar.sync 1, %0;" ::"r"(nwact * 32) : "memory");
            }
            if (mode & 2) {
                if (warp == 0) {
                    double v = 0.0;
                    if (lane < 16) for (int w = 0; w < nwact; ++w) v += part[w * 16 + lane];
                    const uint32_t off = smem_u32(&msg[par][lane]);
                    st_async_f64(mapa_u32(off, 0), v, mapa_u32(smem_u32(&bar[par]), 0));
                }
                mbar_wait(&bar[par], (j >> 1) & 1);
                if (tid == 0 && j + 2 < 128) mbar_arm(&bar[par], 256);
                acc += msg[par][lane];
                if (mode & 1) asm volatile("bar.sync 2, %0;" ::"r"(nwact * 32) : "memory");  // slot reuse
            }
            x[0] += vals[0] * 1e-30 + acc * 1e-30;
        }
    }
    long long t1 = clock64();
    out[tid] = x[0] + acc;
    if (tid == 0) cyc[0] = (t1 - t0) / 128;
}

int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    for (int mode : {0, 8, 128, 64 + 8 + 3, 64 + 128 + 3, 4 + 8 + 3, 4 + 128 + 3}) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 512>>>(mode, o, c);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("{\"mode\": %d, \"cycles_per_column\": %lld}\n", mode, h);
    }
    return 0;
}
