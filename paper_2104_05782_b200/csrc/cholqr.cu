// cholqr.cu -- panel QR by Cholesky-QR2 + Householder reconstruction.
//
// The reference factors every panel with column-by-column Householder
// (proj/src/householder.cpp:48-67), whose 128 dependent column steps make the
// panel QR latency-bound on the GPU (qr_reg.cu: ~2 us per column, 250-360 us
// per 128-column panel).  For a full-rank s x w panel Y (16 <= w <= 128,
// s >= 2w) the same factorization is obtained from level-3 work plus small
// w x w factorizations:
//
//   Cholesky-QR2:  R1 = chol(Y'Y), Q1 = Y R1^{-1};  R2 = chol(Q1'Q1),
//                  Q = Q1 R2^{-1};  R = R2 R1      (R_jj > 0)
//   Householder reconstruction: the reference's convention (beta >= 0, i.e.
//   R_jj >= 0) makes the thin QR unique, so Q = H_1...H_w (:, 0:w) with the
//   reference's reflectors.  Writing H_1...H_w = I - V T V' (V unit lower
//   trapezoidal, T upper, diag(T) = tau):
//       I - Q(0:w, :) = V1 (T V1')     -> LU without pivoting: L = V1, U = T V1'
//       -Q(w:s, :)    = V2 (T V1')     -> V2 = -Q(w:s, :) U^{-1}
//   and tau_j = U_jj.
// The packed result (R above the diagonal, V below) and tau are exactly what
// the Householder kernel produces, up to rounding.
//
// The small factorizations (Cholesky + triangular inverse, LU + inverse) run
// in ONE CTA each, blocked by 32: a 32 x 32 diagonal block is factored (and
// inverted) by one warp in registers with shuffles only, every off-diagonal
// block product is a 32 x 32 warp tile of DMMA (mma.sync m16n8k4 f64) from
// shared memory -- a handful of CTA barriers per 32 columns instead of two
// per column.
//
// Safety: the result is only valid when the path is numerically sound; each
// panel ORs a flag word on the device:
//   * 1/4: Cholesky breakdown (pivot <= 0 or not finite) in pass 1 / pass 2;
//   * 2: min/max diag(R1) < 1e-7 (Cholesky-QR2 needs cond(Y) well below 1/sqrt(eps));
//   * 16: Q1'Q1 farther than 0.1 from I (pass 1 lost too much orthogonality);
//   * 8: an LU pivot |tau_j| < 0.25 (a reflector close to the identity: the
//     reconstruction divides by tau_j).
// Two modes:
//   * deferred (the factorization driver, RUTV_CHOLQR=2): the packed result is
//     written in place without any host synchronisation and the flag word is
//     shared by the whole factorization; the driver reads it once at the end
//     and, if any panel was unsafe, re-runs the factorization with the
//     Householder kernels (randutv.cu);
//   * immediate (RUTV_CHOLQR=1, other callers): the flag is read back after the
//     panel and the caller falls back to the Householder kernel on failure.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rutv_common.cuh"
#include "small_chains.cuh"

namespace rutv {

namespace {

constexpr int kST = 256;  // threads of the small-factorization kernels (8 warps)
constexpr int kW = kST / 32;
constexpr unsigned kFull = 0xffffffffu;

// phase clocks of the last small-factorization launches (debug, rutv_b200_debug_cqr_clocks)
__device__ long long g_cqr_clk[128];
#define CQR_CLK(slot) \
    if (threadIdx.x == 0) g_cqr_clk[(slot)] = clock64()

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// Warp tile: acc (32 x 32) += A (32 x 32) B (32 x 32) with element accessors
// fa(i, k), fb(k, j).  Lane (g, t) = (lane >> 2, lane & 3); accumulator
// acc[mt][nt][r] is element (16 mt + g + 8 (r >= 2), 8 nt + 2 t + (r & 1)).
template <class FA, class FB>
__device__ __forceinline__ void mma32(double (&acc)[2][4][4], FA fa, FB fb) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
        double a[2][2], b[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            a[mt][0] = fa(16 * mt + g, k + t);
            a[mt][1] = fa(16 * mt + g + 8, k + t);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) b[nt] = fb(k + t, 8 * nt + g);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
}

__device__ __forceinline__ void zero32(double (&acc)[2][4][4]) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[mt][nt][r] = 0.0;
}

// visit every accumulator element: f(i, j, value)
template <class F>
__device__ __forceinline__ void each32(const double (&acc)[2][4][4], F f) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) f(16 * mt + g + (r >= 2 ? 8 : 0), 8 * nt + 2 * t + (r & 1), acc[mt][nt][r]);
}

// Shared-memory matrix: column-major P x P, LD = P + 4 (LD = 4 mod 16: the
// DMMA fragment loads of a half-warp hit 16 distinct bank pairs).
struct SMat {
    double* a;
    int ld;
    __device__ __forceinline__ double& operator()(int i, int k) const { return a[i + k * ld]; }
};

// Column-oriented back substitution in one warp: lane k gets column k of
// X = U^{-1} for the 32 x 32 upper block at (j0, j0) of M with reciprocal
// diagonal dinv[j0..]; x[m] for m <= k (0 above).
__device__ __forceinline__ void warp_upper_inv(const SMat& M, int j0, const double* dinv, double (&x)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        const double xi = x[i] * dinv[j0 + i];
        x[i] = xi;
#pragma unroll
        for (int m = 0; m < i; ++m) x[m] -= M(j0 + m, j0 + i) * xi;
    }
}

__host__ __device__ inline size_t small_smem_bytes(int p) {
    const int P = (p + 31) / 32 * 32;
    // A (P x (P+4)), dinv, dg, rowb (2 x 32), XD, XL, tmp (3 x 32 x 36)
    return (static_cast<size_t>(P) * (P + 4) + 2 * P + 64 + 5 * 32 * 36) * sizeof(double);
}

constexpr int TL = 36;  // leading dimension of the 32 x 32 scratch blocks

// A(i, k) = src(i, k) for i, k < p, identity padding up to P; by columns
// (warp w: columns w, w + 8, ...; lanes: rows), 16 loads in flight per thread.
template <class F>
__device__ __forceinline__ void load_square(const SMat& A, int p, int P, F src) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
    for (int k0 = warp; k0 < P; k0 += 4 * kW) {
        double t[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int k = k0 + u * kW, i = lane + 32 * r;
                t[u][r] = (i < p && k < p) ? src(i, k) : (i == k ? 1.0 : 0.0);
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int k = k0 + u * kW, i = lane + 32 * r;
                if (i < P && k < P) A(i, k) = t[u][r];
            }
    }
}

// f(i, k) for i in [r0, r1), k in [c0, c1), by columns (coalesced global stores)
template <class F>
__device__ __forceinline__ void for_rect(int r0, int r1, int c0, int c1, F f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = c0 + warp; k < c1; k += kW)
        for (int i = r0 + lane; i < r1; i += 32) f(i, k);
}

// X = U^{-1} of the upper factor is built one block column per step:
//   X_IJ = -(sum_{L=I..J-1} X_IL U_LJ) X_JJ,   I < J,
// X(i, k), i < k, stored TRANSPOSED in A's strictly lower part (A(k, i)),
// X(k, k) = dinv[k].  Part 1 (with the block-row phase): T_I = sum X_IL U_LJ.
__device__ __forceinline__ double xinv(const SMat& A, const double* dinv, int i, int k) {
    const double v = A(k, i);
    return i < k ? v : (i == k ? dinv[i] : 0.0);
}

__device__ __forceinline__ void inv_part1(const SMat& A, const double* dinv, double* tmp, int J, int task0) {
    const int warp = threadIdx.x >> 5, j0 = 32 * J;
    for (int I = 0; I < J; ++I) {
        if ((task0 + I) % kW != warp) continue;
        const int i0 = 32 * I;
        double acc[2][4][4];
        zero32(acc);
        mma32(
            acc, [&](int i, int m) { return xinv(A, dinv, i0 + i, i0 + m); },
            [&](int m, int c) { return A(i0 + m, j0 + c); });
        for (int L = I + 1; L < J; ++L) {
            const int l0 = 32 * L;
            mma32(
                acc, [&](int i, int m) { return A(l0 + m, i0 + i); }, [&](int m, int c) { return A(l0 + m, j0 + c); });
        }
        double* T = tmp + I * 32 * TL;
        each32(acc, [&](int i, int j, double v) { T[i + j * TL] = v; });
    }
}

// Part 2 (with the trailing phase): X_IJ = -T_I X_JJ (X_JJ in XD, column-major, ld TL)
__device__ __forceinline__ void inv_part2(const SMat& A, const double* XD, const double* tmp, int J, int task0) {
    const int warp = threadIdx.x >> 5, j0 = 32 * J;
    for (int I = 0; I < J; ++I) {
        if ((task0 + I) % kW != warp) continue;
        const int i0 = 32 * I;
        const double* T = tmp + I * 32 * TL;
        double acc[2][4][4];
        zero32(acc);
        mma32(
            acc, [&](int i, int m) { return T[i + m * TL]; }, [&](int m, int c) { return XD[m + c * TL]; });
        each32(acc, [&](int i, int j, double v) { A(j0 + j, i0 + i) = -v; });
    }
}

// Upper Cholesky G = R'R (p x p, p <= 128), X = R^{-1}; optionally Rp = R R1
// (pass 2: the final R = R2 R1).  Flags: breakdown -> brk_bit; pass 1
// (check_ratio): min/max diag(R) < 1e-7 -> 2; pass 2 (check_orth):
// max |G - I| > 0.1 -> 16.
__global__ void __launch_bounds__(kST) cqr_chol_kernel(const double* __restrict__ g, int64_t ldg, int p, double* r,
                                                       double* rinv, const double* __restrict__ r1, double* rp,
                                                       int* flag, int brk_bit, int check_ratio, int check_orth) {
    extern __shared__ double sm[];
    const int NB = (p + 31) >> 5, P = NB * 32;
    const SMat A{sm, P + 4};
    double* dinv = sm + static_cast<size_t>(P) * (P + 4);
    double* rowb = dinv + 2 * P;  // [2][32]
    double* XD = rowb + 64;       // X_JJ
    double* tmp = XD + 2 * 32 * TL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = r1 ? 16 : 0;
    CQR_CLK(base);
    load_square(A, p, P, [&](int i, int k) { return g[i + static_cast<int64_t>(k) * ldg]; });
    __syncthreads();
    // Pass 2 factors G = Q1'Q1 = I + E.  With |E| <= 1e-11 the series R2 = I + U1, R2^-1 = I - U1,
    // U1 = striu(E) + diag(E) / 2, is exact to ||U1||^2 <= (128 * 1e-11)^2 ~ 1.6e-18: no factorization
    // (the four 32-column block steps are ~100 K cycles of this kernel's ~145 K).
    bool series = false;
    if (check_orth) {
        bool bad_orth = false, big = false;
        for_rect(0, p, 0, p, [&](int i, int k) {
            const double e = fabs(A(i, k) - (i == k ? 1.0 : 0.0));
            bad_orth |= e > 0.1;
            big |= !(e <= 1e-11);
        });
        if (__any_sync(kFull, bad_orth) && lane == 0) atomicOr(flag, 16);
        series = __syncthreads_or(big ? 1 : 0) == 0;
        if (series) {
            // upper triangle: R2; strictly lower: R2^-1 transposed (the layout xinv() reads)
            for_rect(0, P, 0, P, [&](int i, int k) {
                if (i < k) {
                    A(k, i) = -A(i, k);
                } else if (i == k) {
                    const double d = 1.0 + 0.5 * (A(k, k) - 1.0);
                    A(k, k) = d;
                    dinv[k] = 1.0 / d;
                }
            });
            __syncthreads();
        }
    }
    CQR_CLK(base + 1);
    bool bad = false;
    for (int J = 0; J < (series ? 0 : NB); ++J) {
        const int j0 = 32 * J;
        if (warp == 0) {
            // diagonal block in registers: lane k holds column j0 + k; row c of
            // R broadcast through shared memory
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = A(j0 + i, j0 + lane);
            // The chain is kept free of data-dependent control flow: a breakdown
            // (pivot <= 0 or not finite) only sets the flag -- the panel is then
            // discarded by the caller -- and 1/R(c, c) is stored after the loop.
            // The next pivot is formed by its owner lane from its own R(c, c+1)
            // (no shared-memory round trip on the column chain), with the same
            // fma as the broadcast update, so the bits agree.
            double myinv = 1.0;
            bool brk = false;
            double d = __shfl_sync(kFull, v[0], 0);
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                brk |= !(d > 0.0) || !isfinite(d);
                const double inv = rsqrt(d), rc = d * inv;
                v[c] = lane == c ? rc : (lane > c ? v[c] * inv : v[c]);  // row c of R
                myinv = lane == c ? inv : myinv;
                if (c + 1 < 32) d = __shfl_sync(kFull, __fma_rn(-v[c], v[c], v[c + 1 < 32 ? c + 1 : c]), c + 1);
                double* rb = rowb + (c & 1) * 32;
                rb[lane] = v[c];
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i > c) {
                        const double rci = rb[i];  // R(c, i)
                        if (lane >= i) v[i] = __fma_rn(-rci, v[c], v[i]);
                    }
                }
            }
            dinv[j0 + lane] = myinv;
            bad |= brk;
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (i <= lane) A(j0 + i, j0 + lane) = v[i];
            __syncwarp();
            double x[32];
            warp_upper_inv(A, j0, dinv, x);
#pragma unroll
            for (int m = 0; m < 32; ++m) XD[m + lane * TL] = x[m];
        }
        __syncthreads();
        CQR_CLK(base + 2 + 3 * J);
        const int nr = NB - 1 - J;
        // block row R(J, K) = X_JJ' A(J, K), K > J (in place); X part 1
        for (int K = J + 1 + warp; K < NB; K += kW) {
            const int k0 = 32 * K;
            double acc[2][4][4];
            zero32(acc);
            mma32(
                acc, [&](int i, int m) { return XD[m + i * TL]; }, [&](int m, int c) { return A(j0 + m, k0 + c); });
            __syncwarp();
            each32(acc, [&](int i, int j, double v) { A(j0 + i, k0 + j) = v; });
        }
        inv_part1(A, dinv, tmp, J, nr);
        __syncthreads();
        CQR_CLK(base + 3 + 3 * J);
        // X_JJ into the diagonal block's lower triangle; trailing
        // A(K, L) -= R(J, K)' R(J, L), J < K <= L; X part 2
        for (int e = tid; e < 32 * 32; e += kST) {
            const int m = e & 31, k = e >> 5;
            if (m < k) A(j0 + k, j0 + m) = XD[m + k * TL];
        }
        int task = 0;
        for (int K = J + 1; K < NB; ++K)
            for (int L = K; L < NB; ++L, ++task) {
                if (task % kW != warp) continue;
                const int k0 = 32 * K, l0 = 32 * L;
                double acc[2][4][4];
                zero32(acc);
                mma32(
                    acc, [&](int i, int m) { return A(j0 + m, k0 + i); }, [&](int m, int c) { return A(j0 + m, l0 + c); });
                each32(acc, [&](int i, int j, double v) { A(k0 + i, l0 + j) -= v; });
            }
        inv_part2(A, XD, tmp, J, task);
        __syncthreads();
        CQR_CLK(base + 4 + 3 * J);
    }
    if (warp == 0 && __any_sync(kFull, bad) && lane == 0) atomicOr(flag, brk_bit);
    CQR_CLK(base + 14);
    for_rect(0, p, 0, p, [&](int i, int k) {
        r[i + static_cast<int64_t>(k) * p] = i <= k ? A(i, k) : 0.0;
        rinv[i + static_cast<int64_t>(k) * p] = xinv(A, dinv, i, k);
    });
    if (check_ratio && warp == 0) {
        double mn = INFINITY, mx = 0.0;
        for (int j = lane; j < p; j += 32) {
            mn = fmin(mn, A(j, j));
            mx = fmax(mx, A(j, j));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
            mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
        }
        if (lane == 0 && !(mn > 1e-7 * mx)) atomicOr(flag, 2);
    }
    if (r1) {  // Rp = R R1 (both upper): block (I, K) = sum_{L=I..K} R_IL R1_LK, R1 from L2
        int t2 = 0;
        for (int I = 0; I < NB; ++I)
            for (int K = I; K < NB; ++K, ++t2) {
                if (t2 % kW != warp) continue;
                const int i0 = 32 * I, k0 = 32 * K;
                double acc[2][4][4];
                zero32(acc);
                for (int L = I; L <= K; ++L) {
                    const int l0 = 32 * L;
                    mma32(
                        acc, [&](int i, int m) { return (l0 + m >= i0 + i) ? A(i0 + i, l0 + m) : 0.0; },
                        [&](int m, int c) {
                            const int row = l0 + m, col = k0 + c;
                            const bool in = row < p && col < p;
                            const double v = r1[in ? row + static_cast<int64_t>(col) * p : 0];
                            return row > col ? 0.0 : (in ? v : (row == col ? 1.0 : 0.0));
                        });
                }
                each32(acc, [&](int i, int j, double v) {
                    const int row = i0 + i, col = k0 + j;
                    if (row < p && col < p) rp[row + static_cast<int64_t>(col) * p] = row <= col ? v : 0.0;
                    if (I != K && k0 + i < p && i0 + j < p)  // the strictly lower block (K, I) is zero
                        rp[(k0 + i) + static_cast<int64_t>(i0 + j) * p] = 0.0;
                });
            }
    }
    __syncthreads();
    CQR_CLK(base + 15);
}

// LU without pivoting of B = I - Q(0:p, 0:p) (p <= 128).  Writes the packed
// top block [R upper (from rfull); L strictly lower] to top (ld ldtop),
// tau = diag(U), and U^{-1} (p x p, ld p).  |pivot| < 0.25 -> flag 8.
__global__ void __launch_bounds__(kST) cqr_lu_kernel(const double* __restrict__ q, int64_t ldq, int p,
                                                     const double* __restrict__ rfull, double* top, int64_t ldtop,
                                                     double* uinv, double* tau, int* flag) {
    extern __shared__ double sm[];
    const int NB = (p + 31) >> 5, P = NB * 32;
    const SMat A{sm, P + 4};
    double* dinv = sm + static_cast<size_t>(P) * (P + 4);
    double* rowb = dinv + 2 * P;
    double* XD = rowb + 64;     // U_JJ^{-1}
    double* XL = XD + 32 * TL;  // L_JJ^{-1}
    double* tmp = XL + 32 * TL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int base = 32;
    CQR_CLK(base);
    load_square(A, p, P, [&](int i, int k) { return (i == k ? 1.0 : 0.0) - q[i + static_cast<int64_t>(k) * ldq]; });
    __syncthreads();
    CQR_CLK(base + 1);
    bool bad = false;
    for (int J = 0; J < NB; ++J) {
        const int j0 = 32 * J;
        if (warp == 0) {
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = A(j0 + i, j0 + lane);
            __syncwarp();
            // Branch-free chain (a small pivot only sets the flag) on a shifting register window,
            // one shared-memory round trip per step (small_chains.cuh, warp_lu16): lane c
            // publishes its pivot and the raw column below it, every lane reads them back, scales
            // by the reciprocal itself and updates with ONE fma per entry; row c of the packed
            // factors goes straight to A.  ~330 cycles per column (a shuffle per multiplier: 800).
            bool brk = false;
            const uint32_t colb = smem_u32(rowb);
#pragma unroll 1
            for (int c = 0; c < 32; ++c) {
                const uint32_t col = colb + 8u * static_cast<uint32_t>((c & 1) * 32);
                const double u0 = v[0];  // U(c, lane) for lane >= c, L(c, lane) for lane < c
                if (lane == c) {
#pragma unroll
                    for (int i = 0; i < 32; i += 2) sts_v2f64(col + 8u * i, v[i], v[i + 1]);
                }
                __syncwarp();
                const double piv = lds_f64(col);
                const double inv = chain_rcp(piv);
                const double a = lane > c ? -(u0 * inv) : (lane == c ? inv - 1.0 : 0.0);
#pragma unroll
                for (int i = 1; i < 32; ++i) v[i - 1] = __fma_rn(lds_f64(col + 8u * i), a, v[i]);
                v[31] = 0.0;
                brk |= !(fabs(piv) >= 0.25) || !isfinite(piv);
                A(j0 + c, j0 + lane) = u0;
                if (lane == c) dinv[j0 + c] = inv;
            }
            bad |= brk;
            __syncwarp();
            double x[32];
            warp_upper_inv(A, j0, dinv, x);  // XD = U_JJ^{-1} (lane k: column k)
#pragma unroll
            for (int m = 0; m < 32; ++m) XD[m + lane * TL] = x[m];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
#pragma unroll
                for (int m = i + 1; m < 32; ++m) x[m] -= A(j0 + m, j0 + i) * x[i];
#pragma unroll
            for (int m = 0; m < 32; ++m) XL[m + lane * TL] = x[m];
        }
        __syncthreads();
        CQR_CLK(base + 2 + 3 * J);
        const int nr = NB - 1 - J;
        // L_JJ out; U(J, K) = XL A(J, K) and L(K, J) = A(K, J) XU for K > J; X part 1
        for_rect(j0, j0 + 32, j0, j0 + 32, [&](int i, int k) {
            if (i > k && i < p && k < p) top[i + static_cast<int64_t>(k) * ldtop] = A(i, k);
        });
        for (int task = warp; task < 2 * nr; task += kW) {
            const int K = J + 1 + (task % nr), k0 = 32 * K;
            double acc[2][4][4];
            zero32(acc);
            if (task < nr) {
                mma32(
                    acc, [&](int i, int m) { return XL[i + m * TL]; }, [&](int m, int c) { return A(j0 + m, k0 + c); });
                __syncwarp();
                each32(acc, [&](int i, int j, double v) { A(j0 + i, k0 + j) = v; });
            } else {
                mma32(
                    acc, [&](int i, int m) { return A(k0 + i, j0 + m); }, [&](int m, int c) { return XD[m + c * TL]; });
                __syncwarp();
                each32(acc, [&](int i, int j, double v) { A(k0 + i, j0 + j) = v; });
            }
        }
        inv_part1(A, dinv, tmp, J, 2 * nr);
        __syncthreads();
        CQR_CLK(base + 3 + 3 * J);
        // L(K, J) out; X_JJ into the diagonal block's lower triangle; trailing
        // A(K, L) -= L(K, J) U(J, L), K, L > J; X part 2
        for_rect(j0 + 32, P, j0, j0 + 32, [&](int i, int k) {
            if (i < p && k < p) top[i + static_cast<int64_t>(k) * ldtop] = A(i, k);
        });
        for (int e = tid; e < 32 * 32; e += kST) {
            const int m = e & 31, k = e >> 5;
            if (m < k) A(j0 + k, j0 + m) = XD[m + k * TL];
        }
        for (int task = warp; task < nr * nr; task += kW) {
            const int K = J + 1 + task / nr, L = J + 1 + task % nr, k0 = 32 * K, l0 = 32 * L;
            double acc[2][4][4];
            zero32(acc);
            mma32(
                acc, [&](int i, int m) { return A(k0 + i, j0 + m); }, [&](int m, int c) { return A(j0 + m, l0 + c); });
            each32(acc, [&](int i, int j, double v) { A(k0 + i, l0 + j) -= v; });
        }
        inv_part2(A, XD, tmp, J, nr * nr);
        __syncthreads();
        CQR_CLK(base + 4 + 3 * J);
    }
    if (warp == 0 && __any_sync(kFull, bad) && lane == 0) atomicOr(flag, 8);
    CQR_CLK(base + 14);
    for_rect(0, p, 0, p, [&](int i, int k) {
        if (i <= k) top[i + static_cast<int64_t>(k) * ldtop] = rfull[i + static_cast<int64_t>(k) * p];
        if (i == k) tau[i] = A(i, i);
        uinv[i + static_cast<int64_t>(k) * p] = xinv(A, dinv, i, k);
    });
    __syncthreads();
    CQR_CLK(base + 16);
}


// Compact-WY T factor (householder.cpp:76-97) by inversion: the forward
// recurrence T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j) is exactly the inverse
// of the upper triangular U = diag(1/tau) + striu(G), G = W'W, so for
// p <= 128 with every tau != 0 T = U^{-1} is built by the same blocked
// inversion as R^{-1} above (diagonal blocks by one warp each, off-diagonal
// block columns by DMMA) -- one CTA, a few barriers.  A tau = 0 reflector
// (householder.cpp:26-27: H = I) has no inverse form; that rare panel takes
// the recurrence column by column.
__global__ void __launch_bounds__(kST) form_t_inv_kernel(const double* __restrict__ g, int64_t ldg,
                                                         const double* __restrict__ tau, int p, double* t,
                                                         int64_t ldt) {
    extern __shared__ double sm[];
    const int NB = (p + 31) >> 5, P = NB * 32;
    const SMat A{sm, P + 4};
    double* dinv = sm + static_cast<size_t>(P) * (P + 4);  // 1 / U_ii = tau_i
    double* tmp = dinv + 2 * P + 64 + 2 * 32 * TL;  // the chol kernel's tmp
    __shared__ int s_zero;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_zero = 0;
    __syncthreads();
    load_square(A, p, P, [&](int i, int k) { return g[i + static_cast<int64_t>(k) * ldg]; });
    for (int i = tid; i < P; i += kST) {
        const double ti = i < p ? tau[i] : 1.0;
        dinv[i] = ti;
        if (ti == 0.0) s_zero = 1;
    }
    __syncthreads();
    if (s_zero) {  // recurrence, column by column (T read back from global)
        for (int j = 0; j < p; ++j) {
            const double tj = tau[j];
            for (int i = tid; i < p; i += kST) {
                double v;
                if (i < j) {
                    double acc = 0.0;
                    for (int m = i; m < j; ++m) acc += t[i + static_cast<int64_t>(m) * ldt] * A(m, j);
                    v = -tj * acc;
                } else {
                    v = i == j ? tj : 0.0;
                }
                t[i + static_cast<int64_t>(j) * ldt] = v;
            }
            __syncthreads();
        }
        return;
    }
    for (int J = warp; J < NB; J += kW) {
        const int j0 = 32 * J;
        double x[32];
        warp_upper_inv(A, j0, dinv, x);
#pragma unroll
        for (int m = 0; m < 32; ++m)
            if (m < lane) A(j0 + lane, j0 + m) = x[m];
    }
    __syncthreads();
    for (int J = 1; J < NB; ++J) {
        inv_part1(A, dinv, tmp, J, 0);
        __syncthreads();
        const int j0 = 32 * J;
        for (int I = warp; I < J; I += kW) {  // X_IJ = -T_I X_JJ
            const int i0 = 32 * I;
            const double* T = tmp + I * 32 * TL;
            double acc[2][4][4];
            zero32(acc);
            mma32(
                acc, [&](int i, int m) { return T[i + m * TL]; },
                [&](int m, int c) { return xinv(A, dinv, j0 + m, j0 + c); });
            each32(acc, [&](int i, int j, double v) { A(j0 + j, i0 + i) = -v; });
        }
        __syncthreads();
    }
    for_rect(0, p, 0, p, [&](int i, int k) { t[i + static_cast<int64_t>(k) * ldt] = xinv(A, dinv, i, k); });
}

__global__ void commit_kernel(int64_t s, int p, const double* __restrict__ topb, const double* __restrict__ l2,
                              int64_t ldl2, double* a, int64_t lda) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < s * p;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % s, j = e / s;
        a[i + j * lda] = i < p ? topb[i + j * p] : l2[(i - p) + j * ldl2];
    }
}

void small_attr() {
    once_per_device(reinterpret_cast<const void*>(cqr_chol_kernel), [] {
        const int bytes = static_cast<int>(small_smem_bytes(128));
        RUTV_CUDA(cudaFuncSetAttribute(cqr_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        RUTV_CUDA(cudaFuncSetAttribute(cqr_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    });
}

// immediate mode (RUTV_CHOLQR=1) for callers outside the factorization driver
bool immediate_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RUTV_CHOLQR");
        return e && std::strcmp(e, "1") == 0;
    }();
    return on;
}

thread_local int* t_deferred_flag = nullptr;

// Tall sub-panels take the fast path by default (immediate mode): rows per
// panel from which Cholesky-QR2 beats the cluster Householder kernel
// (RUTV_CHOLQR_MIN_ROWS, 0 = never).
int64_t tall_min_rows() {
    static const int64_t v = [] {
        const char* e = std::getenv("RUTV_CHOLQR_MIN_ROWS");
        return e ? std::atoll(e) : static_cast<int64_t>(4608);
    }();
    return v;
}

void gemm_w(cudaStream_t st, double alpha, Op ta, const DView& a, Op tb, const DView& b, double beta,
            const DView& c) {
    const int64_t k = ta == Op::N ? a.cols : a.rows;
    const int64_t we = gemm_work_elems(c.rows, c.cols, k);
    DevBuf w(we, st);
    gemm(st, alpha, ta, a, tb, b, beta, c, w.p, we);
}

}  // namespace

// Deferred mode in the factorization driver: opt-in (RUTV_CHOLQR=2).  The
// three single-CTA 128-column factorizations are still latency-bound
// (~65 us Cholesky, ~62 us LU on B200, tools/time_cqr.py): a panel costs
// ~318 us, about the cluster Householder kernel's 250-360 us (qr_reg.cu), so
// the Householder path stays the default.
bool cholqr_deferred_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RUTV_CHOLQR");
        return e && std::strcmp(e, "2") == 0;
    }();
    return on;
}

void cholqr_set_deferred(int* dflag) { t_deferred_flag = dflag; }

bool cholqr_tall(int64_t s) { return tall_min_rows() > 0 && s >= tall_min_rows(); }

bool qr_panel_fast(cudaStream_t st, const DView& y, double* tau) {
    const int64_t s = y.rows, p = y.cols;
    int* dflag = t_deferred_flag;
    if (!dflag && !immediate_enabled() && !cholqr_tall(s)) return false;
    if (p < 16 || p > 128 || s < 2 * p) return false;
    small_attr();
    const size_t smb = small_smem_bytes(static_cast<int>(p));
    const int64_t pp = p * p;
    DevBuf G(pp, st), R1(pp, st), R1i(pp, st), R2(pp, st), R2i(pp, st), R(pp, st), Ui(pp, st), Q1(s * p, st),
        Qb(s * p, st);
    DevBuf F(1, st), Top(dflag ? 1 : pp, st), Tu(dflag ? 1 : p + 1, st);
    int* flag = dflag;
    if (!flag) {
        flag = reinterpret_cast<int*>(F.p);
        RUTV_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    }
    const DView Gv(p, p, p, G.p), Q1v(s, p, s, Q1.p), Qbv(s, p, s, Qb.p);
    const int pi = static_cast<int>(p);
    // pass 1
    gemm_w(st, 1.0, Op::T, y, Op::N, y, 0.0, Gv);
    cqr_chol_kernel<<<1, kST, smb, st>>>(G.p, p, pi, R1.p, R1i.p, nullptr, nullptr, flag, 1, 1, 0);
    note_launch();
    RUTV_CHECK_LAUNCH();
    gemm_w(st, 1.0, Op::N, y, Op::N, DView(p, p, p, R1i.p), 0.0, Q1v);
    // pass 2 (+ R = R2 R1)
    gemm_w(st, 1.0, Op::T, Q1v, Op::N, Q1v, 0.0, Gv);
    cqr_chol_kernel<<<1, kST, smb, st>>>(G.p, p, pi, R2.p, R2i.p, R1.p, R.p, flag, 4, 0, 1);
    note_launch();
    RUTV_CHECK_LAUNCH();
    gemm_w(st, 1.0, Op::N, Q1v, Op::N, DView(p, p, p, R2i.p), 0.0, Qbv);
    // reconstruction: top block and tau, then V2 = -Q(p:s, :) U^{-1}
    double* topp = dflag ? y.data : Top.p;
    const int64_t ldtop = dflag ? y.ld : p;
    double* taup = dflag ? tau : Tu.p;
    cqr_lu_kernel<<<1, kST, smb, st>>>(Qb.p, s, pi, R.p, topp, ldtop, Ui.p, taup, flag);
    note_launch();
    RUTV_CHECK_LAUNCH();
    if (dflag) {
        gemm_w(st, -1.0, Op::N, Qbv.block(p, 0, s - p, p), Op::N, DView(p, p, p, Ui.p), 0.0,
               y.block(p, 0, s - p, p));
        return true;
    }
    gemm_w(st, -1.0, Op::N, Qbv.block(p, 0, s - p, p), Op::N, DView(p, p, p, Ui.p), 0.0, DView(s - p, p, s, Q1.p));
    int hflag = 1;
    RUTV_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    RUTV_CUDA(cudaStreamSynchronize(st));
    if (hflag != 0) {
        static const bool dbg = std::getenv("RUTV_DEBUG") != nullptr;
        if (dbg)
            std::fprintf(stderr, "[rutv] cholqr fallback s=%lld w=%lld flag=%d\n", static_cast<long long>(s),
                         static_cast<long long>(p), hflag);
        return false;
    }
    commit_kernel<<<static_cast<unsigned>(std::min<int64_t>((s * p + 255) / 256, 4 * kNumSMs)), 256, 0, st>>>(
        s, pi, Top.p, Q1.p, s, y.data, y.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
    RUTV_CUDA(cudaMemcpyAsync(tau, Tu.p, static_cast<size_t>(p) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return true;
}

// T of compact WY for p <= 128 (form_t dispatches here).
void form_t_small(cudaStream_t stream, const double* gram, int64_t ldg, const double* tau, int64_t p, double* t,
                  int64_t ldt) {
    once_per_device(reinterpret_cast<const void*>(form_t_inv_kernel), [] {
        RUTV_CUDA(cudaFuncSetAttribute(form_t_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(small_smem_bytes(128))));
    });
    form_t_inv_kernel<<<1, kST, small_smem_bytes(static_cast<int>(p)), stream>>>(gram, ldg, tau, static_cast<int>(p),
                                                                                   t, ldt);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

}  // namespace rutv

// Test hooks (not part of the public header): the small factorizations alone.
// rutv_b200_debug_chol: G (p x p, ld p) -> R, R^{-1}; returns the flag word.
extern "C" int rutv_b200_debug_chol(const double* g, int p, double* r, double* rinv) {
    rutv::small_attr();
    int* flag = nullptr;
    cudaMalloc(&flag, sizeof(int));
    cudaMemset(flag, 0, sizeof(int));
    rutv::cqr_chol_kernel<<<1, rutv::kST, rutv::small_smem_bytes(p)>>>(g, p, p, r, rinv, nullptr, nullptr, flag, 1, 1,
                                                                       0);
    int h = -1;
    cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(flag);
    return h;
}

// rutv_b200_debug_lu: Q (ldq) -> L1 (strictly lower of the packed top with a
// zero R), U = T V1', U^{-1}, tau; returns the flag word.
extern "C" int rutv_b200_debug_lu(const double* q, int64_t ldq, int p, double* l1, double* u, double* uinv,
                                  double* tau) {
    rutv::small_attr();
    int* flag = nullptr;
    double* zr = nullptr;
    cudaMalloc(&flag, sizeof(int));
    cudaMalloc(&zr, sizeof(double) * p * p);
    cudaMemset(flag, 0, sizeof(int));
    cudaMemset(zr, 0, sizeof(double) * p * p);
    rutv::cqr_lu_kernel<<<1, rutv::kST, rutv::small_smem_bytes(p)>>>(q, ldq, p, zr, l1, p, uinv, tau, flag);
    (void)u;
    int h = -1;
    cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(zr);
    cudaFree(flag);
    return h;
}

extern "C" int rutv_b200_debug_cqr_clocks(long long* out64) {
    return cudaMemcpyFromSymbol(out64, rutv::g_cqr_clk, sizeof(long long) * 128) == cudaSuccess ? 0 : 1;
}
