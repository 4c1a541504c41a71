// cholqr.cu -- panel QR by Cholesky-QR2 + Householder reconstruction.
//
// The reference factors every panel with column-by-column Householder
// (proj/src/householder.cpp:48-67), whose 128 dependent column steps make the
// panel QR latency-bound on the GPU (qr_reg.cu: ~2 us per column).  For a
// full-rank s x w panel Y (w <= 128, s >= 2w) the same factorization is
// obtained from level-3 work plus three small w x w factorizations:
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
// Status: opt-in (RUTV_CHOLQR=1), see enabled() below.
// Safety: the path is taken only when it is numerically sound; otherwise the
// panel is left untouched and the caller runs the Householder kernel:
//   * Cholesky breakdown (pivot <= 0 or not finite) in either pass, or
//     min/max diag(R1) < 1e-7 (Cholesky-QR2 needs cond(Y) well below 1/sqrt(eps));
//   * an LU pivot |tau_j| < 0.25 (a reflector close to the identity: the
//     reconstruction divides by tau_j).
// A flag word is read back on the host (one stream synchronisation per panel).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rutv_common.cuh"

namespace rutv {

constexpr int kCT = 512;

// Register-blocked factorizations of a p x p block (p <= 128) by one CTA of
// 512 threads: thread (tx, ty) = (tid & 31, tid >> 5) owns rows ty + 16 a
// (a < 8) and columns tx + 32 b (b < 4) -- 32 entries in registers; a row
// belongs to one warp, so the pivot-row work is warp-uniform.  A step
// publishes the pivot row / column in shared memory (double-buffered) and
// every thread updates its own entries: two barriers per step, no
// shared-memory traffic for the matrix itself.

// X = R^{-1} for the upper triangular R held in shared memory Rs (column-major,
// leading dimension LD): back substitution from the last row, X in registers.
__device__ __forceinline__ void upper_inverse(const double* Rs, int LD, int p, double (&x)[8][4], double* xrow2,
                                              int tx, int ty) {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) x[a][b] = (ty + 16 * a == tx + 32 * b) ? 1.0 : 0.0;
    for (int i = p - 1; i >= 0; --i) {
        double* xrow = xrow2 + (i & 1) * 128;
        const double rinv = 1.0 / Rs[i + i * LD];
        if (ty == (i & 15)) {  // row i owned by warp i % 16
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int k = tx + 32 * b;
                    const bool hit = (ty + 16 * a == i) && k >= i && k < p;
                    const double v = x[a][b] * rinv;
                    x[a][b] = hit ? v : x[a][b];
                    if (hit) xrow[k] = v;
                }
        }
        __syncthreads();
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int r = ty + 16 * a;
            if (r < i) {
                const double rri = Rs[r + i * LD];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int k = tx + 32 * b;
                    if (k >= i && k < p) x[a][b] -= rri * xrow[k];
                }
            }
        }
        __syncthreads();
    }
}

// Upper Cholesky G = R'R, then R^{-1}.  flag |= 1 (breakdown), 2 (diag ratio < 1e-7).
__global__ void __launch_bounds__(kCT) chol_inv_kernel(const double* __restrict__ g, int64_t ldg, int p, double* r,
                                                       double* rinv, int* flag, int check_ratio) {
    extern __shared__ double Rs[];  // p x LD
    __shared__ double rowb[2][128];
    __shared__ double dpub[2];
    const int LD = p + 1, tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    double a[8][4];
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            a[ai][bi] = (i < p && k < p) ? g[i + static_cast<int64_t>(k) * ldg] : 0.0;
        }
    if (tid == 0) dpub[0] = a[0][0];
    __syncthreads();
    bool bad = false;
    for (int j = 0; j < p; ++j) {
        const int par = j & 1;
        const double d = dpub[par];
        if (!(d > 0.0) || !isfinite(d)) bad = true;
        const double rj = bad ? 1.0 : sqrt(d), inv = 1.0 / rj;
        // row j of R (branch-free over the owned entries: a computed index
        // would move the register array to local memory)
        if (ty == (j & 15)) {  // row j owned by warp j % 16
#pragma unroll
            for (int ai = 0; ai < 8; ++ai)
#pragma unroll
                for (int bi = 0; bi < 4; ++bi) {
                    const int i = ty + 16 * ai, k = tx + 32 * bi;
                    const bool hit = (i == j) && k >= j && k < p;
                    const double v = k == j ? rj : a[ai][bi] * inv;
                    a[ai][bi] = hit ? v : a[ai][bi];
                    if (hit) rowb[par][k] = v;
                }
        }
        __syncthreads();
#pragma unroll
        for (int ai = 0; ai < 8; ++ai) {
            const int i = ty + 16 * ai;
            if (i > j && i < p) {
                const double ri = rowb[par][i];
#pragma unroll
                for (int bi = 0; bi < 4; ++bi) {
                    const int k = tx + 32 * bi;
                    if (k >= i && k < p) a[ai][bi] -= ri * rowb[par][k];
                }
            }
        }
        if (ty == ((j + 1) & 15) && tx == ((j + 1) & 31)) {
#pragma unroll
            for (int ai = 0; ai < 8; ++ai)
#pragma unroll
                for (int bi = 0; bi < 4; ++bi)
                    if (ty + 16 * ai == j + 1 && tx + 32 * bi == j + 1) dpub[par ^ 1] = a[ai][bi];
        }
        __syncthreads();
    }
    // R (upper) to global and shared memory
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            if (i < p && k < p) {
                const double v = i <= k ? a[ai][bi] : 0.0;
                r[i + static_cast<int64_t>(k) * p] = v;
                Rs[i + k * LD] = v;
            }
        }
    __syncthreads();
    if (tid == 0) {
        double mn = INFINITY, mx = 0.0;
        for (int j = 0; j < p; ++j) {
            mn = fmin(mn, Rs[j + j * LD]);
            mx = fmax(mx, Rs[j + j * LD]);
        }
        if (bad) atomicOr(flag, check_ratio ? 1 : 4);
        if (check_ratio && !(mn > 1e-7 * mx)) atomicOr(flag, 2);
    }
    double x[8][4];
    upper_inverse(Rs, LD, p, x, &rowb[0][0], tx, ty);
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            if (i < p && k < p) rinv[i + static_cast<int64_t>(k) * p] = i <= k ? x[ai][bi] : 0.0;
        }
}

// LU without pivoting of B = I - Q(0:p, 0:p): L1 strictly lower, U upper,
// tau = diag(U), then U^{-1}.  |pivot| < 0.25 sets flag bit 8.
__global__ void __launch_bounds__(kCT) lu_inv_kernel(const double* __restrict__ q, int64_t ldq, int p, double* l1,
                                                     double* u, double* uinv, double* tau, int* flag) {
    extern __shared__ double Us[];  // p x LD
    __shared__ double rowb[2][128], colb[2][128];
    __shared__ double dpub[2];
    const int LD = p + 1, tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    double a[8][4];
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            a[ai][bi] = (i < p && k < p) ? (i == k ? 1.0 : 0.0) - q[i + static_cast<int64_t>(k) * ldq] : 0.0;
        }
    if (tid == 0) dpub[0] = a[0][0];
    __syncthreads();
    bool bad = false;
    for (int j = 0; j < p; ++j) {
        const int par = j & 1;
        const double piv = dpub[par];
        if (!(fabs(piv) >= 0.25) || !isfinite(piv)) bad = true;
        const double inv = 1.0 / (bad ? 1.0 : piv);
        // column j: multipliers below the diagonal; row j of U (branch-free)
        if (tx == (j & 31) || ty == (j & 15)) {
#pragma unroll
            for (int ai = 0; ai < 8; ++ai)
#pragma unroll
                for (int bi = 0; bi < 4; ++bi) {
                    const int i = ty + 16 * ai, k = tx + 32 * bi;
                    const bool colhit = (k == j) && i > j && i < p;
                    const double m = a[ai][bi] * inv;
                    a[ai][bi] = colhit ? m : a[ai][bi];
                    if (colhit) colb[par][i] = m;
                    if ((i == j) && k > j && k < p) rowb[par][k] = a[ai][bi];
                }
        }
        __syncthreads();
#pragma unroll
        for (int ai = 0; ai < 8; ++ai) {
            const int i = ty + 16 * ai;
            if (i > j && i < p) {
                const double li = colb[par][i];
#pragma unroll
                for (int bi = 0; bi < 4; ++bi) {
                    const int k = tx + 32 * bi;
                    if (k > j && k < p) a[ai][bi] -= li * rowb[par][k];
                }
            }
        }
        if (ty == ((j + 1) & 15) && tx == ((j + 1) & 31)) {
#pragma unroll
            for (int ai = 0; ai < 8; ++ai)
#pragma unroll
                for (int bi = 0; bi < 4; ++bi)
                    if (ty + 16 * ai == j + 1 && tx + 32 * bi == j + 1) dpub[par ^ 1] = a[ai][bi];
        }
        __syncthreads();
    }
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            if (i < p && k < p) {
                l1[i + static_cast<int64_t>(k) * p] = i > k ? a[ai][bi] : 0.0;
                const double uv = i <= k ? a[ai][bi] : 0.0;
                u[i + static_cast<int64_t>(k) * p] = uv;
                Us[i + k * LD] = uv;
                if (i == k) tau[i] = uv;
            }
        }
    __syncthreads();
    if (tid == 0 && bad) atomicOr(flag, 8);
    double x[8][4];
    upper_inverse(Us, LD, p, x, &rowb[0][0], tx, ty);
#pragma unroll
    for (int ai = 0; ai < 8; ++ai)
#pragma unroll
        for (int bi = 0; bi < 4; ++bi) {
            const int i = ty + 16 * ai, k = tx + 32 * bi;
            if (i < p && k < p) uinv[i + static_cast<int64_t>(k) * p] = i <= k ? x[ai][bi] : 0.0;
        }
}

// Blocked (32-wide) right-looking Cholesky G = R'R of a p x p block (p <= 128)
// in shared memory: per block step the 32 x 32 diagonal block is factored by
// one warp (__syncwarp only), the block row by forward substitution (one
// column per thread, the 32 unknowns in registers) and the trailing block by
// a rank-32 update -- 3 CTA barriers per 32 columns instead of 2 per column.
__global__ void __launch_bounds__(kCT) chol_blocked_kernel(const double* __restrict__ g, int64_t ldg, int p,
                                                           double* r, int64_t ldr, int* flag, int check_ratio) {
    extern __shared__ double A[];
    const int NB = (p + 31) >> 5, P = NB * 32, LD = P + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < P * P; e += kCT) {
        const int i = e % P, k = e / P;
        A[i + k * LD] = (i < p && k < p) ? g[i + static_cast<int64_t>(k) * ldg] : (i == k ? 1.0 : 0.0);
    }
    __syncthreads();
    bool bad = false;
    for (int J = 0; J < NB; ++J) {
        const int j0 = 32 * J;
        if (warp == 0) {  // diagonal block in registers: lane k holds column j0 + k
            double v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = A[(j0 + i) + (j0 + lane) * LD];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const double d = __shfl_sync(0xffffffffu, v[c], c);
                if (!(d > 0.0) || !isfinite(d)) bad = true;
                const double rc = bad ? 1.0 : sqrt(d), inv = 1.0 / rc;
                v[c] = lane == c ? rc : (lane > c ? v[c] * inv : v[c]);  // row c of R
#pragma unroll
                for (int i = c + 1; i < 32; ++i) {
                    const double rci = __shfl_sync(0xffffffffu, v[c], i);  // R(c, i) from lane i
                    if (lane >= i) v[i] -= rci * v[c];
                }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) A[(j0 + i) + (j0 + lane) * LD] = v[i];
        }
        __syncthreads();
        const int k0 = j0 + 32;
        for (int k = k0 + tid; k < P; k += kCT) {  // block row: R_JJ' X = A(J, k)
            double x[32];
            double* ak = A + k * LD + j0;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                double acc = ak[c];
#pragma unroll
                for (int i = 0; i < c; ++i) acc -= A[(j0 + i) + (j0 + c) * LD] * x[i];
                x[c] = acc / A[(j0 + c) + (j0 + c) * LD];
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) ak[c] = x[c];
        }
        __syncthreads();
        const int m = P - k0;
        if (m > 0) {  // trailing: A(i, k) -= sum_c R(c, i) R(c, k), i <= k; warp -> rows, lanes -> columns
            for (int ii = warp; ii < m; ii += kCT / 32) {
                const int i = k0 + ii;
                const double* ri = A + i * LD + j0;
                for (int kk = lane; kk < m; kk += 32) {
                    const int k = k0 + kk;
                    if (k < i) continue;
                    const double* rk = A + k * LD + j0;
                    double acc = 0.0;
#pragma unroll 8
                    for (int c = 0; c < 32; ++c) acc += ri[c] * rk[c];
                    A[i + k * LD] -= acc;
                }
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < p * p; e += kCT) {
        const int i = e % p, k = e / p;
        r[i + static_cast<int64_t>(k) * ldr] = i <= k ? A[i + k * LD] : 0.0;
    }
    if (tid == 0) {
        double mn = INFINITY, mx = 0.0;
        for (int j = 0; j < p; ++j) {
            mn = fmin(mn, A[j + j * LD]);
            mx = fmax(mx, A[j + j * LD]);
        }
        if (bad) atomicOr(flag, check_ratio ? 1 : 4);
        if (check_ratio && !(mn > 1e-7 * mx)) atomicOr(flag, 2);
    }
    __syncthreads();
    if (warp == 0 && bad && lane == 0) atomicOr(flag, check_ratio ? 1 : 4);
}

namespace {

// packed panel: R on and above the diagonal, V1 below it in rows < p, V2 rows >= p
__global__ void commit_kernel(int64_t s, int p, const double* __restrict__ rr, const double* __restrict__ l1,
                              const double* __restrict__ l2, int64_t ldl2, double* a, int64_t lda) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < s * p;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % s, j = e / s;
        double v;
        if (i <= j) v = rr[i + j * p];
        else if (i < p) v = l1[i + j * p];
        else v = l2[(i - p) + j * ldl2];
        a[i + j * lda] = v;
    }
}

// Opt-in (RUTV_CHOLQR=1): correct (tests/test_gpu_cholqr.py) but its three
// single-CTA w x w factorizations are still latency-bound (~150 us each at
// w = 128), so the cluster Householder kernel stays the default.
bool enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RUTV_CHOLQR");
        return e && std::strcmp(e, "1") == 0;
    }();
    return on;
}

void gemm_w(cudaStream_t st, double alpha, Op ta, const DView& a, Op tb, const DView& b, double beta,
            const DView& c) {
    const int64_t k = ta == Op::N ? a.cols : a.rows;
    const int64_t we = gemm_work_elems(c.rows, c.cols, k);
    DevBuf w(we, st);
    gemm(st, alpha, ta, a, tb, b, beta, c, w.p, we);
}

}  // namespace

bool qr_panel_fast(cudaStream_t st, const DView& y, double* tau) {
    const int64_t s = y.rows, p = y.cols;
    if (!enabled() || p < 16 || p > 128 || s < 2 * p) return false;
    static bool attr = false;
    if (!attr) {
        RUTV_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        RUTV_CUDA(cudaFuncSetAttribute(chol_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        RUTV_CUDA(cudaFuncSetAttribute(lu_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr = true;
    }
    const size_t sm = static_cast<size_t>(p) * (p + 1) * sizeof(double);
    const int64_t P32 = (p + 31) / 32 * 32;
    const size_t smb = static_cast<size_t>(P32) * (P32 + 1) * sizeof(double);
    const int64_t pp = p * p;
    DevBuf G(pp, st), R1(pp, st), R1i(pp, st), R2(pp, st), R2i(pp, st), R(pp, st), L1(pp, st), U(pp, st),
        Ui(pp, st), tu(p + 1, st), Q1(s * p, st), Qb(s * p, st), F(1, st);
    int* flag = reinterpret_cast<int*>(F.p);
    RUTV_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    const DView Gv(p, p, p, G.p), Q1v(s, p, s, Q1.p), Qbv(s, p, s, Qb.p);
    // pass 1
    gemm_w(st, 1.0, Op::T, y, Op::N, y, 0.0, Gv);
    chol_blocked_kernel<<<1, kCT, smb, st>>>(G.p, p, static_cast<int>(p), R1.p, p, flag, 1);
    note_launch();
    RUTV_CHECK_LAUNCH();
    tri_inv_upper(st, R1.p, p, p, R1i.p, p);
    gemm_w(st, 1.0, Op::N, y, Op::N, DView(p, p, p, R1i.p), 0.0, Q1v);
    // pass 2
    gemm_w(st, 1.0, Op::T, Q1v, Op::N, Q1v, 0.0, Gv);
    chol_blocked_kernel<<<1, kCT, smb, st>>>(G.p, p, static_cast<int>(p), R2.p, p, flag, 0);
    note_launch();
    RUTV_CHECK_LAUNCH();
    tri_inv_upper(st, R2.p, p, p, R2i.p, p);
    gemm_w(st, 1.0, Op::N, Q1v, Op::N, DView(p, p, p, R2i.p), 0.0, Qbv);
    gemm_w(st, 1.0, Op::N, DView(p, p, p, R2.p), Op::N, DView(p, p, p, R1.p), 0.0, DView(p, p, p, R.p));
    // reconstruction
    lu_inv_kernel<<<1, kCT, sm, st>>>(Qb.p, s, static_cast<int>(p), L1.p, U.p, Ui.p, tu.p, flag);
    note_launch();
    RUTV_CHECK_LAUNCH();
    // V2 = -Q(p:s, :) U^{-1}, into Q1 (rows 0..s-p)
    gemm_w(st, -1.0, Op::N, Qbv.block(p, 0, s - p, p), Op::N, DView(p, p, p, Ui.p), 0.0, DView(s - p, p, s, Q1.p));
    int hflag = 1;
    RUTV_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    RUTV_CUDA(cudaStreamSynchronize(st));
    static const bool force = std::getenv("RUTV_CHOLQR_FORCE") != nullptr;  // debug: commit regardless
    if (force) {
        std::fprintf(stderr, "[rutv] cholqr forced commit, flag was %d\n", hflag);
        hflag = 0;
    }
    if (hflag != 0) {
        static const bool dbg = std::getenv("RUTV_DEBUG") != nullptr;
        if (dbg) std::fprintf(stderr, "[rutv] cholqr fallback s=%lld w=%lld flag=%d\n", static_cast<long long>(s),
                              static_cast<long long>(p), hflag);
        return false;
    }
    commit_kernel<<<static_cast<unsigned>(std::min<int64_t>((s * p + 255) / 256, 4 * kNumSMs)), 256, 0, st>>>(
        s, static_cast<int>(p), R.p, L1.p, Q1.p, s, y.data, y.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
    RUTV_CUDA(cudaMemcpyAsync(tau, tu.p, static_cast<size_t>(p) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return true;
}

}  // namespace rutv

// Test hooks (not part of the public header): the small factorizations alone.
extern "C" int rutv_b200_debug_chol(const double* g, int p, double* r, double* rinv) {
    int* flag = nullptr;
    cudaMalloc(&flag, sizeof(int));
    cudaMemset(flag, 0, sizeof(int));
    cudaFuncSetAttribute(rutv::chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    rutv::chol_inv_kernel<<<1, rutv::kCT, static_cast<size_t>(p) * (p + 1) * 8>>>(g, p, p, r, rinv, flag, 1);
    int h = -1;
    cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(flag);
    return h;
}

extern "C" int rutv_b200_debug_lu(const double* q, int64_t ldq, int p, double* l1, double* u, double* uinv,
                                  double* tau) {
    int* flag = nullptr;
    cudaMalloc(&flag, sizeof(int));
    cudaMemset(flag, 0, sizeof(int));
    cudaFuncSetAttribute(rutv::lu_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    rutv::lu_inv_kernel<<<1, rutv::kCT, static_cast<size_t>(p) * (p + 1) * 8>>>(q, ldq, p, l1, u, uinv, tau, flag);
    int h = -1;
    cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(flag);
    return h;
}
