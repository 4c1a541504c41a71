// aux_kernels.cu -- small memory-bound kernels of the randUTV step.
//
// Each restates a reference helper:
//   make_w          proj/src/householder.cpp:37-44
//   write_rect_diag proj/src/randutv_blocked.cpp:32-37
//   copy_upper      proj/src/randutv_blocked.cpp:73-75 (beta_stage's R)
//   form_t          proj/src/householder.cpp:76-97 (Twy recurrence; the Gram
//                   W'W it needs comes from the DMMA GEMM)
#include <algorithm>

#include <cstdlib>
#include <string>

#include "rutv_common.cuh"

namespace rutv {

namespace {

inline int grid_for(int64_t total) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8 * kNumSMs)));
}

#define RUTV_GRID_STRIDE(i, total)                                                          \
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (total); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void set_identity_kernel(int64_t rows, int64_t cols, double* a, int64_t ld) {
    RUTV_GRID_STRIDE(i, rows * cols) {
        const int64_t r = i % rows, c = i / rows;
        a[r + c * ld] = r == c ? 1.0 : 0.0;
    }
}

__global__ void copy_kernel(int64_t rows, int64_t cols, double* d, int64_t ldd, const double* s,
                            int64_t lds) {
    RUTV_GRID_STRIDE(i, rows * cols) {
        const int64_t r = i % rows, c = i / rows;
        d[r + c * ldd] = s[r + c * lds];
    }
}

__global__ void make_w_kernel(int64_t rows, int64_t p, const double* qr, int64_t ldq, double* w,
                              int64_t ldw) {
    RUTV_GRID_STRIDE(i, rows * p) {
        const int64_t r = i % rows, c = i / rows;
        w[r + c * ldw] = r == c ? 1.0 : (r > c ? qr[r + c * ldq] : 0.0);
    }
}

__global__ void rect_diag_kernel(int64_t rows, int64_t cols, double* a, int64_t ld,
                                 const double* sigma, int64_t p) {
    RUTV_GRID_STRIDE(i, rows * cols) {
        const int64_t r = i % rows, c = i / rows;
        a[r + c * ld] = (r == c && r < p) ? sigma[r] : 0.0;
    }
}

__global__ void copy_upper_kernel(int64_t rows, int64_t cols, double* d, int64_t ldd,
                                  const double* s, int64_t lds) {
    RUTV_GRID_STRIDE(i, rows * cols) {
        const int64_t r = i % rows, c = i / rows;
        d[r + c * ldd] = r <= c ? s[r + c * lds] : 0.0;
    }
}

// Twy (p x p, upper) from the Gram matrix G = W'W and tau, blocked by 32,
// computed IN PLACE over G's strict upper triangle (column j of G is consumed
// exactly when column j of T is produced):
//   diagonal blocks: the reference recurrence T(k,j) = -tau_j sum_{l=k}^{j-1}
//   T(k,l) G(l,j) (householder.cpp:84-95), one warp per block, lane k owning
//   row k, the G column broadcast by warp shuffles;
//   block column J: T(0:J0, J) = -T(0:J0, 0:J0) (G(0:J0, J) T_JJ), the
//   standard two-block composition of compact-WY factors.
// One CTA; the working array lives in shared memory for p <= 128 (one HBM
// read of G, one write of T), else in the output buffer.
__global__ void __launch_bounds__(1024) form_t_kernel(const double* __restrict__ gram, int64_t ldg,
                                                      const double* __restrict__ tau, int p,
                                                      double* t, int64_t ldt, int t_in_smem) {
    extern __shared__ __align__(16) double fsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* M = t_in_smem ? fsm : t;
    const int64_t ld = t_in_smem ? p : ldt;
    double* Xs = fsm + (t_in_smem ? static_cast<size_t>(p) * p : 0);  // up to (p-32) x 32
    const int nblk = (p + 31) / 32;
    for (int64_t i = tid; i < static_cast<int64_t>(p) * p; i += blockDim.x) {
        const int64_t r = i % p, c = i / p;
        M[r + c * ld] = r < c ? gram[r + c * ldg] : 0.0;
    }
    __syncthreads();
    if (warp < nblk) {  // diagonal blocks: lane k owns row I0 + k
        const int I0 = warp * 32, bw = min(32, p - I0);
        double* row = M + (I0 + lane);
        for (int j = 0; j < bw; ++j) {
            const double tj = tau[I0 + j];
            double* colj = M + static_cast<int64_t>(I0 + j) * ld + I0;
            const double zl = lane < j ? colj[lane] : 0.0;  // G(I0+lane, I0+j)
            __syncwarp();
            double s = 0.0;
            for (int l = 0; l < j; ++l) {
                const double z = __shfl_sync(0xffffffffu, zl, l);
                if (l >= lane) s += row[static_cast<int64_t>(I0 + l) * ld] * z;
            }
            if (lane < j) colj[lane] = -tj * s;
            else if (lane == j) colj[lane] = tj;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int J = 1; J < nblk; ++J) {  // off-diagonal block columns
        const int J0 = J * 32, bw = min(32, p - J0);
        const int cnt = J0 * bw;
        for (int e = tid; e < cnt; e += blockDim.x) {  // X = G(0:J0, J) T_JJ
            const int r = e % J0, c = e / J0;
            double s = 0.0;
            for (int l = 0; l <= c; ++l)
                s += M[r + static_cast<int64_t>(J0 + l) * ld] * M[(J0 + l) + static_cast<int64_t>(J0 + c) * ld];
            Xs[r + static_cast<size_t>(c) * J0] = s;
        }
        __syncthreads();
        for (int e = tid; e < cnt; e += blockDim.x) {  // T(0:J0, J) = -T(0:J0, 0:J0) X
            const int r = e % J0, c = e / J0;
            double s = 0.0;
            for (int m = r; m < J0; ++m) s += M[r + static_cast<int64_t>(m) * ld] * Xs[m + static_cast<size_t>(c) * J0];
            M[r + static_cast<int64_t>(J0 + c) * ld] = -s;
        }
        __syncthreads();
    }
    if (t_in_smem)
        for (int64_t i = tid; i < static_cast<int64_t>(p) * p; i += blockDim.x) {
            const int64_t r = i % p, c = i / p;
            t[r + c * ldt] = M[r + c * p];
        }
}


// Twy by recursive doubling (p <= 256): the 16 x 16 diagonal blocks by the
// reference recurrence (householder.cpp:84-95; one warp each, lane r holding
// row r in registers), then block columns combined pairwise with doubling
// width h = 16, 32, 64, ...:  T(I, J) = -T(I, I) (G(I, J) T(J, J)) -- the
// compact-WY composition of two adjacent reflector blocks.  Every level is
// two small triangular-times-dense products, 4 x 4 register tiles per thread.
// M (G's strict upper triangle, overwritten by T) lives in shared memory for
// p <= 128, else in the output buffer (L2-resident); the per-level scratch X
// is in shared memory.
constexpr int kFtThreads = 512;

// mode 1: the same recursive doubling computes the inverse X of an upper
// triangular R (input `gram` = R, diagonal included): diagonal blocks by back
// substitution (the recurrence with tau_c -> 1 / R(c, c)), off-diagonal blocks
// X(I, J) = -X(I, I) R(I, J) X(J, J).
__global__ void __launch_bounds__(kFtThreads) form_t_rd_kernel(const double* __restrict__ gram, int64_t ldg,
                                                               const double* __restrict__ tau, int p, double* t,
                                                               int64_t ldt, int m_in_smem, int mode) {
    extern __shared__ __align__(16) double fsm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t LDm = m_in_smem ? p + 1 : ldt;
    double* M = m_in_smem ? fsm : t;
    double* X = fsm + (m_in_smem ? static_cast<size_t>(p) * (p + 1) : 0);
    if (m_in_smem) {  // asynchronous copies: every load in flight at once
        for (int i = tid; i < p * p; i += kFtThreads) {
            const int r = i % p, c = i / p;
            double* dst = M + r + c * LDm;
            if (r < c || (mode == 1 && r == c)) {
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gram + r + c * ldg));
            } else {
                *dst = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    } else {  // staged: 8 loads in flight per thread
        for (int i0 = tid; i0 < p * p; i0 += 8 * kFtThreads) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kFtThreads, r = i % p, c = i / p;
                v[u] = (i < p * p && (r < c || (mode == 1 && r == c))) ? gram[r + c * ldg] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kFtThreads;
                if (i < p * p) M[i % p + (i / p) * LDm] = v[u];
            }
        }
    }
    __syncthreads();
    const int nb = (p + 15) >> 4;
    for (int blk = warp; blk < nb; blk += kFtThreads / 32) {
        const int I0 = blk * 16, bw = min(16, p - I0);
        double trow[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const double tc = c >= bw ? 0.0 : (mode == 1 ? 1.0 / M[(I0 + c) + (I0 + c) * LDm] : tau[I0 + c]);
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int q = 0; q < c; ++q) {
                const double gq = c < bw ? M[(I0 + q) + (I0 + c) * LDm] : 0.0;
                if (q & 1) a1 += trow[q] * gq; else a0 += trow[q] * gq;
            }
            trow[c] = lane < c ? -tc * (a0 + a1) : (lane == c ? tc : 0.0);
        }
        __syncwarp();
        if (lane < bw)
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < bw) M[(I0 + lane) + (I0 + c) * LDm] = trow[c];
        __syncwarp();
    }
    __syncthreads();
    for (int h = 16; h < p; h *= 2) {
        const int npair = (p + 2 * h - 1) / (2 * h);
        const int tr = h >> 2;  // 4-row tiles per block
        // X_pair = G(I, J) T(J, J), X_pair stored h x h at X + pair * h * h (column-major)
        for (int e = tid; e < npair * tr * tr; e += kFtThreads) {
            const int pr = e / (tr * tr), rem = e - pr * tr * tr;
            const int ti = rem % tr, tj = rem / tr;
            const int I0 = pr * 2 * h, J0 = I0 + h;
            if (J0 >= p) continue;
            const int hJ = min(h, p - J0);
            const int r0 = ti, c0 = 4 * tj;  // rows ti + tr*i: lanes read consecutive rows
            if (c0 >= hJ) continue;
            double acc[4][4] = {};
            const int lend = min(hJ, c0 + 4);
#pragma unroll 4
            for (int l = 0; l < lend; ++l) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = M[(I0 + r0 + tr * i) + (J0 + l) * LDm];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) b[jj] = c0 + jj < hJ ? M[(J0 + l) + (J0 + c0 + jj) * LDm] : 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) acc[i][jj] += a[i] * b[jj];
            }
            double* Xp = X + static_cast<size_t>(pr) * h * h;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) Xp[(r0 + tr * i) + (c0 + jj) * h] = acc[i][jj];
        }
        __syncthreads();
        // T(I, J) = -T(I, I) X_pair, T(I, I) upper triangular
        for (int e = tid; e < npair * tr * tr; e += kFtThreads) {
            const int pr = e / (tr * tr), rem = e - pr * tr * tr;
            const int ti = rem % tr, tj = rem / tr;
            const int I0 = pr * 2 * h, J0 = I0 + h;
            if (J0 >= p) continue;
            const int hJ = min(h, p - J0);
            const int r0 = ti, c0 = 4 * tj;  // rows ti + tr*i (T(I,I) is zero left of each row's diagonal)
            if (c0 >= hJ) continue;
            const double* Xp = X + static_cast<size_t>(pr) * h * h;
            double acc[4][4] = {};
#pragma unroll 4
            for (int m = r0; m < h; ++m) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = M[(I0 + r0 + tr * i) + (I0 + m) * LDm];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) b[jj] = Xp[m + (c0 + jj) * h];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) acc[i][jj] += a[i] * b[jj];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (c0 + jj < hJ) M[(I0 + r0 + tr * i) + (J0 + c0 + jj) * LDm] = -acc[i][jj];
        }
        __syncthreads();
    }
    if (m_in_smem)
        for (int i = tid; i < p * p; i += kFtThreads) {
            const int r = i % p, c = i / p;
            t[r + c * ldt] = M[r + c * LDm];
        }
}

}  // namespace

void set_identity(cudaStream_t stream, const DView& a) {
    if (a.rows * a.cols == 0) return;
    set_identity_kernel<<<grid_for(a.rows * a.cols), 256, 0, stream>>>(a.rows, a.cols, a.data, a.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void copy_view(cudaStream_t stream, const DView& dst, const DView& src) {
    if (dst.rows != src.rows || dst.cols != src.cols)
        throw Error(RUTV_ERR_SHAPE, "copy_view shape mismatch");
    if (dst.rows * dst.cols == 0) return;
    copy_kernel<<<grid_for(dst.rows * dst.cols), 256, 0, stream>>>(dst.rows, dst.cols, dst.data,
                                                                    dst.ld, src.data, src.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void make_w(cudaStream_t stream, const DView& qr, int64_t p, const DView& w) {
    if (qr.rows * p == 0) return;
    make_w_kernel<<<grid_for(qr.rows * p), 256, 0, stream>>>(qr.rows, p, qr.data, qr.ld, w.data, w.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void write_rect_diag(cudaStream_t stream, const DView& block, const double* sigma, int64_t p) {
    if (block.rows * block.cols == 0) return;
    rect_diag_kernel<<<grid_for(block.rows * block.cols), 256, 0, stream>>>(
        block.rows, block.cols, block.data, block.ld, sigma, p);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void copy_upper(cudaStream_t stream, const DView& dst, const DView& src) {
    if (dst.rows * dst.cols == 0) return;
    copy_upper_kernel<<<grid_for(dst.rows * dst.cols), 256, 0, stream>>>(
        dst.rows, dst.cols, dst.data, dst.ld, src.data, src.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void form_t(cudaStream_t stream, const double* gram, int64_t ldg, const double* tau, int64_t p,
            double* t, int64_t ldt) {
    if (p == 0) return;
    if (p > 1024) throw Error(RUTV_ERR_NOTIMPL, "form_t: block size above 1024");
    static const bool rd_only = [] {  // RUTV_FORMT=rd: recursive doubling for every p <= 256 (A/B knob)
        const char* e = std::getenv("RUTV_FORMT");
        return e && std::string(e) == "rd";
    }();
    if (p <= 128 && !rd_only) {
        form_t_small(stream, gram, ldg, tau, p, t, ldt);
        return;
    }
    // p > 128: 128-column diagonal blocks by the blocked inversion (form_t_small), block column J
    // by the two-block composition of compact-WY factors on the DMMA GEMM,
    //     T(0:j0, J) = -T(0:j0, 0:j0) (G(0:j0, J) T_JJ)
    // (the reference recurrence householder.cpp:84-95 a block at a time).  X' = T_JJ' G(0:j0, J)'
    // is staged in T's own block below the diagonal, which is zeroed afterwards.  The single-CTA
    // kernels below (RUTV_FORMT=legacy) take 5.1 ms at p = 512 -- on the critical chain of every
    // late step, 2.3 % of config 5's kernel time (profiles/r02_launches_c5_full_b.json).
    static const bool legacy = [] {
        const char* e = std::getenv("RUTV_FORMT");
        return e && std::string(e) == "legacy";
    }();
    if (!rd_only && !legacy && t != gram) {
        const int64_t nbk = 128;
        for (int64_t j0 = 0; j0 < p; j0 += nbk) {
            const int64_t jb = std::min(nbk, p - j0);
            double* tjj = t + j0 + j0 * ldt;
            form_t_small(stream, gram + j0 + j0 * ldg, ldg, tau + j0, jb, tjj, ldt);
            if (j0 == 0) continue;
            const DView Tjj(jb, jb, ldt, tjj), Gj(j0, jb, ldg, const_cast<double*>(gram) + j0 * ldg);
            const DView Xt(jb, j0, ldt, t + j0), T11(j0, j0, ldt, t), Tj(j0, jb, ldt, t + j0 * ldt);
            gemm(stream, 1.0, Op::T, Tjj, Op::T, Gj, 0.0, Xt, nullptr, 0);
            gemm(stream, -1.0, Op::N, T11, Op::T, Xt, 0.0, Tj, nullptr, 0);
            RUTV_CUDA(cudaMemset2DAsync(t + j0, static_cast<size_t>(ldt) * sizeof(double), 0,
                                        static_cast<size_t>(jb) * sizeof(double), static_cast<size_t>(j0), stream));
        }
        return;
    }
    if (p <= 256) {
        static int rcap = 0;
        once_per_device(reinterpret_cast<const void*>(form_t_rd_kernel), [] {
            rcap = dyn_smem_cap(reinterpret_cast<const void*>(form_t_rd_kernel));
            RUTV_CUDA(cudaFuncSetAttribute(form_t_rd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rcap));
        });
        // scratch X: npair h x h blocks per level
        int64_t xe = 1;
        for (int64_t h = 16; h < p; h *= 2) xe = std::max(xe, (p + 2 * h - 1) / (2 * h) * h * h);
        const size_t xs = static_cast<size_t>(xe) * sizeof(double);
        const size_t msz = static_cast<size_t>(p) * (p + 1) * sizeof(double);
        const bool in_smem = msz + xs <= static_cast<size_t>(rcap);
        form_t_rd_kernel<<<1, kFtThreads, in_smem ? msz + xs : xs, stream>>>(gram, ldg, tau, static_cast<int>(p), t,
                                                                          ldt, in_smem ? 1 : 0, 0);
        note_launch();
        RUTV_CHECK_LAUNCH();
        return;
    }
    static int cap = 0;
    once_per_device(reinterpret_cast<const void*>(form_t_kernel), [] {
        cap = dyn_smem_cap(reinterpret_cast<const void*>(form_t_kernel));
        RUTV_CUDA(cudaFuncSetAttribute(form_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    });
    const size_t xs = static_cast<size_t>(std::max<int64_t>(p - 32, 1)) * 32 * sizeof(double);
    const size_t tsm = static_cast<size_t>(p) * p * sizeof(double);
    const bool in_smem = tsm + xs <= static_cast<size_t>(cap);
    if (!in_smem && xs > static_cast<size_t>(cap)) throw Error(RUTV_ERR_NOTIMPL, "form_t: block too large");
    form_t_kernel<<<1, 1024, in_smem ? tsm + xs : xs, stream>>>(gram, ldg, tau, static_cast<int>(p), t, ldt,
                                                                in_smem ? 1 : 0);
    note_launch();
    RUTV_CHECK_LAUNCH();
}


}  // namespace rutv
