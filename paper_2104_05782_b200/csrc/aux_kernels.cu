// aux_kernels.cu -- small memory-bound kernels of the randUTV step.
//
// Each restates a reference helper:
//   make_w          proj/src/householder.cpp:37-44
//   write_rect_diag proj/src/randutv_blocked.cpp:32-37
//   copy_upper      proj/src/randutv_blocked.cpp:73-75 (beta_stage's R)
//   form_t          proj/src/householder.cpp:76-97 (Twy recurrence; the Gram
//                   W'W it needs comes from the DMMA GEMM)
#include <algorithm>

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

// Twy (p x p, upper) from z-vectors = strictly-upper Gram W'W and tau.
// One CTA; thread k owns row k of T.  For column j: T(j,j) = tau_j and
// T(k,j) = -tau_j * sum_{l=k}^{j-1} T(k,l) * G(l,j) for k < j.  T(k,l) for
// fixed l is contiguous in k, so the l-outer loop reads T coalesced.
__global__ void __launch_bounds__(1024) form_t_kernel(const double* gram, int64_t ldg,
                                                      const double* tau, int p, double* t,
                                                      int64_t ldt) {
    extern __shared__ double zs[];  // p
    const int k = threadIdx.x;
    for (int64_t i = threadIdx.x; i < static_cast<int64_t>(p) * p; i += blockDim.x) {
        const int64_t r = i % p, c = i / p;
        if (r > c) t[r + c * ldt] = 0.0;
    }
    for (int j = 0; j < p; ++j) {
        for (int l = threadIdx.x; l < j; l += blockDim.x) zs[l] = gram[l + static_cast<int64_t>(j) * ldg];
        __syncthreads();
        const double tj = tau[j];
        if (k < j) {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int l = k;
            for (; l + 3 < j; l += 4) {
                s0 += t[k + static_cast<int64_t>(l) * ldt] * zs[l];
                s1 += t[k + static_cast<int64_t>(l + 1) * ldt] * zs[l + 1];
                s2 += t[k + static_cast<int64_t>(l + 2) * ldt] * zs[l + 2];
                s3 += t[k + static_cast<int64_t>(l + 3) * ldt] * zs[l + 3];
            }
            for (; l < j; ++l) s0 += t[k + static_cast<int64_t>(l) * ldt] * zs[l];
            t[k + static_cast<int64_t>(j) * ldt] = -tj * ((s0 + s1) + (s2 + s3));
        }
        if (k == j) t[k + static_cast<int64_t>(j) * ldt] = tj;
        __syncthreads();
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
    const int threads = static_cast<int>(std::max<int64_t>(32, (p + 31) / 32 * 32));
    form_t_kernel<<<1, threads, static_cast<size_t>(p) * sizeof(double), stream>>>(
        gram, ldg, tau, static_cast<int>(p), t, ldt);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

}  // namespace rutv
