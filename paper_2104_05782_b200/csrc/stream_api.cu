// stream_api.cu -- asynchronous C-ABI building blocks (no host synchronisation).
//
// The distributed driver (paper_2104_05782_b200/dist.py)
// composes a step of the reference loop (randutv_blocked.cpp:122-155) from
// these entry points plus NCCL collectives.  Every call enqueues on the
// thread's current stream (rutv_b200_set_stream) and returns immediately;
// scratch comes from the stream-ordered pool.  All pointers are DEVICE
// pointers, matrices column-major.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "rutv_common.cuh"

namespace {

thread_local cudaStream_t t_stream = nullptr;

int fill(rutv_status* st, int code, const char* msg, double residual = 0.0) {
    if (st) {
        st->code = code;
        st->reserved = 0;
        st->residual = residual;
        std::snprintf(st->message, sizeof st->message, "%s", msg ? msg : "");
    }
    return code;
}

template <class F>
int guarded(rutv_status* st, F&& f) {
    try {
        f();
        return fill(st, RUTV_OK, "");
    } catch (const rutv::Error& e) {
        return fill(st, e.code, e.what(), e.residual);
    } catch (const std::exception& e) {
        return fill(st, RUTV_ERR_INTERNAL, e.what());
    } catch (...) {
        return fill(st, RUTV_ERR_INTERNAL, "unknown failure");
    }
}

struct Scratch {
    double* p = nullptr;
    cudaStream_t s;
    Scratch(int64_t elems, cudaStream_t st) : s(st) {
        if (elems < 1) elems = 1;
        p = static_cast<double*>(rutv::dev_alloc(static_cast<size_t>(elems) * 8, st));
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

// dst rows [t*b, t*b + w_t) <- src rows [(first + t*stride)*b, ...), t < count
// (scatter = the inverse).  w_t = min(b, src_rows - row_start).
__global__ void block_rows_kernel(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t cols,
                                  int64_t b, int64_t first, int64_t stride, int64_t count, int64_t big_rows,
                                  int scatter) {
    const int64_t rows_small = count * b;
    const int64_t total = rows_small * cols;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t rs = e % rows_small, c = e / rows_small;
        const int64_t t = rs / b, o = rs - t * b;
        const int64_t rb = (first + t * stride) * b + o;
        if (rb >= big_rows) continue;
        if (scatter)
            const_cast<double*>(src)[rb + c * lds] = dst[rs + c * ldd];
        else
            dst[rs + c * ldd] = src[rb + c * lds];
    }
}

}  // namespace

namespace rutv {
void block_rows(cudaStream_t st, double* small, int64_t lds_small, double* big, int64_t ld_big, int64_t big_rows,
                int64_t cols, int64_t b, int64_t first, int64_t stride, int64_t count, bool scatter) {
    const int64_t total = count * b * cols;
    if (total <= 0) return;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs));
    block_rows_kernel<<<blocks, 256, 0, st>>>(small, lds_small, big, ld_big, cols, b, first, stride, count, big_rows,
                                              scatter ? 1 : 0);
    note_launch();
    RUTV_CHECK_LAUNCH();
}
}  // namespace rutv

extern "C" {

void rutv_b200_set_stream(uint64_t stream) { t_stream = reinterpret_cast<cudaStream_t>(stream); }

// Compact-WY pieces of a packed QR (s x p, householder.cpp:37-44, 76-97):
// W (s x p, unit lower trapezoidal), Twy (p x p), M = W Twy' (s x p).
int rutv_b200_form_wy(const double* qr, int64_t s, int64_t ldq, const double* tau, int64_t p, double* W,
                      int64_t ldw, double* M, int64_t ldm, double* twy, int64_t ldt, rutv_status* st) {
    return guarded(st, [&] {
        using rutv::DView;
        using rutv::Op;
        const cudaStream_t cs = t_stream;
        const int64_t we = std::max<int64_t>({rutv::gemm_work_elems(p, p, s), rutv::gemm_work_elems(s, p, p), 1});
        Scratch gram(p * p, cs), gw(we, cs);
        DView Wv(s, p, ldw, W), Mv(s, p, ldm, M);
        rutv::make_w(cs, DView(s, p, ldq, const_cast<double*>(qr)), p, Wv);
        rutv::gemm(cs, 1.0, Op::T, Wv, Op::N, Wv, 0.0, DView(p, p, p, gram.p), gw.p, we);
        rutv::form_t(cs, gram.p, p, tau, p, twy, ldt);
        rutv::gemm(cs, 1.0, Op::N, Wv, Op::T, DView(p, p, ldt, twy), 0.0, Mv, gw.p, we);
    });
}

int rutv_b200_gemm_async(double alpha, int ta, const double* A, int64_t ar, int64_t ac, int64_t lda, int tb,
                         const double* B, int64_t br, int64_t bc, int64_t ldb, double beta, double* C, int64_t m,
                         int64_t n, int64_t ldc, rutv_status* st) {
    return guarded(st, [&] {
        using rutv::DView;
        const int64_t k = ta ? ar : ac;
        const int64_t we = rutv::gemm_work_elems(m, n, k);
        Scratch w(we, t_stream);
        rutv::gemm(t_stream, alpha, ta ? rutv::Op::T : rutv::Op::N, DView(ar, ac, lda, const_cast<double*>(A)),
                   tb ? rutv::Op::T : rutv::Op::N, DView(br, bc, ldb, const_cast<double*>(B)), beta,
                   DView(m, n, ldc, C), w.p, we);
    });
}

int rutv_b200_hqr_async(double* A, int64_t m, int64_t n, int64_t lda, double* tau, rutv_status* st) {
    return guarded(st, [&] {
        const int64_t we = rutv::hqr_work_elems(m, n);
        Scratch w(we, t_stream);
        rutv::hqr_panel(t_stream, rutv::DView(m, n, lda, A), tau, nullptr, 0, w.p, we);
    });
}

int rutv_b200_normal_fill_async(uint64_t seed, uint64_t pos, double* G, int64_t rows, int64_t cols, int64_t ldg,
                                rutv_status* st) {
    return guarded(st, [&] { rutv::normal_fill(t_stream, seed, pos, rutv::DView(rows, cols, ldg, G)); });
}

int rutv_b200_copy_async(double* dst, int64_t rows, int64_t cols, int64_t ldd, const double* src, int64_t lds,
                         rutv_status* st) {
    return guarded(st, [&] {
        rutv::copy_view(t_stream, rutv::DView(rows, cols, ldd, dst), rutv::DView(rows, cols, lds, const_cast<double*>(src)));
    });
}

int rutv_b200_copy_upper_async(double* dst, int64_t rows, int64_t cols, int64_t ldd, const double* src, int64_t lds,
                               rutv_status* st) {
    return guarded(st, [&] {
        rutv::copy_upper(t_stream, rutv::DView(rows, cols, ldd, dst), rutv::DView(rows, cols, lds, const_cast<double*>(src)));
    });
}

int rutv_b200_identity_async(double* a, int64_t rows, int64_t cols, int64_t lda, rutv_status* st) {
    return guarded(st, [&] { rutv::set_identity(t_stream, rutv::DView(rows, cols, lda, a)); });
}

int rutv_b200_rect_diag_async(double* block, int64_t rows, int64_t cols, int64_t ld, const double* sigma, int64_t p,
                              rutv_status* st) {
    return guarded(st, [&] { rutv::write_rect_diag(t_stream, rutv::DView(rows, cols, ld, block), sigma, p); });
}

// Row-block gather (scatter != 0: scatter back) for block-cyclic layouts.
int rutv_b200_block_rows_async(double* small, int64_t lds_small, double* big, int64_t ld_big, int64_t big_rows,
                               int64_t cols, int64_t b, int64_t first, int64_t stride, int64_t count, int scatter,
                               rutv_status* st) {
    return guarded(st, [&] {
        const int64_t total = count * b * cols;
        if (total <= 0) return;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * rutv::kNumSMs));
        block_rows_kernel<<<blocks, 256, 0, t_stream>>>(small, lds_small, big, ld_big, cols, b, first, stride, count,
                                                        big_rows, scatter);
        rutv::note_launch();
        RUTV_CHECK_LAUNCH();
    });
}

// Batched one-sided Jacobi over `count` square problems (host arrays of device
// pointers).  status: device array of 4*count doubles (code, residual, kept,
// sweeps), read by the caller after synchronising.
int rutv_b200_svd_batch_async(int count, const int64_t* n, double* const* A, const int64_t* lda, double* const* U,
                              double* const* sigma, double* const* V, double* status, rutv_status* st) {
    return guarded(st, [&] {
        if (count <= 0) return;
        const cudaStream_t cs = t_stream;
        int64_t nmax = 0, wtot = 0;
        for (int i = 0; i < count; ++i) {
            nmax = std::max(nmax, n[i]);
            wtot += rutv::svd_work_elems(n[i], 30);
        }
        Scratch work(wtot, cs);
        const int64_t dwords = (static_cast<int64_t>(sizeof(rutv::SvdDesc)) * count + 7) / 8;
        Scratch dd(dwords, cs);
        std::vector<rutv::SvdDesc> h(static_cast<size_t>(count));
        int64_t off = 0;
        for (int i = 0; i < count; ++i) {
            h[static_cast<size_t>(i)] = rutv::SvdDesc{A[i], lda[i], static_cast<int>(n[i]), 0, U[i], sigma[i], V[i],
                                                      work.p + off, status + 4 * i};
            off += rutv::svd_work_elems(n[i], 30);
        }
        RUTV_CUDA(cudaMemsetAsync(status, 0, static_cast<size_t>(count) * 32, cs));
        RUTV_CUDA(cudaMemcpyAsync(dd.p, h.data(), sizeof(rutv::SvdDesc) * h.size(), cudaMemcpyHostToDevice, cs));
        rutv::svd_batch(cs, reinterpret_cast<const rutv::SvdDesc*>(dd.p), count, static_cast<int>(nmax), 1e-15, 30);
    });
}

}  // extern "C"
