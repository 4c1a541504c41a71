// capi.cu -- the C-ABI boundary (include/rutv_b200.h).
//
// Every entry point: validate like the reference (ConfigError / ShapeError
// semantics of randutv_blocked.cpp:10-14, gemm.cpp:11-17), run on the device,
// map rutv::Error (and CUDA failures) to the status struct.  No exception
// crosses the C boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "rutv_common.cuh"


using rutv::DView;
using rutv::Error;
using rutv::Op;

namespace {

int fill(rutv_status* st, int code, const char* msg, double residual = 0.0) {
    if (st) {
        st->code = code;
        st->reserved = 0;
        st->residual = residual;
        std::snprintf(st->message, sizeof st->message, "%s", msg ? msg : "");
    }
    return code;
}

// Every public call ends by returning the library pool's freed blocks to the
// driver (beyond a bounded cache): no device memory stays held after a call.
struct TrimAtExit {
    ~TrimAtExit() { rutv::pool_trim(); }
};

template <class F>
int guarded(rutv_status* st, F&& f) {
    TrimAtExit trim;
    try {
        f();
        return fill(st, RUTV_OK, "");
    } catch (const Error& e) {
        return fill(st, e.code, e.what(), e.residual);
    } catch (const std::bad_alloc&) {
        return fill(st, RUTV_ERR_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fill(st, RUTV_ERR_INTERNAL, e.what());
    } catch (...) {
        return fill(st, RUTV_ERR_INTERNAL, "unknown failure");
    }
}

void set_device(int device) {
    RUTV_CUDA(cudaSetDevice(device));
}

void check_opts(const rutv_opts* o) {
    if (!o) throw Error(RUTV_ERR_CONFIG, "null options");
    if (o->b < 1) throw Error(RUTV_ERR_CONFIG, "block size must be >= 1, got " + std::to_string(o->b));
    if (o->q < 0)
        throw Error(RUTV_ERR_CONFIG, "power iteration count must be >= 0, got " + std::to_string(o->q));
}

struct Stream {
    cudaStream_t s = nullptr;
    bool owned = true;
    Stream() { RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    // Caller-provided stream (rutv_opts::stream) when non-zero.
    explicit Stream(uint64_t handle) {
        if (handle) {
            s = reinterpret_cast<cudaStream_t>(handle);
            owned = false;
        } else {
            RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        }
    }
    ~Stream() {
        if (s && owned) cudaStreamDestroy(s);
    }
};

template <class T>
struct DMem {
    T* p = nullptr;
    cudaStream_t st;
    DMem(size_t count, cudaStream_t s) : st(s) {
        if (count == 0) count = 1;
        p = static_cast<T*>(rutv::dev_alloc(count * sizeof(T), s));
    }
    ~DMem() {
        if (p) cudaFreeAsync(p, st);
    }
};

// Deviates the first max_steps loop iterations draw (all of them when max_steps < 0):
// sum over full steps of rows_rem * b (randutv_blocked.cpp:41-44, 122-139).
int64_t drawn_length(int64_t m, int64_t n, int64_t b, int max_steps) {
    int64_t total = 0;
    for (int64_t i = 0; max_steps < 0 || i < max_steps; ++i) {
        const int64_t r0 = i * b, rr = m - r0, cr = n - r0;
        if (rr <= 0 || cr <= 0 || cr <= b) break;
        total += rr * b;
    }
    return total;
}

void run_factorize(const rutv_opts* o, const double* dA, int64_t m, int64_t n, int64_t lda,
                   const double* dG, int64_t g_len, double* dT, int64_t ldt, double* dU, int64_t ldu,
                   double* dV, int64_t ldv, cudaStream_t st) {
    check_opts(o);
    const bool prepass = o->qr_prepass && m > n;
    if (lda < std::max<int64_t>(m, 1) || ldt < std::max<int64_t>(m, 1))
        throw Error(RUTV_ERR_SHAPE, "leading dimension smaller than the row count");
    if (o->build_u && (!dU || ldu < std::max<int64_t>(m, 1))) throw Error(RUTV_ERR_SHAPE, "U buffer");
    if (o->build_v && (!dV || ldv < std::max<int64_t>(n, 1))) throw Error(RUTV_ERR_SHAPE, "V buffer");
    // qr_prepass factors the n x n R with the same seed (randutv_blocked.cpp:88-96)
    if (dG && g_len < drawn_length(prepass ? n : m, n, o->b, o->max_steps))
        throw Error(RUTV_ERR_SHAPE, "explicit G shorter than the stream the factorization draws");
    rutv::FactorArgs fa{o->b,  o->q, o->build_u != 0, o->build_v != 0, o->seed, o->max_steps, dA, lda,
                        dG,    dT,   ldt,             dU,             ldu,     dV,          ldv,
                        o->overlap != 0};
    if (prepass)
        rutv::factorize_prepass_device(st, o->device, m, n, fa);
    else if (m != n)
        rutv::factorize_rect_device(st, o->device, m, n, fa);
    else
        rutv::factorize_device(st, o->device, n, fa);
}

}  // namespace

extern "C" {

void rutv_b200_default_opts(rutv_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->b = 128;
    o->q = 1;
    o->build_u = 1;
    o->build_v = 1;
    o->seed = 0;
    o->device = 0;
    o->max_steps = -1;
    o->overlap = 1;
    o->grid_p = 1;
    o->grid_q = 1;
}

int64_t rutv_b200_stream_length(int64_t m, int64_t n, int64_t b) {
    if (b < 1) return 0;
    int64_t total = 0;
    for (int64_t i = 0;; ++i) {
        const int64_t r0 = i * b, rr = m - r0, cr = n - r0;
        if (rr <= 0 || cr <= 0 || cr <= b) break;
        total += rr * b;
    }
    return total;
}

double rutv_b200_flops(int64_t n, int64_t b, int32_t q) {
    double f = 0.0;
    if (b < 1) return 0.0;
    for (int64_t i = 0;; ++i) {
        const double r0 = static_cast<double>(i * b), s = static_cast<double>(n - i * b);
        const double bb = static_cast<double>(b), nn = static_cast<double>(n);
        if (s <= 0) break;
        if (s <= bb) {
            f += 2 * r0 * s * s + 4 * nn * s * s;
            break;
        }
        f += 2 * s * s * bb * (1 + 2 * q);                          // sketch + power
        f += 4 * s * s * bb + 2 * s * bb * bb;                      // V-apply on T22
        f += 4 * r0 * s * bb + 2 * r0 * bb * bb;                    // V-apply on T-above
        f += 4 * nn * s * bb + 2 * nn * bb * bb;                    // V-apply on V
        f += 4 * s * bb * (s - bb) + 2 * bb * bb * (s - bb);        // Qu' on T22(:, b:)
        f += 4 * nn * s * bb + 2 * nn * bb * bb;                    // U accumulate
        f += 2 * bb * bb * (s - bb) + 2 * r0 * bb * bb + 4 * nn * bb * bb;  // beta strip, Vs/Us
        f += 4 * bb * bb * (s - bb / 3);                            // two Householder QRs
    }
    return f;
}

int rutv_b200_factorize(const rutv_opts* o, const double* A, int64_t m, int64_t n, int64_t lda,
                        const double* G, int64_t g_len, double* T, int64_t ldt, double* U,
                        int64_t ldu, double* V, int64_t ldv, rutv_status* st) {
    return guarded(st, [&] {
        check_opts(o);
        set_device(o->device);
        rutv::pool_keep_this_call(o->keep_workspace != 0);
        Stream s(o->stream);
        const int64_t mm = std::max<int64_t>(m, 0), nn = std::max<int64_t>(n, 0);
        const bool prepass = o->qr_prepass && m > n;  // the inner n x n run draws the stream
        const int64_t glen = G ? drawn_length(prepass ? n : m, n, o->b, o->max_steps) : 0;
        if (G && glen > 0 && g_len < glen) throw Error(RUTV_ERR_SHAPE, "explicit G shorter than the stream");
        if (std::max(o->grid_p, 1) * std::max(o->grid_q, 1) > 1) {  // sharded over a P x Q grid (dist.cu)
            if (m != n || prepass) throw Error(RUTV_ERR_NOTIMPL, "the sharded path factors square matrices");
            if (o->build_u && (!U || ldu < std::max<int64_t>(m, 1))) throw Error(RUTV_ERR_SHAPE, "U buffer");
            if (o->build_v && (!V || ldv < std::max<int64_t>(n, 1))) throw Error(RUTV_ERR_SHAPE, "V buffer");
            if (lda < std::max<int64_t>(m, 1) || ldt < std::max<int64_t>(m, 1))
                throw Error(RUTV_ERR_SHAPE, "leading dimension smaller than the row count");
            rutv::factorize_grid_host(o, A, n, lda, G, glen, T, ldt, U, ldu, V, ldv);
            return;
        }
        auto h2d = [&](double* d, int64_t ldd, const double* h, int64_t ldh, int64_t r, int64_t c) {
            if (r * c > 0)
                RUTV_CUDA(cudaMemcpy2DAsync(d, static_cast<size_t>(ldd) * 8, h, static_cast<size_t>(ldh) * 8,
                                            static_cast<size_t>(r) * 8, static_cast<size_t>(c), cudaMemcpyHostToDevice,
                                            s.s));
        };
        auto d2h = [&](double* h, int64_t ldh, const double* d, int64_t ldd, int64_t r, int64_t c) {
            if (h && r * c > 0)
                RUTV_CUDA(cudaMemcpy2DAsync(h, static_cast<size_t>(ldh) * 8, d, static_cast<size_t>(ldd) * 8,
                                            static_cast<size_t>(r) * 8, static_cast<size_t>(c), cudaMemcpyDeviceToHost,
                                            s.s));
        };
        {
            DMem<double> dG(G ? static_cast<size_t>(std::max<int64_t>(glen, 1)) : 1, s.s);
            if (G && glen > 0)
                RUTV_CUDA(cudaMemcpyAsync(dG.p, G, static_cast<size_t>(glen) * 8, cudaMemcpyHostToDevice, s.s));
            if (m == n) {
                // Square: ONE stacked device buffer [V; T] (V on top, ld = 2n) plus U,
                // factored in place -- A is uploaded straight into T's rows, the
                // results are read back from the same buffers: HBM peak 3 n^2 doubles
                // plus O(n b) workspace (config 5: 60 GB of 180).
                const int64_t vr = o->build_v ? nn : 0;
                const int64_t ld = std::max<int64_t>((vr + nn + 3) / 4 * 4, 1), ldu4 = std::max<int64_t>((nn + 3) / 4 * 4, 1);
                DMem<double> vt(static_cast<size_t>(ld * nn), s.s);
                DMem<double> dU(o->build_u ? static_cast<size_t>(ldu4 * nn) : 1, s.s);
                double* dT = vt.p + vr;
                h2d(dT, ld, A, lda, nn, nn);
                run_factorize(o, dT, n, n, ld, G ? dG.p : nullptr, glen, dT, ld, o->build_u ? dU.p : nullptr, ldu4,
                              o->build_v ? vt.p : nullptr, ld, s.s);
                d2h(T, ldt, dT, ld, nn, nn);
                if (o->build_u) d2h(U, ldu, dU.p, ldu4, nn, nn);
                if (o->build_v) d2h(V, ldv, vt.p, ld, nn, nn);
                RUTV_CUDA(cudaStreamSynchronize(s.s));
            } else {
                DMem<double> dA(static_cast<size_t>(mm * nn), s.s), dT(static_cast<size_t>(mm * nn), s.s);
                DMem<double> dU(o->build_u ? static_cast<size_t>(mm * mm) : 1, s.s);
                DMem<double> dV(o->build_v ? static_cast<size_t>(nn * nn) : 1, s.s);
                h2d(dA.p, std::max<int64_t>(mm, 1), A, lda, mm, nn);
                run_factorize(o, dA.p, m, n, std::max<int64_t>(mm, 1), G ? dG.p : nullptr, glen, dT.p,
                              std::max<int64_t>(mm, 1), o->build_u ? dU.p : nullptr, std::max<int64_t>(mm, 1),
                              o->build_v ? dV.p : nullptr, std::max<int64_t>(nn, 1), s.s);
                d2h(T, ldt, dT.p, std::max<int64_t>(mm, 1), mm, nn);
                if (o->build_u) d2h(U, ldu, dU.p, std::max<int64_t>(mm, 1), mm, mm);
                if (o->build_v) d2h(V, ldv, dV.p, std::max<int64_t>(nn, 1), nn, nn);
                RUTV_CUDA(cudaStreamSynchronize(s.s));
            }
        }
        RUTV_CUDA(cudaStreamSynchronize(s.s));  // the buffers' stream-ordered frees, before the trim
    });
}

int rutv_b200_factorize_device(const rutv_opts* o, const double* dA, int64_t m, int64_t n,
                               int64_t lda, const double* dG, int64_t g_len, double* dT,
                               int64_t ldt, double* dU, int64_t ldu, double* dV, int64_t ldv,
                               rutv_status* st) {
    return guarded(st, [&] {
        check_opts(o);
        set_device(o->device);
        rutv::pool_keep_this_call(o->keep_workspace != 0);
        Stream s(o->stream);
        run_factorize(o, dA, m, n, lda, dG, g_len, dT, ldt, dU, ldu, dV, ldv, s.s);
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

int rutv_b200_release_workspace(int device) {
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return RUTV_ERR_CUDA;
    }
    rutv::pool_release(device);
    return RUTV_OK;
}

int rutv_b200_last_profile(const char** names, double* ms, int cap) {
    return rutv::last_profile(names, ms, cap);
}

uint64_t rutv_b200_launch_count(void) { return rutv::launch_count(); }

int rutv_b200_host_alloc(size_t bytes, void** p, rutv_status* st) {
    return guarded(st, [&] {
        if (!p) throw Error(RUTV_ERR_SHAPE, "null output pointer");
        *p = nullptr;
        const cudaError_t e = cudaHostAlloc(p, bytes ? bytes : 8, cudaHostAllocPortable);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            throw Error(RUTV_ERR_OOM, "pinned host allocation of " + std::to_string(bytes) + " bytes failed");
        }
        RUTV_CUDA(e);
    });
}

int rutv_b200_copy_matrix_async(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                                int64_t cols, uint64_t stream, rutv_status* st) {
    return guarded(st, [&] {
        if (rows < 0 || cols < 0 || ldd < std::max<int64_t>(rows, 1) || lds < std::max<int64_t>(rows, 1))
            throw Error(RUTV_ERR_SHAPE, "copy_matrix: bad shape or leading dimension");
        if (rows * cols == 0) return;
        RUTV_CUDA(cudaMemcpy2DAsync(dst, static_cast<size_t>(ldd) * 8, src, static_cast<size_t>(lds) * 8,
                                    static_cast<size_t>(rows) * 8, static_cast<size_t>(cols), cudaMemcpyDefault,
                                    reinterpret_cast<cudaStream_t>(stream)));
    });
}

int rutv_b200_host_free(void* p, rutv_status* st) {
    return guarded(st, [&] {
        if (p) RUTV_CUDA(cudaFreeHost(p));
    });
}

int rutv_b200_gemm_profile(double* flops, double* ms, int64_t* launches) {
    return rutv::gemm_profile_get(flops, ms, launches);
}

int rutv_b200_gemm(int device, double alpha, int ta, const double* A, int64_t ar, int64_t ac,
                   int64_t lda, int tb, const double* B, int64_t br, int64_t bc, int64_t ldb,
                   double beta, double* C, int64_t m, int64_t n, int64_t ldc, rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        Stream s;
        const Op oa = ta ? Op::T : Op::N, ob = tb ? Op::T : Op::N;
        const int64_t k = ta ? ar : ac;
        const int64_t we = rutv::gemm_work_elems(m, n, k);
        DMem<double> w(static_cast<size_t>(std::max<int64_t>(we, 1)), s.s);
        rutv::gemm(s.s, alpha, oa, DView(ar, ac, lda, const_cast<double*>(A)), ob,
                   DView(br, bc, ldb, const_cast<double*>(B)), beta, DView(m, n, ldc, C), w.p, we);
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

int rutv_b200_hqr(int device, double* A, int64_t m, int64_t n, int64_t lda, double* tau,
                  double* twy, int64_t ldt, rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        Stream s;
        const int64_t we = rutv::hqr_work_elems(m, n) + m * std::min(m, n);
        DMem<double> w(static_cast<size_t>(std::max<int64_t>(we, 1)), s.s);
        rutv::hqr_panel(s.s, DView(m, n, lda, A), tau, twy, ldt, w.p, we);
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

static void apply_common(cudaStream_t s, const double* qr, int64_t sr, int64_t ldq, const double* twy,
                         int64_t p, int64_t ldt, double* B, int64_t other, int64_t ldb, bool right) {
    // M = W Twy';  right: B (other x sr) <- B - (B W) M';  left: B (sr x other) <- B - M (W' B)
    DMem<double> W(static_cast<size_t>(std::max<int64_t>(sr * p, 1)), s);
    DMem<double> M(static_cast<size_t>(std::max<int64_t>(sr * p, 1)), s);
    DMem<double> Z(static_cast<size_t>(std::max<int64_t>(other * p, 1)), s);
    const int64_t we = std::max({rutv::gemm_work_elems(other, p, sr), rutv::gemm_work_elems(p, other, sr),
                                 rutv::gemm_work_elems(sr, p, p), int64_t(1)});
    DMem<double> gw(static_cast<size_t>(we), s);
    DView Wv(sr, p, sr, W.p), Mv(sr, p, sr, M.p);
    rutv::make_w(s, DView(sr, p, ldq, const_cast<double*>(qr)), p, Wv);
    rutv::gemm(s, 1.0, Op::N, Wv, Op::T, DView(p, p, ldt, const_cast<double*>(twy)), 0.0, Mv, gw.p, we);
    if (right) {
        DView Bv(other, sr, ldb, B), Zv(other, p, std::max<int64_t>(other, 1), Z.p);
        rutv::gemm(s, 1.0, Op::N, Bv, Op::N, Wv, 0.0, Zv, gw.p, we);
        rutv::gemm(s, -1.0, Op::N, Zv, Op::T, Mv, 1.0, Bv, gw.p, we);
    } else {
        DView Bv(sr, other, ldb, B), Zv(p, other, std::max<int64_t>(p, 1), Z.p);
        rutv::gemm(s, 1.0, Op::T, Wv, Op::N, Bv, 0.0, Zv, gw.p, we);
        rutv::gemm(s, -1.0, Op::N, Mv, Op::N, Zv, 1.0, Bv, gw.p, we);
    }
}

int rutv_b200_apply_q_right(int device, const double* qr, int64_t s, int64_t ldq, const double* twy,
                            int64_t p, int64_t ldt, double* B, int64_t rows, int64_t ldb,
                            rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        if (p == 0 || rows == 0) return;  // householder.cpp:131
        Stream sm;
        apply_common(sm.s, qr, s, ldq, twy, p, ldt, B, rows, ldb, true);
        RUTV_CUDA(cudaStreamSynchronize(sm.s));
    });
}

int rutv_b200_apply_qt_left(int device, const double* qr, int64_t s, int64_t ldq, const double* twy,
                            int64_t p, int64_t ldt, double* B, int64_t cols, int64_t ldb,
                            rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        if (p == 0 || cols == 0) return;  // householder.cpp:105
        Stream sm;
        apply_common(sm.s, qr, s, ldq, twy, p, ldt, B, cols, ldb, false);
        RUTV_CUDA(cudaStreamSynchronize(sm.s));
    });
}

int rutv_b200_svd_block(int device, const double* A, int64_t n, int64_t lda, double tol,
                        int max_sweeps, double* U, double* sigma, double* V, rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        Stream s;
        const int64_t we = rutv::svd_work_elems(n, max_sweeps) + 16;
        DMem<double> w(static_cast<size_t>(we), s.s), stat(4, s.s);
        RUTV_CUDA(cudaMemsetAsync(stat.p, 0, 32, s.s));
        rutv::svd_block(s.s, DView(n, n, lda, const_cast<double*>(A)), U, sigma, V, w.p, we, stat.p, tol,
                        max_sweeps);
        double hs[4];
        RUTV_CUDA(cudaMemcpyAsync(hs, stat.p, 32, cudaMemcpyDeviceToHost, s.s));
        RUTV_CUDA(cudaStreamSynchronize(s.s));
        if (std::getenv("RUTV_DEBUG"))
            std::fprintf(stderr, "[rutv] svd_block n=%lld code=%g residual=%g kept=%g sweeps=%g\n",
                         static_cast<long long>(n), hs[0], hs[1], hs[2], hs[3]);
        if (hs[0] == RUTV_ERR_CONVERGENCE)
            throw Error(RUTV_ERR_CONVERGENCE, "jacobi sweeps exhausted", hs[1]);
    });
}

int rutv_b200_normal_fill(int device, uint64_t seed, uint64_t pos, double* G, int64_t rows,
                          int64_t cols, int64_t ldg, rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        Stream s;
        rutv::normal_fill(s.s, seed, pos, DView(rows, cols, ldg, G));
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

}  // extern "C"

extern "C" {

int rutv_b200_gaussian_matrix(int device, int64_t m, int64_t n, uint64_t seed, double* A,
                              int64_t lda, rutv_status* st) {
    return guarded(st, [&] {
        set_device(device);
        Stream s;
        rutv::normal_fill(s.s, seed, 0, DView(m, n, lda, A));
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

int rutv_b200_spectrum_matrix(int device, int64_t m, int64_t n, const double* sigma, double beta,
                              uint64_t seed, double* A, int64_t lda, rutv_status* st) {
    return guarded(st, [&] {
        const int64_t p = std::min(m, n);
        if (!sigma && !(beta > 0.0)) throw Error(RUTV_ERR_CONFIG, "geometric_matrix: decay factor must be positive");
        set_device(device);
        Stream s;
        std::vector<double> hs(static_cast<size_t>(std::max<int64_t>(p, 1)));
        double acc = 1.0;
        for (int64_t j = 0; j < p; ++j) {
            hs[static_cast<size_t>(j)] = sigma ? sigma[j] : acc;
            acc *= beta;
        }
        DMem<double> ds(static_cast<size_t>(std::max<int64_t>(p, 1)), s.s);
        RUTV_CUDA(cudaMemcpyAsync(ds.p, hs.data(), static_cast<size_t>(std::max<int64_t>(p, 1)) * 8,
                                  cudaMemcpyHostToDevice, s.s));
        rutv::spectrum_matrix(s.s, m, n, ds.p, seed, DView(m, n, lda, A));
        RUTV_CUDA(cudaStreamSynchronize(s.s));
    });
}

}  // extern "C"
