// step_api.cu -- the reference's public step-level API on the device.
//
// randutv_blocked.hpp:41-72 exposes, besides randutv(), the three stages one
// step of the blocked driver is made of; the reference's own harnesses use them
// for first-k-step runs (and the ref_shim replay in oracle/ref_shim.cpp):
//   build_v_alpha(t22, b, q, rng) -> StepTransform   randutv_blocked.cpp:40-55
//   build_u_alpha(panel)          -> StepTransform   randutv_blocked.cpp:57-63
//   beta_stage(t22, bw)           -> BetaFactors     randutv_blocked.cpp:65-81
// Each is restated here with the product's kernels (DMMA GEMM, cluster
// Householder QR with the reference house() convention, batched Jacobi SVD),
// in two C-ABI flavours: DEVICE pointers (stream-ordered, no host copies) and
// HOST pointers (what the C++ drop-in header's Matrix types bind to).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

void gemm_w(cudaStream_t st, double alpha, Op ta, const DView& a, Op tb, const DView& b, double beta,
            const DView& c) {
    const int64_t k = ta == Op::N ? a.cols : a.rows;
    const int64_t we = gemm_work_elems(c.rows, c.cols, k);
    DevBuf w(we, st);
    gemm(st, alpha, ta, a, tb, b, beta, c, w.p, we);
}

// hqr_inplace + form_wy_t (householder.cpp:48-97): packed QR in place, tau, Twy (p x p).
void qr_wy(cudaStream_t st, const DView& a, double* tau, double* twy) {
    const int64_t p = std::min(a.rows, a.cols);
    if (p == 0) return;
    const int64_t we = hqr_work_elems(a.rows, a.cols) + a.rows * p;
    DevBuf w(we, st);
    hqr_panel(st, a, tau, twy, p, w.p, we);
}

}  // namespace

// build_v_alpha (randutv_blocked.cpp:40-55).  qr: cols x b (ld cols); tau: min(cols, b);
// twy: p x p.  G (rows x b) is deviates pos .. pos + rows*b of RngState(seed), drawn on
// the device, or taken from dG (the host stream, bit-identical parity mode).
void build_v_alpha_device(cudaStream_t st, const DView& t22, int64_t b, int q, uint64_t seed, uint64_t pos,
                          const double* dG, double* qr, double* tau, double* twy) {
    const int64_t rows = t22.rows, cols = t22.cols;
    DevBuf Gb(dG ? 1 : rows * b, st), Zb(rows * b, st);
    DView g(rows, b, std::max<int64_t>(rows, 1), dG ? const_cast<double*>(dG) : Gb.p);
    if (!dG && rows * b > 0) normal_fill(st, seed, pos, g);
    DView y(cols, b, std::max<int64_t>(cols, 1), qr), z(rows, b, std::max<int64_t>(rows, 1), Zb.p);
    gemm_w(st, 1.0, Op::T, t22, Op::N, g, 0.0, y);
    for (int it = 0; it < q; ++it) {
        gemm_w(st, 1.0, Op::N, t22, Op::N, y, 0.0, z);
        gemm_w(st, 1.0, Op::T, t22, Op::N, z, 0.0, y);
    }
    qr_wy(st, y, tau, twy);
}

// build_u_alpha (randutv_blocked.cpp:57-63): the panel is factored in place; qr_copy
// (rows x cols, ld rows) receives the packed panel.
void build_u_alpha_device(cudaStream_t st, const DView& panel, double* qr_copy, double* tau, double* twy) {
    qr_wy(st, panel, tau, twy);
    if (qr_copy) copy_view(st, DView(panel.rows, panel.cols, std::max<int64_t>(panel.rows, 1), qr_copy), panel);
}

// beta_stage (randutv_blocked.cpp:65-81).  U: rt x rt, V: bw x bw (ld rt / bw),
// rt = min(rows, bw); Jacobi status (4 doubles) at dev_status.
void beta_stage_device(cudaStream_t st, const DView& t22, int64_t bw, double* U, double* V, double* dev_status) {
    const int64_t rows = t22.rows, cols = t22.cols;
    if (bw < 1 || bw > cols)
        throw Error(RUTV_ERR_SHAPE, "beta_stage: panel width " + std::to_string(bw) + " against " +
                                        std::to_string(cols) + " columns");
    const int64_t rt = std::min(rows, bw);
    DevBuf R(rt * bw, st), S(std::min(rt, bw) + 1, st);
    DView rv(rt, bw, std::max<int64_t>(rt, 1), R.p);
    copy_upper(st, rv, t22.block(0, 0, rt, bw));
    svd_full_device(st, rv, U, S.p, V, dev_status);
    write_rect_diag(st, t22.block(0, 0, rows, bw), S.p, std::min(rt, bw));
    if (cols > bw && rt > 0) {
        DView strip = t22.block(0, bw, rt, cols - bw);
        DevBuf tmp(rt * (cols - bw), st);
        DView tv(rt, cols - bw, std::max<int64_t>(rt, 1), tmp.p);
        gemm_w(st, 1.0, Op::T, DView(rt, rt, std::max<int64_t>(rt, 1), U), Op::N, strip, 0.0, tv);
        copy_view(st, strip, tv);
    }
}

}  // namespace rutv

// ------------------------------------------------------------------------ C ABI
namespace {

using rutv::DevBuf;
using rutv::DView;
using rutv::Error;

struct CallStream {
    cudaStream_t s = nullptr;
    bool own = false;
    CallStream(int device, uint64_t handle) {
        RUTV_CUDA(cudaSetDevice(device));
        if (handle) {
            s = reinterpret_cast<cudaStream_t>(handle);
        } else {
            RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own = true;
        }
    }
    ~CallStream() {
        if (own) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

int status(rutv_status* st, int code, const char* msg, double residual = 0.0) {
    if (st) {
        st->code = code;
        st->reserved = 0;
        st->residual = residual;
        std::snprintf(st->message, sizeof st->message, "%s", msg ? msg : "");
    }
    return code;
}

template <class F>
int run(rutv_status* st, F&& f) {
    int rc;
    try {
        f();
        rc = status(st, RUTV_OK, "");
    } catch (const Error& e) {
        rc = status(st, e.code, e.what(), e.residual);
    } catch (const std::exception& e) {
        rc = status(st, RUTV_ERR_INTERNAL, e.what());
    }
    rutv::pool_trim();
    return rc;
}

void check_view(int64_t rows, int64_t cols, int64_t ld) {
    if (rows < 0 || cols < 0) throw Error(RUTV_ERR_SHAPE, "negative matrix dimension");
    if (ld < std::max<int64_t>(rows, 1)) throw Error(RUTV_ERR_SHAPE, "leading dimension smaller than the row count");
}

void jacobi_status(cudaStream_t s, const double* dst) {
    double h[4];
    RUTV_CUDA(cudaMemcpyAsync(h, dst, sizeof h, cudaMemcpyDeviceToHost, s));
    RUTV_CUDA(cudaStreamSynchronize(s));
    if (h[0] == RUTV_ERR_CONVERGENCE) throw Error(RUTV_ERR_CONVERGENCE, "jacobi sweeps exhausted", h[1]);
}

void h2d(double* d, int64_t ldd, const double* h, int64_t ldh, int64_t r, int64_t c, cudaStream_t s) {
    if (r * c > 0)
        RUTV_CUDA(cudaMemcpy2DAsync(d, static_cast<size_t>(ldd) * 8, h, static_cast<size_t>(ldh) * 8,
                                    static_cast<size_t>(r) * 8, static_cast<size_t>(c), cudaMemcpyHostToDevice, s));
}
void d2h(double* h, int64_t ldh, const double* d, int64_t ldd, int64_t r, int64_t c, cudaStream_t s) {
    if (h && r * c > 0)
        RUTV_CUDA(cudaMemcpy2DAsync(h, static_cast<size_t>(ldh) * 8, d, static_cast<size_t>(ldd) * 8,
                                    static_cast<size_t>(r) * 8, static_cast<size_t>(c), cudaMemcpyDeviceToHost, s));
}

}  // namespace

extern "C" {

int rutv_b200_build_v_alpha_device(int device, uint64_t stream, const double* t22, int64_t rows, int64_t cols,
                                   int64_t ld, int64_t b, int q, uint64_t seed, uint64_t pos, const double* G,
                                   double* qr, double* tau, double* twy, rutv_status* st) {
    return run(st, [&] {
        if (b < 1) throw Error(RUTV_ERR_CONFIG, "block size must be >= 1, got " + std::to_string(b));
        if (q < 0) throw Error(RUTV_ERR_CONFIG, "power iteration count must be >= 0, got " + std::to_string(q));
        check_view(rows, cols, ld);
        CallStream cs(device, stream);
        rutv::build_v_alpha_device(cs.s, DView(rows, cols, ld, const_cast<double*>(t22)), b, q, seed, pos, G, qr,
                                   tau, twy);
        RUTV_CUDA(cudaStreamSynchronize(cs.s));
    });
}

int rutv_b200_build_u_alpha_device(int device, uint64_t stream, double* panel, int64_t rows, int64_t cols,
                                   int64_t ld, double* qr_copy, double* tau, double* twy, rutv_status* st) {
    return run(st, [&] {
        check_view(rows, cols, ld);
        CallStream cs(device, stream);
        rutv::build_u_alpha_device(cs.s, DView(rows, cols, ld, panel), qr_copy, tau, twy);
        RUTV_CUDA(cudaStreamSynchronize(cs.s));
    });
}

int rutv_b200_beta_stage_device(int device, uint64_t stream, double* t22, int64_t rows, int64_t cols, int64_t ld,
                                int64_t bw, double* U, double* V, rutv_status* st) {
    return run(st, [&] {
        check_view(rows, cols, ld);
        CallStream cs(device, stream);
        DevBuf js(4, cs.s);
        RUTV_CUDA(cudaMemsetAsync(js.p, 0, 32, cs.s));
        rutv::beta_stage_device(cs.s, DView(rows, cols, ld, t22), bw, U, V, js.p);
        jacobi_status(cs.s, js.p);
    });
}

int rutv_b200_build_v_alpha(int device, const double* t22, int64_t rows, int64_t cols, int64_t ld, int64_t b, int q,
                            uint64_t seed, uint64_t pos, const double* G, double* qr, double* tau, double* twy,
                            rutv_status* st) {
    return run(st, [&] {
        if (b < 1) throw Error(RUTV_ERR_CONFIG, "block size must be >= 1, got " + std::to_string(b));
        if (q < 0) throw Error(RUTV_ERR_CONFIG, "power iteration count must be >= 0, got " + std::to_string(q));
        check_view(rows, cols, ld);
        CallStream cs(device, 0);
        const int64_t p = std::min(cols, b);
        {
            DevBuf dT(rows * cols, cs.s), dG(G ? rows * b : 1, cs.s), dQ(cols * b, cs.s), dtau(p + 1, cs.s),
                dtw(p * p + 1, cs.s);
            h2d(dT.p, std::max<int64_t>(rows, 1), t22, ld, rows, cols, cs.s);
            if (G) h2d(dG.p, std::max<int64_t>(rows, 1), G, std::max<int64_t>(rows, 1), rows, b, cs.s);
            rutv::build_v_alpha_device(cs.s, DView(rows, cols, std::max<int64_t>(rows, 1), dT.p), b, q, seed, pos,
                                       G ? dG.p : nullptr, dQ.p, dtau.p, dtw.p);
            d2h(qr, std::max<int64_t>(cols, 1), dQ.p, std::max<int64_t>(cols, 1), cols, b, cs.s);
            d2h(tau, std::max<int64_t>(p, 1), dtau.p, std::max<int64_t>(p, 1), p, 1, cs.s);
            d2h(twy, std::max<int64_t>(p, 1), dtw.p, std::max<int64_t>(p, 1), p, p, cs.s);
            RUTV_CUDA(cudaStreamSynchronize(cs.s));
        }
        RUTV_CUDA(cudaStreamSynchronize(cs.s));
    });
}

int rutv_b200_build_u_alpha(int device, double* panel, int64_t rows, int64_t cols, int64_t ld, double* qr_copy,
                            double* tau, double* twy, rutv_status* st) {
    return run(st, [&] {
        check_view(rows, cols, ld);
        CallStream cs(device, 0);
        const int64_t p = std::min(rows, cols), l = std::max<int64_t>(rows, 1);
        {
            DevBuf dP(rows * cols, cs.s), dtau(p + 1, cs.s), dtw(p * p + 1, cs.s);
            h2d(dP.p, l, panel, ld, rows, cols, cs.s);
            rutv::build_u_alpha_device(cs.s, DView(rows, cols, l, dP.p), nullptr, dtau.p, dtw.p);
            d2h(panel, ld, dP.p, l, rows, cols, cs.s);
            d2h(qr_copy, l, dP.p, l, rows, cols, cs.s);
            d2h(tau, std::max<int64_t>(p, 1), dtau.p, std::max<int64_t>(p, 1), p, 1, cs.s);
            d2h(twy, std::max<int64_t>(p, 1), dtw.p, std::max<int64_t>(p, 1), p, p, cs.s);
            RUTV_CUDA(cudaStreamSynchronize(cs.s));
        }
        RUTV_CUDA(cudaStreamSynchronize(cs.s));
    });
}

int rutv_b200_beta_stage(int device, double* t22, int64_t rows, int64_t cols, int64_t ld, int64_t bw, double* U,
                         double* V, rutv_status* st) {
    return run(st, [&] {
        check_view(rows, cols, ld);
        if (bw < 1 || bw > cols)
            throw Error(RUTV_ERR_SHAPE, "beta_stage: panel width " + std::to_string(bw) + " against " +
                                            std::to_string(cols) + " columns");
        CallStream cs(device, 0);
        const int64_t rt = std::min(rows, bw), l = std::max<int64_t>(rows, 1);
        {
            DevBuf dT(rows * cols, cs.s), dU(rt * rt + 1, cs.s), dV(bw * bw, cs.s), js(4, cs.s);
            RUTV_CUDA(cudaMemsetAsync(js.p, 0, 32, cs.s));
            h2d(dT.p, l, t22, ld, rows, cols, cs.s);
            rutv::beta_stage_device(cs.s, DView(rows, cols, l, dT.p), bw, dU.p, dV.p, js.p);
            jacobi_status(cs.s, js.p);
            d2h(t22, ld, dT.p, l, rows, cols, cs.s);
            d2h(U, std::max<int64_t>(rt, 1), dU.p, std::max<int64_t>(rt, 1), rt, rt, cs.s);
            d2h(V, bw, dV.p, bw, bw, bw, cs.s);
            RUTV_CUDA(cudaStreamSynchronize(cs.s));
        }
        RUTV_CUDA(cudaStreamSynchronize(cs.s));
    });
}

}  // extern "C"
