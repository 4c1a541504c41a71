// randutv.cu -- host driver of the B200 blocked randUTV (one GPU).
//
// Restates randutv::randutv (proj/src/randutv_blocked.cpp:84-157) step for
// step; every device operation is one of our sm_100a kernels (no cuBLAS /
// cuSOLVER, no host fallback).  Per step i (r0 = i*b, s = n - r0):
//   sketch    G -> Y = T22' G, q x (Z = T22 Y, Y = T22' Z)          :41-50
//   V-QR      Y = Q_v R (house() convention), W_v, Twy_v            :52-53
//   V-apply   [V; T(:, r0:)] <- [V; T(:, r0:)] Q_v                    :140-143
//   U-QR      panel T22(:, 0:b) = Q_u R in place, W_u, Twy_u         :146
//   Qu'-apply T22(:, b:) <- Q_u' T22(:, b:)                         :147
//   U-apply   U(:, r0:) <- U(:, r0:) Q_u                             :148
//   beta      svd(triu(T22(0:b,0:b))), diag write, strip Us' *,
//             right-multiplies by Vs / Us                           :150-154
// and the ragged tail (s <= b) is one dense SVD (:129-137).
//
// HBM layout: V (n x n) and T (n x n) are stacked in ONE column-major buffer
// VT of (n + n) rows, V on top (rows 0..n) and T below (rows n..2n), so the
// V-side transform of step i is a single pair of GEMMs over rows
// [0, 2n) x columns [r0, n): the reference's three apply_q_right calls on
// T22, T(0:r0, r0:) and V(:, r0:) collapse into one, and the rows that are
// off the critical path (V and the finished T rows) are the contiguous
// prefix [0, n + r0).  Block reflectors are applied in the form
//   B Q = B - (B W) M',   Q' B = B - M (W' B),   M = W Twy'
// (M formed once per step, shared by every target), which is the
// reference's three-GEMM apply with the small Twy product re-associated.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Stream-ordered device allocation from a pool that keeps its memory between
// calls (cudaMallocAsync), so repeated factorizations do not pay cudaMalloc.
struct DevBuf {
    double* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(int64_t elems, cudaStream_t s) : st(s) {
        if (elems <= 0) elems = 1;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), static_cast<size_t>(elems) * 8, s);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            throw Error(RUTV_ERR_OOM, "device allocation of " + std::to_string(elems * 8) + " bytes failed");
        }
        RUTV_CUDA(e);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        std::swap(p, o.p);
        std::swap(st, o.st);
        return *this;
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

void configure_pool(int device) {
    static bool done[64] = {};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

struct Profiler {
    bool on = false;
    cudaStream_t st;
    std::vector<std::string> names;
    std::vector<double> ms;
    std::vector<cudaEvent_t> evs;
    std::vector<int> ev_phase;
    void mark(int phase) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        evs.push_back(e);
        ev_phase.push_back(phase);
    }
    void finish() {
        if (!on) return;
        cudaEventSynchronize(evs.back());
        ms.assign(names.size(), 0.0);
        for (size_t i = 1; i < evs.size(); ++i) {
            float t = 0.f;
            cudaEventElapsedTime(&t, evs[i - 1], evs[i]);
            ms[ev_phase[i]] += t;
        }
        for (auto e : evs) cudaEventDestroy(e);
        evs.clear();
    }
};

thread_local std::vector<std::string> t_prof_names;
thread_local std::vector<double> t_prof_ms;

enum Phase { P_START, P_SKETCH, P_QRV, P_APPLYV, P_QRU, P_APPLYU, P_SVD, P_BETA, P_FINAL, P_N };
const char* kPhaseNames[P_N] = {"start", "sketch", "qr_v", "apply_v", "qr_u", "apply_u",
                                "svd", "beta", "final"};

}  // namespace


// Factorizes a square n x n device matrix; results written to the device
// output views.  Throws rutv::Error.
void factorize_device(cudaStream_t st, int device, int64_t n, const FactorArgs& fa) {
    const int64_t b = fa.b;
    configure_pool(device);
    Profiler prof;
    prof.on = std::getenv("RUTV_PROFILE") && std::strcmp(std::getenv("RUTV_PROFILE"), "0") != 0;
    prof.st = st;
    for (int i = 0; i < P_N; ++i) prof.names.push_back(kPhaseNames[i]);
    prof.mark(P_START);
    gemm_profile_begin();

    const bool bu = fa.build_u, bv = fa.build_v;
    const int64_t vr = bv ? n : 0;          // V rows on top of T in VT
    const int64_t ldvt = rup(std::max<int64_t>(vr + n, 1), 4);
    const int64_t ldu = rup(std::max<int64_t>(n, 1), 4);
    const int64_t bb = std::min(b, std::max<int64_t>(n, 1));

    DevBuf VT(ldvt * std::max<int64_t>(n, 1), st);
    DevBuf U(bu ? ldu * n : 1, st);
    DView vt(vr + n, n, ldvt, VT.p);
    DView tmat = vt.block(vr, 0, n, n);
    DView umat(n, n, ldu, U.p);

    // T := A, U := I, V := I   (randutv_blocked.cpp:114-120)
    copy_view(st, tmat, DView(n, n, fa.lda, const_cast<double*>(fa.dA)));
    if (bu) set_identity(st, umat);
    if (bv) set_identity(st, vt.block(0, 0, n, n));

    const int64_t sb = std::max<int64_t>(n * bb, 1);
    DevBuf G(fa.dG ? 1 : sb, st), Y(sb, st), Z(sb, st), Wv(sb, st), Mv(sb, st), Wu(sb, st), Mu(sb, st);
    DevBuf Zx(std::max<int64_t>((vr + n) * bb, 1), st);  // B*W for all VT rows / U rows
    DevBuf Zl(std::max<int64_t>(bb * n, 1), st);         // W'*B from the left, strip temp
    DevBuf Twy(bb * bb, st), Gram(bb * bb, st), tau(bb + 1, st);
    DevBuf Rb(bb * bb, st), Us(bb * bb, st), Vs(bb * bb, st), sig(bb + 1, st);
    const int64_t nsteps_max = n / std::max<int64_t>(b, 1) + 2;
    DevBuf jstat(4 * nsteps_max, st);
    RUTV_CUDA(cudaMemsetAsync(jstat.p, 0, static_cast<size_t>(4 * nsteps_max) * 8, st));
    const int64_t svdw = svd_work_elems(bb, 30);
    DevBuf SvdW(svdw, st);
    int64_t gw_elems = std::max<int64_t>({gemm_work_elems(n, bb, n), gemm_work_elems(bb, n, n),
                                          gemm_work_elems(vr + n, bb, n), gemm_work_elems(bb, bb, n),
                                          gemm_work_elems(bb, n, bb), 1});
    DevBuf GW(gw_elems, st);
    const int64_t hqw = hqr_work_elems(n, bb);
    DevBuf HQ(hqw, st);

    auto gemm_ = [&](double alpha, Op ta, const DView& a, Op tb, const DView& bm, double beta,
                     const DView& c) { gemm(st, alpha, ta, a, tb, bm, beta, c, GW.p, gw_elems); };

    // Compact-WY pieces of a packed panel qr (s x p): W, Twy, M = W Twy'.
    auto form_wy = [&](const DView& qr, int64_t p, double* wbuf, double* mbuf) {
        const int64_t s = qr.rows;
        DView W(s, p, s, wbuf), M(s, p, s, mbuf);
        make_w(st, qr, p, W);
        gemm_(1.0, Op::T, W, Op::N, W, 0.0, DView(p, p, p, Gram.p));
        form_t(st, Gram.p, p, tau.p, p, Twy.p, p);
        gemm_(1.0, Op::N, W, Op::T, DView(p, p, p, Twy.p), 0.0, M);
    };

    uint64_t pos = 0;  // stream position P_i
    int steps = 0;
    int jcount = 0;
    for (int64_t i = 0;; ++i) {
        const int64_t r0 = i * b, s = n - r0;
        if (s <= 0) break;
        if (fa.max_steps >= 0 && steps >= fa.max_steps) break;
        ++steps;
        DView t22 = tmat.block(r0, r0, s, s);

        if (s <= b) {  // ragged tail: one dense SVD (randutv_blocked.cpp:129-137)
            prof.mark(P_BETA);
            DView Xin(s, s, s, Rb.p);
            copy_view(st, Xin, t22);
            svd_block(st, Xin, Us.p, sig.p, Vs.p, SvdW.p, svdw, jstat.p + 4 * jcount++, 1e-15, 30);
            prof.mark(P_SVD);
            write_rect_diag(st, t22, sig.p, s);
            DView VsV(s, s, s, Vs.p), UsV(s, s, s, Us.p);
            if (vr + r0 > 0) {
                DView X = vt.block(0, r0, vr + r0, s);
                DView tmp(vr + r0, s, vr + r0, Zx.p);
                gemm_(1.0, Op::N, X, Op::N, VsV, 0.0, tmp);
                copy_view(st, X, tmp);
            }
            if (bu) {
                DView X = umat.block(0, r0, n, s);
                DView tmp(n, s, n, Zx.p);
                gemm_(1.0, Op::N, X, Op::N, UsV, 0.0, tmp);
                copy_view(st, X, tmp);
            }
            prof.mark(P_BETA);
            break;
        }

        // ---- sketch (build_v_alpha, randutv_blocked.cpp:41-50)
        DView Gv(s, b, s, fa.dG ? const_cast<double*>(fa.dG) + pos : G.p);
        if (!fa.dG) normal_fill(st, fa.seed, pos, Gv);
        pos += static_cast<uint64_t>(s * b);
        DView Yv(s, b, s, Y.p), Zv(s, b, s, Z.p);
        gemm_(1.0, Op::T, t22, Op::N, Gv, 0.0, Yv);
        for (int it = 0; it < fa.q; ++it) {
            gemm_(1.0, Op::N, t22, Op::N, Yv, 0.0, Zv);
            gemm_(1.0, Op::T, t22, Op::N, Zv, 0.0, Yv);
        }
        prof.mark(P_SKETCH);
        // ---- V-side QR (:52-53)
        hqr_panel(st, Yv, tau.p, nullptr, 0, HQ.p, hqw);
        form_wy(Yv, b, Wv.p, Mv.p);
        prof.mark(P_QRV);
        // ---- V-apply on all VT rows, columns r0.. (:140-143)
        {
            DView X = vt.block(0, r0, vr + n, s);
            DView ZxV(vr + n, b, vr + n, Zx.p);
            gemm_(1.0, Op::N, X, Op::N, DView(s, b, s, Wv.p), 0.0, ZxV);
            gemm_(-1.0, Op::N, ZxV, Op::T, DView(s, b, s, Mv.p), 1.0, X);
        }
        prof.mark(P_APPLYV);
        // ---- U-side QR of the panel, in place (build_u_alpha, :58-64)
        DView panel = t22.block(0, 0, s, b);
        hqr_panel(st, panel, tau.p, nullptr, 0, HQ.p, hqw);
        form_wy(panel, b, Wu.p, Mu.p);
        prof.mark(P_QRU);
        // ---- Q_u' on T22(:, b:) (:147) and U accumulate (:148)
        {
            DView B = t22.block(0, b, s, s - b);
            DView Zlv(b, s - b, b, Zl.p);
            gemm_(1.0, Op::T, DView(s, b, s, Wu.p), Op::N, B, 0.0, Zlv);
            gemm_(-1.0, Op::N, DView(s, b, s, Mu.p), Op::N, Zlv, 1.0, B);
            if (bu) {
                DView X = umat.block(0, r0, n, s);
                DView ZxU(n, b, n, Zx.p);
                gemm_(1.0, Op::N, X, Op::N, DView(s, b, s, Wu.p), 0.0, ZxU);
                gemm_(-1.0, Op::N, ZxU, Op::T, DView(s, b, s, Mu.p), 1.0, X);
            }
        }
        prof.mark(P_APPLYU);
        // ---- beta_stage (:66-82) and the small right-multiplies (:152-154)
        DView Rv(b, b, b, Rb.p);
        copy_upper(st, Rv, t22.block(0, 0, b, b));
        svd_block(st, Rv, Us.p, sig.p, Vs.p, SvdW.p, svdw, jstat.p + 4 * jcount++, 1e-15, 30);
        prof.mark(P_SVD);
        write_rect_diag(st, panel, sig.p, b);
        DView VsV(b, b, b, Vs.p), UsV(b, b, b, Us.p);
        {
            DView strip = t22.block(0, b, b, s - b);
            DView tmp(b, s - b, b, Zl.p);
            gemm_(1.0, Op::T, UsV, Op::N, strip, 0.0, tmp);
            copy_view(st, strip, tmp);
        }
        if (vr + r0 > 0) {
            DView X = vt.block(0, r0, vr + r0, b);
            DView tmp(vr + r0, b, vr + r0, Zx.p);
            gemm_(1.0, Op::N, X, Op::N, VsV, 0.0, tmp);
            copy_view(st, X, tmp);
        }
        if (bu) {
            DView X = umat.block(0, r0, n, b);
            DView tmp(n, b, n, Zx.p);
            gemm_(1.0, Op::N, X, Op::N, UsV, 0.0, tmp);
            copy_view(st, X, tmp);
        }
        prof.mark(P_BETA);
    }

    // results out (T rows vr.., V rows 0..n)
    copy_view(st, DView(n, n, fa.ldt, fa.dT), tmat);
    if (bu && fa.dU) copy_view(st, DView(n, n, fa.ldu, fa.dU), umat);
    if (bv && fa.dV) copy_view(st, DView(n, n, fa.ldv, fa.dV), vt.block(0, 0, n, n));
    prof.mark(P_FINAL);

    // Jacobi statuses: ConvergenceError surfaces like the reference's exception.
    std::vector<double> hs(static_cast<size_t>(4 * std::max(jcount, 1)));
    if (jcount > 0)
        RUTV_CUDA(cudaMemcpyAsync(hs.data(), jstat.p, static_cast<size_t>(4 * jcount) * 8,
                                  cudaMemcpyDeviceToHost, st));
    RUTV_CUDA(cudaStreamSynchronize(st));
    prof.finish();
    gemm_profile_end();
    if (prof.on) {
        t_prof_names = prof.names;
        t_prof_ms = prof.ms;
    }
    for (int k = 0; k < jcount; ++k)
        if (hs[4 * k] == RUTV_ERR_CONVERGENCE)
            throw Error(RUTV_ERR_CONVERGENCE,
                        "jacobi sweeps exhausted after 30 sweeps", hs[4 * k + 1]);
}

int last_profile(const char** names, double* ms, int cap) {
    const int n = std::min<int>(cap, static_cast<int>(t_prof_ms.size()));
    for (int i = 0; i < n; ++i) {
        if (names) names[i] = kPhaseNames[i];
        if (ms) ms[i] = t_prof_ms[static_cast<size_t>(i)];
    }
    return n;
}

}  // namespace rutv
