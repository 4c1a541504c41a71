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
// V-side transform of step i is over rows [0, 2n) x columns [r0, n): the
// reference's three apply_q_right calls on T22, T(0:r0, r0:) and V(:, r0:)
// become the critical rows [n + r0, 2n) (T22) plus ONE off-critical block,
// the contiguous prefix [0, n + r0) (V and the finished T rows).  Block
// reflectors are applied as
//   B Q = B - (B W) M',   Q' B = B - M (W' B),   M = W Twy'
// (M formed once per step, shared by every target) -- the reference's
// three-GEMM apply with the small Twy product re-associated.
//
// Schedule.  Stream A (the caller's) carries the critical chain, the only
// work the NEXT step's trailing matrix depends on:
//   sketch -> QR(Y) -> V-apply on T22 -> QR(panel) -> Qu' on T22(:, b:).
// Stream B carries the V/U accumulation of the step.  The beta stage is
// DEFERRED: beta_stage only ever left-multiplies finished ROW blocks
// (strip T(r0:r0+b, r0+b:) by Us') and right-multiplies finished COLUMN
// blocks (T(0:r0, r0:r0+b), U(:, r0:r0+b), V(:, r0:r0+b) by Vs / Us) and
// writes the finished panel columns; later steps only right-multiply columns
// >= r0+b.  Left and right multiplications commute, so every step's R is
// saved and all SVDs run as ONE batched launch after the loop, followed by
// the strips (disjoint row blocks) and the right-multiplies (disjoint column
// blocks).  Mathematically identical to the reference order; the rounding
// differs only at the ulp level.  Results are bit-identical with overlap off.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Profiler {
    bool on = false;
    cudaStream_t st;
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
    void finish(int nphase) {
        if (!on) return;
        cudaEventSynchronize(evs.back());
        ms.assign(static_cast<size_t>(nphase), 0.0);
        for (size_t i = 1; i < evs.size(); ++i) {
            float t = 0.f;
            cudaEventElapsedTime(&t, evs[i - 1], evs[i]);
            ms[static_cast<size_t>(ev_phase[i])] += t;
        }
        for (auto e : evs) cudaEventDestroy(e);
        evs.clear();
    }
};

thread_local std::vector<double> t_prof_ms;

enum Phase { P_START, P_SKETCH, P_QRV, P_APPLYV, P_QRU, P_APPLYU, P_SVD, P_BETA, P_FINAL, P_WYV, P_WYU, P_N };
const char* kPhaseNames[P_N] = {"start", "sketch", "qr_v", "apply_v", "qr_u", "apply_u",
                                "svd", "beta", "final", "wy_v", "wy_u"};

}  // namespace

// One factorization.  With `cqr` the panel QRs take the Cholesky-QR2 path in
// deferred mode (cholqr.cu); returns false -- before anything is written to
// the caller's outputs -- when one of its panels was numerically unsafe.
static bool factorize_impl(cudaStream_t st_in, int device, int64_t n, const FactorArgs& fa, bool cqr) {
    const int64_t b = fa.b;
    Profiler prof;
    prof.on = std::getenv("RUTV_PROFILE") && std::strcmp(std::getenv("RUTV_PROFILE"), "0") != 0;
    prof.st = st_in;
    prof.mark(P_START);
    gemm_profile_begin();
    const char* ov_env = std::getenv("RUTV_OVERLAP");
    // RUTV_PROFILE=1: phase times with the streams serialised; =2: phase times of
    // the critical stream with the overlap kept (a timeline of the real schedule)
    const bool prof_overlap = prof.on && std::strcmp(std::getenv("RUTV_PROFILE"), "2") == 0;
    const bool overlap = fa.overlap && (!prof.on || prof_overlap) && !(ov_env && std::strcmp(ov_env, "0") == 0);

    const bool bu = fa.build_u, bv = fa.build_v;
    const int64_t vr = bv ? n : 0;  // V rows on top of T in VT
    const int64_t bb = std::min(b, std::max<int64_t>(n, 1));
    // In-place outputs (no n x n copies, HBM peak = the caller's buffers + O(n b)
    // workspace): U is always factored in the caller's U; T and V when V sits
    // directly on top of T in one caller buffer (dT == dV + n, ldt == ldv -- the
    // stacked layout bench.py and the host-pointer entry allocate) or when V is
    // not built.  The deferred Cholesky-QR2 mode may re-run the factorization, so
    // it keeps private buffers and leaves the caller's A intact.
    const bool vt_inplace = !cqr && n > 0 && (!bv || (fa.dV && fa.dT == fa.dV + n && fa.ldt == fa.ldv));
    const bool u_inplace = !cqr && bu && fa.dU;
    const int64_t ldvt = vt_inplace ? (bv ? fa.ldv : fa.ldt) : rup(std::max<int64_t>(vr + n, 1), 4);
    const int64_t ldu = u_inplace ? fa.ldu : rup(std::max<int64_t>(n, 1), 4);

    // ---- step plan: r0, s and kind of every loop iteration (max_steps honoured)
    struct StepInfo {
        int64_t r0, s;
        bool tail;
    };
    std::vector<StepInfo> plan;
    for (int64_t i = 0;; ++i) {
        const int64_t r0 = i * b, s = n - r0;
        if (s <= 0) break;
        if (fa.max_steps >= 0 && static_cast<int>(plan.size()) >= fa.max_steps) break;
        plan.push_back({r0, s, s <= b});
        if (s <= b) break;
    }
    const int nsteps = static_cast<int>(plan.size());

    // Streams.  With overlap the critical chain runs on a HIGH-priority stream
    // A (and its look-ahead helper C), the V/U accumulation on a low-priority
    // stream B: when both have blocks waiting, the block scheduler hands free
    // SMs to the critical chain first and B fills the rest (the panel QR
    // kernels leave ~130 SMs idle).  Stream A first waits for the caller's
    // stream (the input may still be in flight there); the call ends with a
    // host synchronisation on A, so the results are complete on return.
    // Stream D (high priority) forms Twy and M = W Twy' of each panel while A
    // already runs the big W-only product of the apply (X W, resp. W' B).
    // Stream E (low priority), RUTV_SVD_STREAM=1 only: each step's b x b Jacobi SVD is
    // launched as soon as its R is saved, beside the following steps, instead of the one
    // batched launch after the loop.  Measured 3x SLOWER (config 1 15.9 -> 52.3 ms,
    // config 2 49.1 -> 97.0 ms): a resident Jacobi cluster holds its SMs for ~3 ms, and
    // the 16-CTA panel-QR clusters on the critical chain cannot be placed in a GPC until
    // it leaves.  Kept as an experiment switch; the batched launch is the product.
    const char* sv_env = std::getenv("RUTV_SVD_STREAM");
    const bool svd_per_step = sv_env && std::strcmp(sv_env, "0") != 0;
    cudaStream_t st = st_in, sB = st_in, sC = st_in, sD = st_in, sE = st_in;
    if (overlap) {
        int prio_lo = 0, prio_hi = 0;
        RUTV_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sE, cudaStreamNonBlocking, prio_lo));
        RUTV_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio_hi));
        // C (look-ahead GEMMs that run beside the panel QR) one level below A:
        // a pending QR cluster must not wait behind C's CTAs for its 16 SMs.
        const int prio_mid = prio_hi < prio_lo ? prio_hi + 1 : prio_hi;
        RUTV_CUDA(cudaStreamCreateWithPriority(&sC, cudaStreamNonBlocking, prio_mid));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sD, cudaStreamNonBlocking, prio_hi));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sB, cudaStreamNonBlocking, prio_lo));
        cudaEvent_t e_in;
        RUTV_CUDA(cudaEventCreateWithFlags(&e_in, cudaEventDisableTiming));
        RUTV_CUDA(cudaEventRecord(e_in, st_in));
        RUTV_CUDA(cudaStreamWaitEvent(st, e_in, 0));
        cudaEventDestroy(e_in);
    }
    struct StreamGuard {
        cudaStream_t s;
        bool own;
        ~StreamGuard() {  // declared before every buffer: runs after their stream-ordered frees
            if (own) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        }
    } sguardA{st, overlap}, sguard{sB, overlap}, sguardC{sC, overlap}, sguardD{sD, overlap}, sguardE{sE, overlap};
    if (prof_overlap) {  // re-anchor the timeline on the critical stream
        prof.st = st;
        prof.mark(P_START);
    }
    std::vector<cudaEvent_t> events;
    struct EventGuard {
        std::vector<cudaEvent_t>& ev;
        ~EventGuard() {
            for (auto e : ev) cudaEventDestroy(e);
        }
    } eguard{events};
    auto record = [&](cudaStream_t s) {
        cudaEvent_t e;
        RUTV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        RUTV_CUDA(cudaEventRecord(e, s));
        events.push_back(e);
        return e;
    };
    auto wait = [&](cudaStream_t s, cudaEvent_t e) {
        if (overlap && e) RUTV_CUDA(cudaStreamWaitEvent(s, e, 0));
    };

    DevBuf VT(vt_inplace ? 1 : ldvt * std::max<int64_t>(n, 1), st);
    DevBuf U(bu && !u_inplace ? ldu * n : 1, st);
    DView vt(vr + n, n, ldvt, vt_inplace ? (bv ? fa.dV : fa.dT) : VT.p);
    DView tmat = vt.block(vr, 0, n, n);
    DView umat(n, n, ldu, u_inplace ? fa.dU : U.p);

    // T := A, U := I, V := I   (randutv_blocked.cpp:114-120)
    if (tmat.data != fa.dA || tmat.ld != fa.lda) copy_view(st, tmat, DView(n, n, fa.lda, const_cast<double*>(fa.dA)));
    if (bu) set_identity(st, umat);
    if (bv) set_identity(st, vt.block(0, 0, n, n));

    const int64_t sb = std::max<int64_t>(n * bb, 1);
    // stream A private
    DevBuf G(fa.dG ? 1 : sb, st), Y(sb, st), Z(sb, st), ZxA(std::max<int64_t>((vr + n) * bb, 1), st);
    // sketch hoisting (see the step loop): the next step's G and Y, H = M_u(b:, :)' G
    DevBuf G2(fa.dG ? 1 : sb, st), Y2(sb, st), Hh(bb * bb, st);
    double* Gb[2] = {G.p, G2.p};
    double* Yb[2] = {Y.p, Y2.p};
    const char* hoist_env = std::getenv("RUTV_HOIST");
    const bool hoist = !(hoist_env && std::strcmp(hoist_env, "0") == 0);
    DevBuf ZlA(sb, st), Twy(bb * bb, st), Gram(bb * bb, st), tau(bb + 1, st), tauU(bb + 1, st);
    // double-buffered A -> B hand-off
    DevBuf Wv0(sb, st), Wv1(sb, st), Mv0(sb, st), Mv1(sb, st);
    DevBuf Wu0(sb, st), Wu1(sb, st), Mu0(sb, st), Mu1(sb, st);
    double* Wv[2] = {Wv0.p, Wv1.p};
    double* Mv[2] = {Mv0.p, Mv1.p};
    double* Wu[2] = {Wu0.p, Wu1.p};
    double* Mu[2] = {Mu0.p, Mu1.p};
    // stream B private
    DevBuf ZxB(std::max<int64_t>((vr + n) * bb, 1), st);
    // deferred beta stage: every step's R, Us, Vs, sigma, status, scratch
    const int ns = std::max(nsteps, 1);
    const int64_t svdw = svd_work_elems(bb, 30);
    DevBuf Rall(ns * bb * bb, st), Usall(ns * bb * bb, st), Vsall(ns * bb * bb, st);
    DevBuf Sall(ns * (bb + 1), st), Jst(ns * 4, st), SvdW(ns * svdw, st);
    const int64_t desc_words = (static_cast<int64_t>(sizeof(SvdDesc)) * ns + 7) / 8;
    DevBuf Ddesc(desc_words, st);
    RUTV_CUDA(cudaMemsetAsync(Jst.p, 0, static_cast<size_t>(ns) * 32, st));
    // every step's SVD problem descriptor (known from the plan), uploaded once
    int64_t svd_nmax = 0;
    if (nsteps > 0) {
        std::vector<SvdDesc> descs(static_cast<size_t>(nsteps));
        for (int i = 0; i < nsteps; ++i) {
            const StepInfo& si = plan[static_cast<size_t>(i)];
            const int64_t w = si.tail ? si.s : b;
            svd_nmax = std::max(svd_nmax, w);
            const int64_t off = static_cast<int64_t>(i) * bb * bb;
            descs[static_cast<size_t>(i)] =
                SvdDesc{Rall.p + off, w, static_cast<int>(w), 0, Usall.p + off,
                        Sall.p + static_cast<int64_t>(i) * (bb + 1), Vsall.p + off,
                        SvdW.p + static_cast<int64_t>(i) * svdw, Jst.p + 4 * i};
        }
        RUTV_CUDA(cudaMemcpyAsync(Ddesc.p, descs.data(), sizeof(SvdDesc) * descs.size(), cudaMemcpyHostToDevice,
                                  st));
        RUTV_CUDA(cudaStreamSynchronize(st));  // the host vector dies at this scope's end
    }
    const SvdDesc* ddesc = reinterpret_cast<const SvdDesc*>(Ddesc.p);
    auto launch_svd = [&](int i, int64_t w) {  // step i's Jacobi on stream E, after R_i is saved
        if (!svd_per_step) return;
        wait(sE, record(st));
        svd_batch(sE, ddesc + i, 1, static_cast<int>(w), 1e-15, 30);
    };
    const int64_t gw_elems =
        std::max<int64_t>({gemm_work_elems(n, bb, n), gemm_work_elems(bb, n, n), gemm_work_elems(vr + n, bb, n),
                           gemm_work_elems(bb, bb, n), gemm_work_elems(bb, n, bb), gemm_work_elems(vr + n, bb, bb),
                           1});
    DevBuf GWA(gw_elems, st), GWB(gw_elems, st), GWC(gw_elems, st), GWD(gw_elems, st);
    const int64_t hqw = hqr_work_elems(n, bb);
    DevBuf HQ(hqw, st);
    DevBuf Cqf(1, st);  // Cholesky-QR2 safety flags of every panel (deferred mode)
    int* cqr_flag = cqr ? reinterpret_cast<int*>(Cqf.p) : nullptr;
    if (cqr_flag) RUTV_CUDA(cudaMemsetAsync(cqr_flag, 0, sizeof(int), st));
    struct DeferGuard {
        explicit DeferGuard(int* f) { cholqr_set_deferred(f); }
        ~DeferGuard() { cholqr_set_deferred(nullptr); }
    } dguard(cqr_flag);
    // allocations are stream-ordered on st; streams B and C must see them
    {
        const cudaEvent_t ev = record(st);
        wait(sB, ev);
        wait(sC, ev);
        wait(sD, ev);
        wait(sE, ev);
    }
    // declared after every buffer -> destroyed first: stream B drains before any
    // buffer is released (also on the exception path)
    struct JoinGuard {
        cudaStream_t a, s, c, d, e;
        bool own;
        ~JoinGuard() {
            if (own) {
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(s);
                cudaStreamSynchronize(c);
                cudaStreamSynchronize(d);
                cudaStreamSynchronize(e);
            }
        }
    } jguard{st, sB, sC, sD, sE, overlap};

    auto gemmA = [&](double alpha, Op ta, const DView& a, Op tb, const DView& bm, double beta,
                     const DView& c) { gemm(st, alpha, ta, a, tb, bm, beta, c, GWA.p, gw_elems); };
    auto gemmB = [&](double alpha, Op ta, const DView& a, Op tb, const DView& bm, double beta,
                     const DView& c) { gemm(sB, alpha, ta, a, tb, bm, beta, c, GWB.p, gw_elems); };

    // Compact-WY pieces of a packed panel qr (s x p): W on stream A, then
    // Twy (Gram + form_wy_t) and M = W Twy' on stream D; returns D's event.
    auto form_wy = [&](const DView& qr, int64_t p, const double* taus, double* wbuf, double* mbuf) {
        const int64_t s = qr.rows;
        DView W(s, p, s, wbuf), M(s, p, s, mbuf);
        make_w(st, qr, p, W);
        wait(sD, record(st));
        gemm(sD, 1.0, Op::T, W, Op::N, W, 0.0, DView(p, p, p, Gram.p), GWD.p, gw_elems);
        form_t(sD, Gram.p, p, taus, p, Twy.p, p);
        gemm(sD, 1.0, Op::N, W, Op::T, DView(p, p, p, Twy.p), 0.0, M, GWD.p, gw_elems);
        return record(sD);
    };

    uint64_t pos = 0;  // stream position P_i
    bool have_y = false;  // Y of this step formed by the previous one
    std::vector<cudaEvent_t> evB;
    NvtxRange loop_range("rutv/steps");
    // NVTX phase ranges of the step (host enqueue order; Nsight projects them onto the
    // kernels launched inside): sketch / qr_v / apply_v / qr_u / apply_u / accumulate
    struct Phase {
        bool open = false;
        void operator()(const char* name) {
            if (open) nvtxRangePop();
            nvtxRangePushA(name);
            open = true;
        }
        ~Phase() {
            if (open) nvtxRangePop();
        }
    };
    for (int i = 0; i < nsteps; ++i) {
        Phase phase;
        const int64_t r0 = plan[static_cast<size_t>(i)].r0, s = plan[static_cast<size_t>(i)].s;
        DView t22 = tmat.block(r0, r0, s, s);
        double* Ri = Rall.p + static_cast<int64_t>(i) * bb * bb;
        if (plan[static_cast<size_t>(i)].tail) {  // ragged tail: dense s x s block (:129-137)
            copy_view(st, DView(s, s, s, Ri), t22);
            launch_svd(i, s);
            break;
        }
        const int par = i & 1;
        if (i >= 2) wait(st, evB[static_cast<size_t>(i - 2)]);  // slot `par` free again
        const bool hoist_next = hoist && i + 1 < nsteps && !plan[static_cast<size_t>(i + 1)].tail;

        phase("rutv/sketch");
        // ---- sketch (build_v_alpha, randutv_blocked.cpp:41-50).  Y = T22' G was
        // already formed during the previous step when it was hoisted (below).
        DView Yv(s, b, s, Yb[par]), Zv(s, b, s, Z.p);
        if (!have_y) {
            DView Gv(s, b, s, fa.dG ? const_cast<double*>(fa.dG) + pos : Gb[par]);
            if (!fa.dG) normal_fill(st, fa.seed, pos, Gv);
            gemmA(1.0, Op::T, t22, Op::N, Gv, 0.0, Yv);
        }
        have_y = false;
        pos += static_cast<uint64_t>(s * b);
        for (int it = 0; it < fa.q; ++it) {
            gemmA(1.0, Op::N, t22, Op::N, Yv, 0.0, Zv);
            gemmA(1.0, Op::T, t22, Op::N, Zv, 0.0, Yv);
        }
        prof.mark(P_SKETCH);
        phase("rutv/qr_v");
        // ---- V-side QR (:52-53)
        hqr_panel(st, Yv, tau.p, nullptr, 0, HQ.p, hqw);
        prof.mark(P_QRV);
        const cudaEvent_t evTv = form_wy(Yv, b, tau.p, Wv[par], Mv[par]);
        prof.mark(P_WYV);
        DView WvV(s, b, s, Wv[par]), MvV(s, b, s, Mv[par]);
        cudaEvent_t evR = nullptr, evV = nullptr, evPan = nullptr;
        {  // V-apply, critical rows: T22 (:140).  Panel-first look-ahead: the
           // U-side QR only needs T22 Q_v's first b columns, so those are
           // updated first on stream A and the other s-b columns on stream C,
           // overlapping the panel QR.  Zx = X W needs only W: it runs while
           // stream D forms Twy and M.
            DView X = vt.block(vr + r0, r0, s, s);
            DView Zx(s, b, s, ZxA.p);
            gemmA(1.0, Op::N, X, Op::N, WvV, 0.0, Zx);
            wait(st, evTv);
            evV = record(st);  // W_v, M_v ready for stream B
            gemmA(-1.0, Op::N, Zx, Op::T, DView(b, b, s, Mv[par]), 1.0, X.block(0, 0, s, b));
            evPan = record(st);  // panel columns updated: C may start (enqueued after QR_u)
        }
        prof.mark(P_APPLYV);
        phase("rutv/qr_u");
        // ---- U-side QR of the panel, in place (build_u_alpha, :58-64)
        DView panel = t22.block(0, 0, s, b);
        auto stream_c_work = [&] {  // the other s-b columns of the V-apply, then the hoisted sketch
            DView X = vt.block(vr + r0, r0, s, s);
            DView Zx(s, b, s, ZxA.p);
            wait(sC, evPan);
            gemm(sC, -1.0, Op::N, Zx, Op::T, DView(s - b, b, s, Mv[par] + b), 1.0, X.block(0, b, s, s - b),
                 GWC.p, gw_elems);
            // Sketch hoisting.  The next trailing matrix is T22' = B(b:, :) - M_u(b:, :) Zl
            // with B = (T22 Q_v)(:, b:) -- final right here -- and Zl = W_u' B, so
            //   Y' = T22'^T G' = B(b:, :)^T G' - Zl^T (M_u(b:, :)^T G').
            // The big product P = B(b:, :)^T G' runs now on stream C, on the SMs
            // the panel QR leaves idle; the b-wide correction follows Q_u' on A.
            // Mathematically the reference's Y = T22'^T G (randutv_blocked.cpp:45).
            if (hoist_next) {
                const int64_t s2 = s - b;
                DView G2v(s2, b, s2, fa.dG ? const_cast<double*>(fa.dG) + pos : Gb[par ^ 1]);
                if (!fa.dG) normal_fill(sC, fa.seed, pos, G2v);
                gemm(sC, 1.0, Op::T, X.block(b, b, s2, s2), Op::N, G2v, 0.0, DView(s2, b, s2, Yb[par ^ 1]), GWC.p,
                     gw_elems);
            }
            evR = record(sC);
        };
        // Stream C is enqueued after the QR_u launch so the QR cluster gets its SMs before
        // C's CTAs fill the GPU -- except for tall panels, whose Cholesky-QR2 sub-panels
        // synchronise the host with stream A (safety flag): there C must already be queued.
        const bool c_first = overlap && cholqr_tall(s);
        if (c_first) stream_c_work();
        hqr_panel(st, panel, tauU.p, nullptr, 0, HQ.p, hqw);
        prof.mark(P_QRU);
        if (!c_first) stream_c_work();
        const cudaEvent_t evTu = form_wy(panel, b, tauU.p, Wu[par], Mu[par]);
        copy_upper(st, DView(b, b, b, Ri), t22.block(0, 0, b, b));  // beta_stage's R (:73-75)
        launch_svd(i, b);
        prof.mark(P_WYU);
        DView WuV(s, b, s, Wu[par]), MuV(s, b, s, Mu[par]);
        wait(st, evR);
        {  // Q_u' on T22(:, b:) (:147); Zl = W_u' B overlaps D's Twy / M_u
            DView B = t22.block(0, b, s, s - b);
            DView Zl(b, s - b, b, ZlA.p);
            gemmA(1.0, Op::T, WuV, Op::N, B, 0.0, Zl);
            wait(st, evTu);
            gemmA(-1.0, Op::N, MuV, Op::N, Zl, 1.0, B);
            if (hoist_next) {  // Y' = P - Zl^T (M_u(b:, :)^T G')
                const int64_t s2 = s - b;
                DView G2v(s2, b, s2, fa.dG ? const_cast<double*>(fa.dG) + pos : Gb[par ^ 1]);
                DView H(b, b, b, Hh.p);
                gemmA(1.0, Op::T, MuV.block(b, 0, s2, b), Op::N, G2v, 0.0, H);
                gemmA(-1.0, Op::T, DView(b, s2, b, ZlA.p), Op::N, H, 1.0, DView(s2, b, s2, Yb[par ^ 1]));
                have_y = true;
            }
        }
        const cudaEvent_t evU = record(st);
        prof.mark(P_APPLYU);

        phase("rutv/accumulate");
        // ======== stream B: V / U accumulation of step i ========
        wait(sB, evV);
        if (vr + r0 > 0) {  // V-apply on V and T(0:r0, r0:) (:141-143)
            DView X = vt.block(0, r0, vr + r0, s);
            DView Zx(vr + r0, b, vr + r0, ZxB.p);
            gemmB(1.0, Op::N, X, Op::N, WvV, 0.0, Zx);
            gemmB(-1.0, Op::N, Zx, Op::T, MvV, 1.0, X);
        }
        wait(sB, evU);
        if (bu) {  // U accumulate (:148)
            DView X = umat.block(0, r0, n, s);
            DView Zx(n, b, n, ZxB.p);
            gemmB(1.0, Op::N, X, Op::N, WuV, 0.0, Zx);
            gemmB(-1.0, Op::N, Zx, Op::T, MuV, 1.0, X);
        }
        evB.push_back(record(sB));
        prof.mark(P_APPLYU);
    }
    if (overlap) wait(st, record(sB));  // join

    // ======== deferred beta stage (:66-82, :129-137, :150-154) ========
    NvtxRange beta_range("rutv/deferred_beta");
    if (nsteps > 0) {
        if (svd_per_step)
            wait(st, record(sE));  // the per-step Jacobis (launched during the loop) are done
        else
            svd_batch(st, ddesc, nsteps, static_cast<int>(svd_nmax), 1e-15, 30);
        prof.mark(P_SVD);
        const cudaEvent_t evS = record(st);
        // Products with the SVD factors: one grouped in-place launch per kind
        // when the blocks fit the grouped kernel (w <= 128), else per-step GEMMs.
        const bool grouped = bb <= small_mul_max_w();
        int64_t ext_r = 0, ext_l = 0;
        for (const StepInfo& si : plan) {
            ext_r += vr + si.r0 + n;
            ext_l += si.s;
        }
        const size_t gsb = small_mul_scratch_bytes(static_cast<size_t>(nsteps), std::max(ext_r, ext_l));
        DevBuf GsA(static_cast<int64_t>(2 * gsb / 8 + 8), st), GsB(static_cast<int64_t>(gsb / 8 + 8), st);
        DevBuf GsD(static_cast<int64_t>(nsteps * sizeof(RectDiagDesc) / 8 + 8), st);
        // U right-multiplies on stream B (disjoint buffer)
        if (bu && grouped) {
            wait(sB, evS);
            std::vector<SmallMulDesc> ud;
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                const int64_t w = si.tail ? si.s : b;
                ud.push_back({umat.data + si.r0 * umat.ld, umat.ld, n, w, Usall.p + static_cast<int64_t>(i) * bb * bb, w,
                              static_cast<int>(w), 0});
            }
            small_mul_grouped(sB, false, ud, GsB.p, gsb);
        } else if (bu) {
            wait(sB, evS);
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                const int64_t w = si.tail ? si.s : b;
                const int64_t off = static_cast<int64_t>(i) * bb * bb;
                DView X = umat.block(0, si.r0, n, w);
                DView tmp(n, w, n, ZxB.p);
                gemmB(1.0, Op::N, X, Op::N, DView(w, w, w, Usall.p + off), 0.0, tmp);
                copy_view(sB, X, tmp);
            }
        }
        // diagonal writes (finished panel columns), then strips (row blocks),
        // then V/T right-multiplies (column blocks) on stream A
        {
            std::vector<RectDiagDesc> rd;
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                const int64_t w = si.tail ? si.s : b;
                DView blk = tmat.block(si.r0, si.r0, si.s, w);
                rd.push_back({blk.data, blk.rows, blk.cols, blk.ld, Sall.p + static_cast<int64_t>(i) * (bb + 1), w});
            }
            rect_diag_grouped(st, rd, GsD.p, static_cast<size_t>(nsteps) * sizeof(RectDiagDesc));
        }
        if (grouped) {
            std::vector<SmallMulDesc> sd, vd;
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                const int64_t off = static_cast<int64_t>(i) * bb * bb;
                const int64_t w = si.tail ? si.s : b;
                if (!si.tail && si.s > b) {
                    DView strip = tmat.block(si.r0, si.r0 + b, b, si.s - b);
                    sd.push_back({strip.data, strip.ld, b, si.s - b, Usall.p + off, b, static_cast<int>(b), 0});
                }
                if (vr + si.r0 > 0) {
                    DView X = vt.block(0, si.r0, vr + si.r0, w);
                    vd.push_back({X.data, X.ld, vr + si.r0, w, Vsall.p + off, w, static_cast<int>(w), 0});
                }
            }
            // strips (row blocks) strictly before the column-block right-multiplies
            small_mul_grouped(st, true, sd, GsA.p, gsb);
            small_mul_grouped(st, false, vd, reinterpret_cast<char*>(GsA.p) + gsb, gsb);
        } else {
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                if (si.tail) continue;
                const int64_t off = static_cast<int64_t>(i) * bb * bb;
                DView strip = tmat.block(si.r0, si.r0 + b, b, si.s - b);
                DView tmp(b, si.s - b, b, ZlA.p);
                gemmA(1.0, Op::T, DView(b, b, b, Usall.p + off), Op::N, strip, 0.0, tmp);
                copy_view(st, strip, tmp);
            }
            for (int i = 0; i < nsteps; ++i) {
                const StepInfo& si = plan[static_cast<size_t>(i)];
                const int64_t w = si.tail ? si.s : b;
                if (vr + si.r0 == 0) continue;
                const int64_t off = static_cast<int64_t>(i) * bb * bb;
                DView X = vt.block(0, si.r0, vr + si.r0, w);
                DView tmp(vr + si.r0, w, vr + si.r0, ZxA.p);
                gemmA(1.0, Op::N, X, Op::N, DView(w, w, w, Vsall.p + off), 0.0, tmp);
                copy_view(st, X, tmp);
            }
        }
        if (bu && overlap) wait(st, record(sB));
        prof.mark(P_BETA);
    }

    if (cqr_flag) {  // any unsafe Cholesky-QR2 panel: the caller re-runs with Householder
        int hflag = 0;
        RUTV_CUDA(cudaMemcpyAsync(&hflag, cqr_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        RUTV_CUDA(cudaStreamSynchronize(st));
        if (hflag != 0) {
            static const bool dbg = std::getenv("RUTV_DEBUG") != nullptr;
            if (dbg) std::fprintf(stderr, "[rutv] cholqr flag %d: re-running with Householder panels\n", hflag);
            return false;
        }
    }
    // results out (T rows vr.., V rows 0..n)
    if (!vt_inplace) {
        copy_view(st, DView(n, n, fa.ldt, fa.dT), tmat);
        if (bv && fa.dV) copy_view(st, DView(n, n, fa.ldv, fa.dV), vt.block(0, 0, n, n));
    }
    if (bu && fa.dU && !u_inplace) copy_view(st, DView(n, n, fa.ldu, fa.dU), umat);
    prof.mark(P_FINAL);

    // Jacobi statuses: ConvergenceError surfaces like the reference's exception
    // (the first failing step in step order, as the reference would throw).
    std::vector<double> hs(static_cast<size_t>(4 * ns), 0.0);
    if (nsteps > 0)
        RUTV_CUDA(cudaMemcpyAsync(hs.data(), Jst.p, static_cast<size_t>(4 * nsteps) * 8,
                                  cudaMemcpyDeviceToHost, st));
    RUTV_CUDA(cudaStreamSynchronize(st));
    prof.finish(P_N);
    gemm_profile_end();
    if (prof.on) t_prof_ms = prof.ms;
    for (int k = 0; k < nsteps; ++k)
        if (hs[static_cast<size_t>(4 * k)] == RUTV_ERR_CONVERGENCE)
            throw Error(RUTV_ERR_CONVERGENCE, "jacobi sweeps exhausted after 30 sweeps",
                        hs[static_cast<size_t>(4 * k + 1)]);
    return true;
}

void factorize_device(cudaStream_t st_in, int device, int64_t n, const FactorArgs& fa) {
    NvtxRange range("rutv/factorize");
    if (cholqr_deferred_enabled() && factorize_impl(st_in, device, n, fa, true)) return;
    factorize_impl(st_in, device, n, fa, false);
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
