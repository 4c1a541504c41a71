// rect.cu -- general m x n randUTV, rectangular dense SVDs, qr_prepass.
//
// The square driver (randutv.cu) is the tuned hot path (stacked V/T buffer,
// three streams, deferred batched beta stage).  Rectangular inputs take this
// straight restatement of randutv::randutv (proj/src/randutv_blocked.cpp:84-157)
// on one stream, built from the same sm_100a kernels:
//
//   per step i: r0 = i b, rows_rem = m - r0, cols_rem = n - r0 (stop when
//   either is <= 0); cols_rem <= b -> one dense svd_full of T22 (:129-137);
//   else sketch G (rows_rem x b, stream position advancing by rows_rem b),
//   Y = T22' G (cols_rem x b), q power steps, QR(Y) -> V-apply on T22,
//   T(0:r0, r0:), V(:, r0:); QR of the panel T22(:, 0:b) with
//   min(rows_rem, b) reflectors -> Qu' on T22(:, b:), U(:, r0:) Qu;
//   beta_stage with rt = min(rows_rem, b) (:66-82) and the right-multiplies.
//
// svd_full (jacobi_svd.cpp:150-193) for an m' x n' block: square -> the
// batched Jacobi kernel; tall -> Householder QR, Jacobi on R, U = Q_e U_R,
// then U completed to m' x m'; wide -> the same on A' with V completed.
// complete_orthonormal (jacobi_svd.cpp:198-240) keeps the reference's
// candidate order (identity columns e_0, e_1, ..., acceptance norm > 0.25,
// then seeded Gaussian candidates with 1e-6): candidates are processed in
// blocks, projected against the existing basis with two GEMM passes
// (classical Gram-Schmidt twice) and then, one CTA, against the vectors
// accepted earlier in the same block -- the reference's two-pass
// modified Gram-Schmidt up to rounding.
//
// qr_prepass (m > n, :88-112): A = Q R, randUTV of R (n x n, the square
// driver), T = [T_R; 0], U = Q diag(U_R, I), V = V_R.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

constexpr int kCandBlock = 128;  // completion candidates per block

__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* a, int64_t lda, double* t,
                                 int64_t ldt) {
    __shared__ double tile[32][33];
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, j0 = static_cast<int64_t>(blockIdx.y) * 32;
    for (int dj = threadIdx.y; dj < 32; dj += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + dj;
        if (i < rows && j < cols) tile[dj][threadIdx.x] = a[i + j * lda];
    }
    __syncthreads();
    for (int di = threadIdx.y; di < 32; di += blockDim.y) {
        const int64_t j = j0 + threadIdx.x, i = i0 + di;  // t(j, i) = a(i, j)
        if (i < rows && j < cols) t[j + i * ldt] = tile[threadIdx.x][di];
    }
}

// dst (p x p) = lower triangle from src's upper: dst(j, i) = src(i, j), i <= j
__global__ void upper_transpose_kernel(int64_t p, const double* src, int64_t lds, double* dst, int64_t ldd) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < p * p;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % p, c = e / p;  // dst(r, c) = src(c, r) if c <= r
        dst[r + c * ldd] = c <= r ? src[c + r * lds] : 0.0;
    }
}

__global__ void identity_cols_kernel(int64_t k, int64_t c0, int nb, double* P, int64_t ldp) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < k * nb;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % k, t = e / k;
        P[i + t * ldp] = i == c0 + t ? 1.0 : 0.0;
    }
}

// One CTA: each candidate column of P, in order, is orthogonalised twice
// against the basis columns accepted from THIS block (Q(:, h0..have)); it is
// accepted when its norm exceeds `accept` (appended to Q, normalised).
__global__ void __launch_bounds__(1024) complete_block_kernel(double* Q, int64_t ldq, int64_t k, int* have_io,
                                                              double* P, int64_t ldp, int nb, double accept) {
    __shared__ double dots[kCandBlock];
    __shared__ double red[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int h0 = *have_io;
    int have = h0;
    for (int t = 0; t < nb && have < k; ++t) {
        double* u = P + static_cast<int64_t>(t) * ldp;
        const int nacc = have - h0;
        for (int pass = 0; pass < 2 && nacc > 0; ++pass) {
            for (int a = warp; a < nacc; a += nw) {
                const double* q = Q + static_cast<int64_t>(h0 + a) * ldq;
                double s = 0.0;
                for (int64_t i = lane; i < k; i += 32) s += q[i] * u[i];
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) dots[a] = s;
            }
            __syncthreads();
            for (int64_t i = tid; i < k; i += blockDim.x) {
                double v = u[i];
                for (int a = 0; a < nacc; ++a) v -= dots[a] * Q[i + static_cast<int64_t>(h0 + a) * ldq];
                u[i] = v;
            }
            __syncthreads();
        }
        double s = 0.0;
        for (int64_t i = tid; i < k; i += blockDim.x) s += u[i] * u[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot += red[w];
        const double nrm = sqrt(tot);
        if (nrm > accept) {
            for (int64_t i = tid; i < k; i += blockDim.x) Q[i + static_cast<int64_t>(have) * ldq] = u[i] / nrm;
            ++have;
        }
        __syncthreads();
    }
    if (tid == 0) *have_io = have;
}

inline int grid1(int64_t total) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 4 * kNumSMs)));
}

void gemm_s(cudaStream_t st, double alpha, Op ta, const DView& a, Op tb, const DView& b, double beta,
            const DView& c) {
    const int64_t k = ta == Op::N ? a.cols : a.rows;
    const int64_t we = gemm_work_elems(c.rows, c.cols, k);
    DevBuf w(we, st);
    gemm(st, alpha, ta, a, tb, b, beta, c, w.p, we);
}

// X <- X M (M square, through a temporary; randutv_blocked.cpp:17-23)
void right_multiply(cudaStream_t st, const DView& x, const DView& mm) {
    if (x.rows == 0 || x.cols == 0) return;
    DevBuf t(x.rows * mm.cols, st);
    DView tv(x.rows, mm.cols, x.rows, t.p);
    gemm_s(st, 1.0, Op::N, x, Op::N, mm, 0.0, tv);
    copy_view(st, x, tv);
}

// X <- M' X (:25-30)
void left_multiply_t(cudaStream_t st, const DView& x, const DView& mm) {
    if (x.rows == 0 || x.cols == 0) return;
    DevBuf t(mm.cols * x.cols, st);
    DView tv(mm.cols, x.cols, mm.cols, t.p);
    gemm_s(st, 1.0, Op::T, mm, Op::N, x, 0.0, tv);
    copy_view(st, x, tv);
}

void transpose(cudaStream_t st, const DView& a, const DView& t) {
    if (a.rows * a.cols == 0) return;
    dim3 grid(static_cast<unsigned>((a.rows + 31) / 32), static_cast<unsigned>((a.cols + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(a.rows, a.cols, a.data, a.ld, t.data, t.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

// Householder QR of a copy of `a` (s x w, s >= w): packed result + tau.
struct QrCopy {
    DevBuf qr, tau;
    int64_t s, w;
    QrCopy(cudaStream_t st, const DView& a) : qr(a.rows * a.cols, st), tau(a.cols + 1, st), s(a.rows), w(a.cols) {
        copy_view(st, view(), a);
        const int64_t hw = hqr_work_elems(s, w);
        DevBuf scr(hw, st);
        hqr_panel(st, view(), tau.p, nullptr, 0, scr.p, hw);
    }
    DView view() const { return DView(s, w, std::max<int64_t>(s, 1), qr.p); }
};

}  // namespace

// Orthonormal completion of q (k x r, first r columns of the k x k buffer q.data / q.ld).
void complete_orthonormal_device(cudaStream_t st, const DView& q, int64_t r) {
    const int64_t k = q.rows;
    if (r >= k) return;
    DevBuf P(k * kCandBlock, st), Z(static_cast<int64_t>(kCandBlock) * k, st);
    int* dhave = nullptr;
    dhave = static_cast<int*>(dev_alloc(sizeof(int), st));
    struct Free {
        int* p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } fr{dhave, st};
    int have = static_cast<int>(r);
    auto project = [&](int nb) {  // P -= Q Q' P, twice (classical Gram-Schmidt, 2 passes)
        if (have == 0) return;
        DView Qv = q.block(0, 0, k, have), Pv(k, nb, k, P.p), Zv(have, nb, have, Z.p);
        for (int pass = 0; pass < 2; ++pass) {
            gemm_s(st, 1.0, Op::T, Qv, Op::N, Pv, 0.0, Zv);
            gemm_s(st, -1.0, Op::N, Qv, Op::N, Zv, 1.0, Pv);
        }
    };
    auto run_block = [&](int nb, double accept) {
        RUTV_CUDA(cudaMemcpyAsync(dhave, &have, sizeof(int), cudaMemcpyHostToDevice, st));
        complete_block_kernel<<<1, 1024, 0, st>>>(q.data, q.ld, k, dhave, P.p, k, nb, accept);
        note_launch();
        RUTV_CHECK_LAUNCH();
        RUTV_CUDA(cudaMemcpyAsync(&have, dhave, sizeof(int), cudaMemcpyDeviceToHost, st));
        RUTV_CUDA(cudaStreamSynchronize(st));
    };
    for (int64_t c0 = 0; c0 < k && have < k; c0 += kCandBlock) {
        const int nb = static_cast<int>(std::min<int64_t>(kCandBlock, k - c0));
        identity_cols_kernel<<<grid1(k * nb), 256, 0, st>>>(k, c0, nb, P.p, k);
        note_launch();
        RUTV_CHECK_LAUNCH();
        project(nb);
        run_block(nb, 0.25);
    }
    // rare fallback: seeded Gaussian candidates (jacobi_svd.cpp:228-236)
    for (int guard = 0; have < k && guard < 1000; ++guard) {
        normal_fill(st, 0xC0317E7Eu, static_cast<uint64_t>(guard) * static_cast<uint64_t>(k), DView(k, 1, k, P.p));
        project(1);
        run_block(1, 1e-6);
    }
    if (have < k) throw Error(RUTV_ERR_INTERNAL, "orthonormal completion failed");
}

// Reference svd_full of a (m' x n'): U (m' x m', ld m'), sigma (min), V (n' x n', ld n').
// Jacobi status doubles (4) at dev_status.
void svd_full_device(cudaStream_t st, const DView& a, double* U, double* sigma, double* V, double* dev_status) {
    const int64_t mr = a.rows, nc = a.cols;
    if (mr == 0 || nc == 0) {
        if (mr) set_identity(st, DView(mr, mr, mr, U));
        if (nc) set_identity(st, DView(nc, nc, nc, V));
        return;
    }
    if (mr == nc) {
        const int64_t we = svd_work_elems(mr, 30) + 16;
        DevBuf w(we, st);
        svd_block(st, a, U, sigma, V, w.p, we, dev_status, 1e-15, 30);
        return;
    }
    const bool tall = mr > nc;
    const int64_t p = std::min(mr, nc), big = std::max(mr, nc);
    // factor the tall orientation: B = A (tall) or A' (wide), B = Q R
    DevBuf Bt(tall ? 1 : nc * mr, st);
    DView Bv = a;
    if (!tall) {
        Bv = DView(nc, mr, nc, Bt.p);
        transpose(st, a, Bv);
    }
    QrCopy f(st, Bv);
    // square core: R (tall) or R' (wide)
    DevBuf Rc(p * p, st), Ui(p * p, st), Vi(p * p, st);
    DView Rv(p, p, p, Rc.p);
    if (tall) {
        copy_upper(st, Rv, f.view().block(0, 0, p, p));
    } else {
        upper_transpose_kernel<<<grid1(p * p), 256, 0, st>>>(p, f.qr.p, f.view().ld, Rc.p, p);
        note_launch();
        RUTV_CHECK_LAUNCH();
    }
    {
        const int64_t we = svd_work_elems(p, 30) + 16;
        DevBuf w(we, st);
        svd_block(st, Rv, Ui.p, sigma, Vi.p, w.p, we, dev_status, 1e-15, 30);
    }
    // Q_e (big x p) times the core's factor on the long side, then complete it
    DevBuf Qe(big * p, st);
    {
        const int64_t fw = form_q_work_elems(big, p);
        DevBuf scr(fw, st);
        form_q(st, f.view(), f.tau.p, p, DView(big, p, big, Qe.p), scr.p, fw);
    }
    double* longf = tall ? U : V;
    double* core = tall ? Ui.p : Vi.p;
    double* shortf = tall ? V : U;
    DView L(big, big, big, longf);
    gemm_s(st, 1.0, Op::N, DView(big, p, big, Qe.p), Op::N, DView(p, p, p, core), 0.0, L.block(0, 0, big, p));
    complete_orthonormal_device(st, L, p);
    copy_view(st, DView(p, p, p, shortf), DView(p, p, p, tall ? Vi.p : Ui.p));
}

void factorize_rect_device(cudaStream_t st, int device, int64_t m, int64_t n, const FactorArgs& fa) {
    (void)device;
    const int64_t b = fa.b;
    const bool bu = fa.build_u, bv = fa.build_v;
    const int64_t ldt = std::max<int64_t>(m, 1);
    DevBuf Tb(m * n, st), Ub(bu ? m * m : 1, st), Vb(bv ? n * n : 1, st);
    DView T(m, n, ldt, Tb.p), Um(m, m, ldt, Ub.p), Vm(n, n, std::max<int64_t>(n, 1), Vb.p);
    copy_view(st, T, DView(m, n, fa.lda, const_cast<double*>(fa.dA)));
    if (bu) set_identity(st, Um);
    if (bv) set_identity(st, Vm);
    int nsvd = 0;
    const int max_svd = static_cast<int>(std::min(m, n) / std::max<int64_t>(b, 1)) + 2;
    DevBuf Jst(4 * max_svd, st);
    RUTV_CUDA(cudaMemsetAsync(Jst.p, 0, static_cast<size_t>(max_svd) * 32, st));
    uint64_t pos = 0;
    int steps = 0;
    for (int64_t i = 0;; ++i) {
        const int64_t r0 = i * b, rr = m - r0, cr = n - r0;
        if (rr <= 0 || cr <= 0) break;
        if (fa.max_steps >= 0 && steps >= fa.max_steps) break;
        ++steps;
        DView t22 = T.block(r0, r0, rr, cr);
        if (cr <= b) {  // dense tail (:129-137)
            DevBuf A2(rr * cr, st), Us(rr * rr, st), Vs(cr * cr, st), sg(std::min(rr, cr) + 1, st);
            DView a2(rr, cr, rr, A2.p);
            copy_view(st, a2, t22);
            svd_full_device(st, a2, Us.p, sg.p, Vs.p, Jst.p + 4 * nsvd++);
            write_rect_diag(st, t22, sg.p, std::min(rr, cr));
            if (r0 > 0) right_multiply(st, T.block(0, r0, r0, cr), DView(cr, cr, cr, Vs.p));
            if (bu) right_multiply(st, Um.block(0, r0, m, rr), DView(rr, rr, rr, Us.p));
            if (bv) right_multiply(st, Vm.block(0, r0, n, cr), DView(cr, cr, cr, Vs.p));
            break;
        }
        // ---- sketch (build_v_alpha, :41-50)
        DevBuf Gb(fa.dG ? 1 : rr * b, st), Yb(cr * b, st), Zb(rr * b, st);
        DView G(rr, b, rr, fa.dG ? const_cast<double*>(fa.dG) + pos : Gb.p);
        if (!fa.dG) normal_fill(st, fa.seed, pos, G);
        pos += static_cast<uint64_t>(rr * b);
        DView Y(cr, b, cr, Yb.p), Z(rr, b, rr, Zb.p);
        gemm_s(st, 1.0, Op::T, t22, Op::N, G, 0.0, Y);
        for (int it = 0; it < fa.q; ++it) {
            gemm_s(st, 1.0, Op::N, t22, Op::N, Y, 0.0, Z);
            gemm_s(st, 1.0, Op::T, t22, Op::N, Z, 0.0, Y);
        }
        // ---- V side: W, Twy, M = W Twy'; B <- B - (B W) M'  (:52-53, :140-143)
        auto wy = [&](const DView& qr, int64_t p, const double* tau, DevBuf& W, DevBuf& M) {
            const int64_t s = qr.rows;
            DevBuf Gm(p * p, st), Tw(p * p, st);
            DView Wv(s, p, s, W.p), Mv(s, p, s, M.p);
            make_w(st, qr, p, Wv);
            gemm_s(st, 1.0, Op::T, Wv, Op::N, Wv, 0.0, DView(p, p, p, Gm.p));
            form_t(st, Gm.p, p, tau, p, Tw.p, p);
            gemm_s(st, 1.0, Op::N, Wv, Op::T, DView(p, p, p, Tw.p), 0.0, Mv);
        };
        DevBuf tv(b + 1, st);
        {
            const int64_t hw = hqr_work_elems(cr, b);
            DevBuf scr(hw, st);
            hqr_panel(st, Y, tv.p, nullptr, 0, scr.p, hw);
        }
        DevBuf Wv(cr * b, st), Mv(cr * b, st);
        wy(Y, b, tv.p, Wv, Mv);
        auto apply_right = [&](const DView& X, const DView& W, const DView& M) {
            if (X.rows == 0 || X.cols == 0) return;
            DevBuf zb(X.rows * W.cols, st);
            DView Zx(X.rows, W.cols, X.rows, zb.p);
            gemm_s(st, 1.0, Op::N, X, Op::N, W, 0.0, Zx);
            gemm_s(st, -1.0, Op::N, Zx, Op::T, M, 1.0, X);
        };
        const DView WvV(cr, b, cr, Wv.p), MvV(cr, b, cr, Mv.p);
        apply_right(t22, WvV, MvV);
        if (r0 > 0) apply_right(T.block(0, r0, r0, cr), WvV, MvV);
        if (bv) apply_right(Vm.block(0, r0, n, cr), WvV, MvV);
        // ---- U side (build_u_alpha, :58-64; :146-148)
        const int64_t pu = std::min(rr, b);
        DView panel = t22.block(0, 0, rr, b);
        DevBuf tu(b + 1, st);
        {
            const int64_t hw = hqr_work_elems(rr, b);
            DevBuf scr(hw, st);
            hqr_panel(st, panel, tu.p, nullptr, 0, scr.p, hw);
        }
        DevBuf Wu(rr * pu, st), Mu(rr * pu, st);
        wy(panel, pu, tu.p, Wu, Mu);
        const DView WuV(rr, pu, rr, Wu.p), MuV(rr, pu, rr, Mu.p);
        {  // Qu' T22(:, b:) = B - M (W' B)
            DView B = t22.block(0, b, rr, cr - b);
            DevBuf zb(pu * (cr - b), st);
            DView Zl(pu, cr - b, pu, zb.p);
            gemm_s(st, 1.0, Op::T, WuV, Op::N, B, 0.0, Zl);
            gemm_s(st, -1.0, Op::N, MuV, Op::N, Zl, 1.0, B);
        }
        if (bu) apply_right(Um.block(0, r0, m, rr), WuV, MuV);
        // ---- beta stage (:66-82, :150-154)
        const int64_t rt = pu;
        DevBuf Rb(rt * b, st), Us(rt * rt, st), Vs(b * b, st), sg(rt + 1, st);
        DView Rv(rt, b, rt, Rb.p);
        copy_upper(st, Rv, t22.block(0, 0, rt, b));
        svd_full_device(st, Rv, Us.p, sg.p, Vs.p, Jst.p + 4 * nsvd++);
        write_rect_diag(st, t22.block(0, 0, rr, b), sg.p, rt);
        left_multiply_t(st, t22.block(0, b, rt, cr - b), DView(rt, rt, rt, Us.p));
        if (r0 > 0) right_multiply(st, T.block(0, r0, r0, b), DView(b, b, b, Vs.p));
        if (bu) right_multiply(st, Um.block(0, r0, m, rt), DView(rt, rt, rt, Us.p));
        if (bv) right_multiply(st, Vm.block(0, r0, n, b), DView(b, b, b, Vs.p));
    }
    copy_view(st, DView(m, n, fa.ldt, fa.dT), T);
    if (bu && fa.dU) copy_view(st, DView(m, m, fa.ldu, fa.dU), Um);
    if (bv && fa.dV) copy_view(st, DView(n, n, fa.ldv, fa.dV), Vm);
    std::vector<double> hs(static_cast<size_t>(4 * max_svd), 0.0);
    RUTV_CUDA(cudaMemcpyAsync(hs.data(), Jst.p, hs.size() * 8, cudaMemcpyDeviceToHost, st));
    RUTV_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < nsvd; ++k)
        if (hs[static_cast<size_t>(4 * k)] == RUTV_ERR_CONVERGENCE)
            throw Error(RUTV_ERR_CONVERGENCE, "jacobi sweeps exhausted after 30 sweeps",
                        hs[static_cast<size_t>(4 * k + 1)]);
}

void factorize_prepass_device(cudaStream_t st, int device, int64_t m, int64_t n, const FactorArgs& fa) {
    // A = Q R (householder.cpp:48-67 via the cluster QR), then the square driver on R
    QrCopy f(st, DView(m, n, fa.lda, const_cast<double*>(fa.dA)));
    DevBuf Rb(n * n, st), Ti(n * n, st), Ui(fa.build_u ? n * n : 1, st), Vi(fa.build_v ? n * n : 1, st);
    DView R(n, n, std::max<int64_t>(n, 1), Rb.p);
    copy_upper(st, R, f.view().block(0, 0, n, n));
    FactorArgs in = fa;
    in.dA = Rb.p;
    in.lda = std::max<int64_t>(n, 1);
    in.dT = Ti.p;
    in.ldt = std::max<int64_t>(n, 1);
    in.dU = fa.build_u ? Ui.p : nullptr;
    in.ldu = std::max<int64_t>(n, 1);
    in.dV = fa.build_v ? fa.dV : nullptr;
    in.ldv = fa.ldv;
    factorize_device(st, device, n, in);
    // T = [T_R; 0]
    DView T(m, n, fa.ldt, fa.dT);
    write_rect_diag(st, T, nullptr, 0);
    copy_view(st, T.block(0, 0, n, n), DView(n, n, std::max<int64_t>(n, 1), Ti.p));
    if (fa.build_u && fa.dU) {  // U = Q diag(U_R, I)
        DView U(m, m, fa.ldu, fa.dU);
        set_identity(st, U);
        copy_view(st, U.block(0, 0, n, n), DView(n, n, std::max<int64_t>(n, 1), Ui.p));
        const int64_t fw = form_q_work_elems(m, m);
        DevBuf scr(fw, st);
        apply_q_left_blocked(st, f.view(), f.tau.p, n, U, scr.p, fw);
    }
    RUTV_CUDA(cudaStreamSynchronize(st));
}

}  // namespace rutv
