// gen.cu -- on-device test-matrix generators.
//
// gaussian_matrix (proj/src/metrics.cpp:90-93): A(i,j) = normal_at(seed, i + j*m).
// geometric_matrix / spectrum matrices (metrics.cpp:24-28, 95-110):
//   U = form_q(hqr(G1), p), V = form_q(hqr(G2), p) with G1 (m x p) drawn
//   first and G2 (n x p) next from one RngState(seed); U(:, j) *= sigma_j;
//   A = U V'.
// Same construction, our kernels: the cluster Householder QR (reference
// convention), a blocked form_q (householder.cpp:155-173 applies H_p..H_1 to
// the identity; here block reflectors of <= 128 columns, last to first), the
// DMMA GEMM.  Bits differ from the CPU generator only through rounding and
// libm ulps in the device RNG, so this is the input path for sizes the CPU
// generator cannot reach (config 4 needs an n = 30000 Haar product).
#include <algorithm>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

__global__ void scale_cols_kernel(int64_t rows, int64_t cols, double* a, int64_t ld, const double* s) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i % rows, c = i / rows;
        a[r + c * ld] *= s[c];
    }
}

}  // namespace

// X (m x ncols) := leading ncols columns of Q = H_1 ... H_p from packed qr (m x p).
void form_q(cudaStream_t st, const DView& qr, const double* tau, int64_t p, const DView& x,
            double* scratch, int64_t scratch_elems) {
    set_identity(st, x);
    apply_q_left_blocked(st, qr, tau, p, x, scratch, scratch_elems);
}

void apply_q_left_blocked(cudaStream_t st, const DView& qr, const double* tau, int64_t p, const DView& x,
                          double* scratch, int64_t scratch_elems) {
    const int64_t m = qr.rows, ncols = x.cols;
    if (p == 0 || ncols == 0) return;
    const int64_t nb = 128;
    double* W = scratch;
    double* Gm = W + m * nb;
    double* Tk = Gm + nb * nb;
    double* Z = Tk + nb * nb;
    double* Z2 = Z + nb * ncols;
    double* gw = Z2 + nb * ncols;
    const int64_t gw_elems = scratch_elems - (gw - scratch);
    if (gw_elems < 0) throw Error(RUTV_ERR_INTERNAL, "form_q scratch too small");
    const int64_t nblk = (p + nb - 1) / nb;
    for (int64_t k = nblk - 1; k >= 0; --k) {
        const int64_t j0 = k * nb, jb = std::min(nb, p - j0), rows = m - j0;
        DView sub = qr.block(j0, j0, rows, jb);
        DView Wv(rows, jb, rows, W), Gv(jb, jb, jb, Gm), Tv(jb, jb, jb, Tk);
        make_w(st, sub, jb, Wv);
        gemm(st, 1.0, Op::T, Wv, Op::N, Wv, 0.0, Gv, gw, gw_elems);
        form_t(st, Gm, jb, tau + j0, jb, Tk, jb);
        DView X = x.block(j0, 0, rows, ncols);
        DView Zv(jb, ncols, jb, Z), Z2v(jb, ncols, jb, Z2);
        gemm(st, 1.0, Op::T, Wv, Op::N, X, 0.0, Zv, gw, gw_elems);
        gemm(st, 1.0, Op::N, Tv, Op::N, Zv, 0.0, Z2v, gw, gw_elems);
        gemm(st, -1.0, Op::N, Wv, Op::N, Z2v, 1.0, X, gw, gw_elems);
    }
}

int64_t form_q_work_elems(int64_t m, int64_t ncols) {
    const int64_t nb = 128;
    return m * nb + 2 * nb * nb + 2 * nb * ncols +
           std::max({gemm_work_elems(nb, nb, m), gemm_work_elems(nb, ncols, m), int64_t(1)}) + 64;
}

void spectrum_matrix(cudaStream_t st, int64_t m, int64_t n, const double* sigma_dev, uint64_t seed,
                     const DView& a) {
    const int64_t p = std::min(m, n);
    if (p == 0) {
        if (m * n > 0) {
            // zeros
            RUTV_CUDA(cudaMemset2DAsync(a.data, static_cast<size_t>(a.ld) * 8, 0, static_cast<size_t>(m) * 8,
                                        static_cast<size_t>(n), st));
        }
        return;
    }
    auto alloc = [&](int64_t elems) {
        double* ptr = nullptr;
        ptr = static_cast<double*>(dev_alloc(static_cast<size_t>(std::max<int64_t>(elems, 1)) * 8, st));
        return ptr;
    };
    double* g1 = alloc(m * p);
    double* g2 = alloc(n * p);
    double* t1 = alloc(p);
    double* t2 = alloc(p);
    double* u = alloc(m * p);
    double* v = alloc(n * p);
    const int64_t hw = std::max(hqr_work_elems(m, p), hqr_work_elems(n, p));
    const int64_t fw = std::max(form_q_work_elems(m, p), form_q_work_elems(n, p));
    const int64_t gwe = std::max<int64_t>(gemm_work_elems(m, n, p), 1);
    double* scr = alloc(std::max({hw, fw, gwe}));
    DView G1(m, p, m, g1), G2(n, p, n, g2), U(m, p, m, u), V(n, p, n, v);
    normal_fill(st, seed, 0, G1);
    normal_fill(st, seed, static_cast<uint64_t>(m * p), G2);
    hqr_panel(st, G1, t1, nullptr, 0, scr, hw);
    form_q(st, G1, t1, p, U, scr, fw);
    hqr_panel(st, G2, t2, nullptr, 0, scr, hw);
    form_q(st, G2, t2, p, V, scr, fw);
    scale_cols_kernel<<<std::max<int64_t>(1, std::min<int64_t>((m * p + 255) / 256, 8 * kNumSMs)), 256, 0, st>>>(
        m, p, u, m, sigma_dev);
    note_launch();
    RUTV_CHECK_LAUNCH();
    gemm(st, 1.0, Op::N, U, Op::T, V, 0.0, a, scr, gwe);
    for (double* ptr : {g1, g2, t1, t2, u, v, scr}) cudaFreeAsync(ptr, st);
}

}  // namespace rutv
