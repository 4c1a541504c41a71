// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled together with the reference sources
// where they lie under /root/reference/proj/src (recipe: oracle/Makefile) into
// oracle/_ref/librandutv_ref.so, which is git-ignored.  It is used to
// (a) pin the C restatement oracle/rutv_oracle.c bit-for-bit,
// (b) generate the golden fixtures in tests/golden/ (oracle/make_golden.py),
// (c) time the reference CPU path for bench.py --impl reference.
//
// ref_randutv calls randutv::randutv (proj/src/randutv_blocked.cpp:84-157)
// directly.  ref_randutv_steps replays the same loop through the reference's
// public step API (build_v_alpha / apply_q_right / build_u_alpha /
// apply_qt_left / beta_stage, randutv_blocked.hpp:39-72) so it can stop after
// k steps; it reproduces randutv() bit for bit when run to completion
// (checked in tests/test_oracle_pin.py).
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "randutv/errors.hpp"
#include "randutv/householder.hpp"
#include "randutv/jacobi_svd.hpp"
#include "randutv/matrix.hpp"
#include "randutv/matrix_io.hpp"
#include "randutv/matrix_ops.hpp"
#include "randutv/metrics.hpp"
#include "randutv/randutv_ab.hpp"
#include "randutv/randutv_blocked.hpp"
#include "randutv/rng.hpp"

using namespace randutv;

namespace {

int status_of(const std::exception_ptr& p, double* residual) {
    try {
        std::rethrow_exception(p);
    } catch (const ConfigError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const IndexError&) {
        return 3;
    } catch (const ConvergenceError& e) {
        if (residual) *residual = e.residual;
        return 4;
    } catch (const IoError&) {
        return 10;
    } catch (const std::bad_alloc&) {
        return 7;
    } catch (...) {
        return 9;
    }
}

void put(double* dst, const Matrix& m) {
    if (!m.empty())
        std::memcpy(dst, m.data(), sizeof(double) * static_cast<size_t>(m.rows() * m.cols()));
}

void set_block(MatrixView dst, const Matrix& src) { copy_into(dst, src.view()); }

}  // namespace

extern "C" {

int ref_randutv(const double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int q,
                int build_u, int build_v, uint64_t seed, int qr_prepass, double* t, double* u,
                double* v, double* residual) {
    try {
        UTVConfig cfg;
        cfg.b = b;
        cfg.q = q;
        cfg.build_u = build_u != 0;
        cfg.build_v = build_v != 0;
        cfg.seed = seed;
        cfg.qr_prepass = qr_prepass != 0;
        UTVResult r = randutv::randutv(ConstMatrixView(m, n, lda, a), cfg);
        put(t, r.t);
        if (build_u && u) put(u, r.u);
        if (build_v && v) put(v, r.v);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), residual);
    }
}

// Step-limited replica of randutv() over the public step API.  Helpers
// right-multiply / rectangular-diagonal writes are re-expressed with gemm +
// copy_into exactly as randutv_blocked.cpp:17-37 does.
int ref_randutv_steps(const double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int q,
                      int build_u, int build_v, uint64_t seed, int max_steps, double* t, double* u,
                      double* v, double* residual) {
    try {
        if (b < 1 || q < 0) throw ConfigError("bad config");
        Matrix T = to_matrix(ConstMatrixView(m, n, lda, a));
        Matrix U = build_u ? Matrix::identity(m, m) : Matrix();
        Matrix V = build_v ? Matrix::identity(n, n) : Matrix();
        RngState rng(seed);
        auto rmul = [](MatrixView x, const Matrix& mm) {
            if (x.rows == 0 || x.cols == 0) return;
            Matrix tmp(x.rows, mm.cols());
            gemm(1.0, Trans::N, x, Trans::N, mm.view(), 0.0, tmp.view());
            copy_into(x, tmp.view());
        };
        auto rect_diag = [](MatrixView blk, const std::vector<double>& s) {
            const idx p = static_cast<idx>(s.size());
            for (idx j = 0; j < blk.cols; ++j)
                for (idx i = 0; i < blk.rows; ++i)
                    blk(i, j) = (i == j && i < p) ? s[static_cast<size_t>(i)] : 0.0;
        };
        int steps = 0;
        for (idx i = 0;; ++i) {
            const idx r0 = i * b, rr = m - r0, cr = n - r0;
            if (rr <= 0 || cr <= 0) break;
            if (max_steps >= 0 && steps >= max_steps) break;
            ++steps;
            MatrixView t22 = T.view(r0, r0, rr, cr);
            if (cr <= b) {
                SvdTriple s = svd_full(ConstMatrixView(t22));
                rect_diag(t22, s.sigma);
                if (r0 > 0) rmul(T.view(0, r0, r0, cr), s.v);
                if (build_u) rmul(U.view(0, r0, m, rr), s.u);
                if (build_v) rmul(V.view(0, r0, n, cr), s.v);
                break;
            }
            StepTransform sv = build_v_alpha(ConstMatrixView(t22), b, q, rng);
            apply_q_right(sv.qr.view(), sv.twy.view(), t22);
            if (r0 > 0) apply_q_right(sv.qr.view(), sv.twy.view(), T.view(0, r0, r0, cr));
            if (build_v) apply_q_right(sv.qr.view(), sv.twy.view(), V.view(0, r0, n, cr));
            StepTransform su = build_u_alpha(t22.block(0, 0, rr, b));
            apply_qt_left(su.qr.view(), su.twy.view(), t22.block(0, b, rr, cr - b));
            if (build_u) apply_q_right(su.qr.view(), su.twy.view(), U.view(0, r0, m, rr));
            BetaFactors bf = beta_stage(t22, b);
            const idx rt = bf.u.rows();
            if (r0 > 0) rmul(T.view(0, r0, r0, b), bf.v);
            if (build_u) rmul(U.view(0, r0, m, rt), bf.u);
            if (build_v) rmul(V.view(0, r0, n, b), bf.v);
        }
        put(t, T);
        if (build_u && u) put(u, U);
        if (build_v && v) put(v, V);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), residual);
    }
}

void ref_normal_fill(uint64_t seed, uint64_t pos, double* out, int64_t count) {
    RngState r(seed, pos);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next_normal();
}

int ref_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* a) {
    try {
        put(a, gaussian_matrix(m, n, seed));
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

int ref_geometric_matrix(int64_t m, int64_t n, double beta, uint64_t seed, double* a) {
    try {
        put(a, geometric_matrix(m, n, beta, seed));
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

int ref_hqr(const double* a, int64_t m, int64_t n, int64_t lda, double* qr, double* tau,
            double* twy) {
    try {
        HouseholderFactor f = hqr(ConstMatrixView(m, n, lda, a));
        put(qr, f.qr);
        std::memcpy(tau, f.tau.data(), sizeof(double) * f.tau.size());
        Matrix tw = form_wy_t(f.qr.view(), f.tau);
        put(twy, tw);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

int ref_svd_block(const double* a, int64_t n, int64_t lda, double tol, int max_sweeps, double* u,
                  double* sigma, double* v, double* residual) {
    try {
        SvdOptions opt;
        opt.tol = tol;
        opt.max_sweeps = max_sweeps;
        SvdTriple s = svd_block(ConstMatrixView(n, n, lda, a), opt);
        put(u, s.u);
        put(v, s.v);
        std::memcpy(sigma, s.sigma.data(), sizeof(double) * s.sigma.size());
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), residual);
    }
}

int ref_svd_full(const double* a, int64_t m, int64_t n, int64_t lda, double* u, double* sigma,
                 double* v) {
    try {
        SvdTriple s = svd_full(ConstMatrixView(m, n, lda, a));
        put(u, s.u);
        put(v, s.v);
        std::memcpy(sigma, s.sigma.data(), sizeof(double) * s.sigma.size());
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

int ref_gemm(double alpha, int ta, const double* a, int64_t ar, int64_t ac, int64_t lda, int tb,
             const double* b, int64_t br, int64_t bc, int64_t ldb, double beta, double* c,
             int64_t m, int64_t n, int64_t ldc) {
    try {
        gemm(alpha, ta ? Trans::T : Trans::N, ConstMatrixView(ar, ac, lda, a),
             tb ? Trans::T : Trans::N, ConstMatrixView(br, bc, ldb, b), beta,
             MatrixView(m, n, ldc, c));
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

// The reference's multi-threaded algorithm-by-blocks driver (randutv_ab.hpp:46):
// timed as the CPU baseline with every host thread (b must divide m and n).
int ref_randutv_ab(const double* a, int64_t m, int64_t n, int64_t lda, int64_t b, int q, uint64_t seed,
                   int workers, double* t, double* u, double* v, double* residual) {
    try {
        UTVConfig cfg;
        cfg.b = b;
        cfg.q = q;
        cfg.seed = seed;
        UTVResult r = randutv_ab(ConstMatrixView(m, n, lda, a), cfg, workers);
        put(t, r.t);
        if (u) put(u, r.u);
        if (v) put(v, r.v);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), residual);
    }
}

// .rutv I/O (matrix_io.cpp:40-70).  ref_read_rutv: dims when out == nullptr.
int ref_write_rutv(const char* path, const double* a, int64_t m, int64_t n, int64_t lda) {
    try {
        write_rutv(path, ConstMatrixView(m, n, lda, a));
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

int ref_read_rutv(const char* path, int64_t* m, int64_t* n, double* out) {
    try {
        Matrix r = read_rutv(path);
        *m = r.rows();
        *n = r.cols();
        if (out) put(out, r);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

// lowrank_error (metrics.cpp:32-46) with square U (m x m), T (m x n), V (n x n).
int ref_lowrank_error(const double* a, const double* t, const double* u, const double* v, int64_t m, int64_t n,
                      int64_t k, int spectral, double* out) {
    try {
        UTVResult r;
        r.t = to_matrix(ConstMatrixView(m, n, m, t));
        r.u = to_matrix(ConstMatrixView(m, m, m, u));
        r.v = to_matrix(ConstMatrixView(n, n, n, v));
        *out = lowrank_error(ConstMatrixView(m, n, m, a), r, k, spectral ? Norm::Spectral : Norm::Frobenius);
        return 0;
    } catch (...) {
        return status_of(std::current_exception(), nullptr);
    }
}

}  // extern "C"
