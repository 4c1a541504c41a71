// randutv_b200/randutv.hpp -- C++ drop-in for the reference's blocked randUTV entry point.
//
// The reference (proj/include/randutv/randutv_blocked.hpp:11-39) exposes
//     randutv::UTVResult randutv::randutv(randutv::ConstMatrixView a,
//                                         const randutv::UTVConfig& cfg);
// with column-major Matrix / MatrixView types (proj/include/randutv/matrix.hpp)
// and exceptions derived from randutv::Error (proj/include/randutv/errors.hpp).
// This header restates exactly that surface -- same namespace, type names,
// field names, defaults and exception classes -- and implements randutv() by
// calling the B200 C ABI (include/rutv_b200.h, librutv_b200.so).  A caller
// of the reference recompiles against this header and links
// -lrutv_b200 instead of the reference library; nothing else changes.
//
// Header-only; needs only <rutv_b200.h> and the shared library at link time.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../rutv_b200.h"

namespace randutv {

using idx = std::int64_t;

// ---- errors.hpp:9-50 ----
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct IndexError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct ConvergenceError : Error {
    double residual;
    ConvergenceError(const std::string& msg, double r) : Error(msg), residual(r) {}
};

class Matrix;

// ---- matrix.hpp:18-60: non-owning column-major views, (i, j) at data[i + j*ld] ----
struct MatrixView {
    idx rows = 0, cols = 0, ld = 0;
    double* data = nullptr;
    MatrixView() = default;
    MatrixView(idx r, idx c, idx l, double* d) : rows(r), cols(c), ld(l), data(d) {}
    double& operator()(idx i, idx j) const { return data[i + j * ld]; }
    MatrixView block(idx i0, idx j0, idx nr, idx nc) const {
        if (i0 < 0 || j0 < 0 || nr < 0 || nc < 0 || i0 + nr > rows || j0 + nc > cols)
            throw IndexError("subview out of range");
        return MatrixView(nr, nc, ld, data + i0 + j0 * ld);
    }
};

struct ConstMatrixView {
    idx rows = 0, cols = 0, ld = 0;
    const double* data = nullptr;
    ConstMatrixView() = default;
    ConstMatrixView(idx r, idx c, idx l, const double* d) : rows(r), cols(c), ld(l), data(d) {}
    ConstMatrixView(const MatrixView& v) : rows(v.rows), cols(v.cols), ld(v.ld), data(v.data) {}
    inline ConstMatrixView(const Matrix& m);
    double operator()(idx i, idx j) const { return data[i + j * ld]; }
};

// ---- matrix.hpp:63-118: owning column-major matrix, ld = rows ----
class Matrix {
public:
    Matrix() = default;
    Matrix(idx rows, idx cols) : rows_(rows), cols_(cols) {
        if (rows < 0 || cols < 0) throw ShapeError("negative matrix dimension");
        data_.assign(static_cast<size_t>(rows) * static_cast<size_t>(cols), 0.0);
    }
    static Matrix identity(idx rows, idx cols) {
        Matrix m(rows, cols);
        for (idx k = 0; k < (rows < cols ? rows : cols); ++k) m(k, k) = 1.0;
        return m;
    }
    idx rows() const { return rows_; }
    idx cols() const { return cols_; }
    idx ld() const { return rows_; }
    bool empty() const { return rows_ == 0 || cols_ == 0; }
    double& operator()(idx i, idx j) { return data_[static_cast<size_t>(i + j * rows_)]; }
    double operator()(idx i, idx j) const { return data_[static_cast<size_t>(i + j * rows_)]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    MatrixView view() { return MatrixView(rows_, cols_, rows_, data_.data()); }
    ConstMatrixView view() const { return ConstMatrixView(rows_, cols_, rows_, data_.data()); }

private:
    idx rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

inline ConstMatrixView::ConstMatrixView(const Matrix& m)
    : rows(m.rows()), cols(m.cols()), ld(m.ld()), data(m.data()) {}

// ---- randutv_blocked.hpp:11-31 ----
struct UTVConfig {
    idx b = 128;
    int q = 1;
    bool build_u = true;
    bool build_v = true;
    std::uint64_t seed = 0;
    bool qr_prepass = false;
    int device = 0;  // B200 addition: CUDA device ordinal
    int grid_p = 1;  // B200 addition: shard over a grid_p x grid_q block-cyclic grid of GPUs
    int grid_q = 1;  //   (devices 0 .. grid_p*grid_q - 1, NCCL; square inputs)
};

struct UTVResult {
    Matrix t;
    Matrix u;
    Matrix v;
    UTVConfig config;
};

namespace detail {
inline void rethrow(const rutv_status& st) {
    const std::string msg(st.message);
    switch (st.code) {
        case RUTV_OK: return;
        case RUTV_ERR_CONFIG: throw ConfigError(msg);
        case RUTV_ERR_SHAPE: throw ShapeError(msg);
        case RUTV_ERR_INDEX: throw IndexError(msg);
        case RUTV_ERR_CONVERGENCE: throw ConvergenceError(msg, st.residual);
        default: throw Error("rutv_b200: " + msg);
    }
}
}  // namespace detail

// randutv_blocked.hpp:39 -- A = U T V' on the B200; U / V are 0 x 0 when their
// build flag is off, exactly like the reference.
inline UTVResult randutv(ConstMatrixView a, const UTVConfig& cfg) {
    rutv_opts o;
    rutv_b200_default_opts(&o);
    o.b = cfg.b;
    o.q = cfg.q;
    o.build_u = cfg.build_u ? 1 : 0;
    o.build_v = cfg.build_v ? 1 : 0;
    o.seed = cfg.seed;
    o.qr_prepass = cfg.qr_prepass ? 1 : 0;
    o.device = cfg.device;
    o.grid_p = cfg.grid_p;
    o.grid_q = cfg.grid_q;
    UTVResult r;
    r.config = cfg;
    r.t = Matrix(a.rows, a.cols);
    if (cfg.build_u) r.u = Matrix(a.rows, a.rows);
    if (cfg.build_v) r.v = Matrix(a.cols, a.cols);
    rutv_status st;
    std::memset(&st, 0, sizeof st);
    const idx m = a.rows, n = a.cols;
    rutv_b200_factorize(&o, a.data, m, n, a.ld > 0 ? a.ld : 1, nullptr, 0, r.t.data(), m > 0 ? m : 1,
                        cfg.build_u ? r.u.data() : nullptr, m > 0 ? m : 1,
                        cfg.build_v ? r.v.data() : nullptr, n > 0 ? n : 1, &st);
    detail::rethrow(st);
    return r;
}

// ---- rng.hpp:18-46: counter-based stream, deviate d a pure function of (seed, d) ----
struct RngState {
    std::uint64_t seed = 0;
    std::uint64_t pos = 0;
    explicit RngState(std::uint64_t s = 0, std::uint64_t start = 0) : seed(s), pos(start) {}
    double normal_at(std::uint64_t d) const { return rutv_b200_normal_at(seed, d); }
    double next_normal() { return normal_at(pos++); }
};

// ---- randutv_blocked.hpp:41-72: the public step API ----
struct StepTransform {
    Matrix qr;
    std::vector<double> tau;
    Matrix twy;
};

struct BetaFactors {
    Matrix u;  // rt x rt, rt = min(rows(t22), bw)
    Matrix v;  // bw x bw
};

// Right transform of one step (randutv_blocked.cpp:40-55); consumes rows(t22) * b
// deviates of rng, drawn on the device from the same counter-based stream.
inline StepTransform build_v_alpha(ConstMatrixView t22, idx b, int q, RngState& rng) {
    if (b < 1) throw ConfigError("block size must be >= 1, got " + std::to_string(b));
    if (q < 0) throw ConfigError("power iteration count must be >= 0, got " + std::to_string(q));
    const idx rows = t22.rows, cols = t22.cols, p = cols < b ? cols : b;
    StepTransform r;
    r.qr = Matrix(cols, b);
    r.tau.assign(static_cast<size_t>(p), 0.0);
    r.twy = Matrix(p, p);
    rutv_status st;
    std::memset(&st, 0, sizeof st);
    rutv_b200_build_v_alpha(0, t22.data, rows, cols, t22.ld > 0 ? t22.ld : 1, b, q, rng.seed, rng.pos, nullptr,
                            r.qr.data(), r.tau.data(), r.twy.data(), &st);
    detail::rethrow(st);
    rng.pos += static_cast<std::uint64_t>(rows * b);
    return r;
}

// Left transform of one step (randutv_blocked.cpp:57-63): the panel is factored in place.
inline StepTransform build_u_alpha(MatrixView panel) {
    const idx p = panel.rows < panel.cols ? panel.rows : panel.cols;
    StepTransform r;
    r.qr = Matrix(panel.rows, panel.cols);
    r.tau.assign(static_cast<size_t>(p), 0.0);
    r.twy = Matrix(p, p);
    rutv_status st;
    std::memset(&st, 0, sizeof st);
    rutv_b200_build_u_alpha(0, panel.data, panel.rows, panel.cols, panel.ld > 0 ? panel.ld : 1, r.qr.data(),
                            r.tau.data(), r.twy.data(), &st);
    detail::rethrow(st);
    return r;
}

// Diagonalization stage (randutv_blocked.cpp:65-81), t22 updated in place.
inline BetaFactors beta_stage(MatrixView t22, idx bw) {
    if (bw < 1 || bw > t22.cols)
        throw ShapeError("beta_stage: panel width " + std::to_string(bw) + " against " + std::to_string(t22.cols) +
                         " columns");
    const idx rt = t22.rows < bw ? t22.rows : bw;
    BetaFactors f{Matrix(rt, rt), Matrix(bw, bw)};
    rutv_status st;
    std::memset(&st, 0, sizeof st);
    rutv_b200_beta_stage(0, t22.data, t22.rows, t22.cols, t22.ld > 0 ? t22.ld : 1, bw, f.u.data(), f.v.data(), &st);
    detail::rethrow(st);
    return f;
}

}  // namespace randutv
