// Reference-style caller compiled against the B200 drop-in header.
// Mirrors the reference's own usage (tests/test_randutv_blocked.cpp:40-78):
// factor, then check ||A - U T V'||_F / ||A||_F and U'U = I.
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "randutv_b200/randutv.hpp"

int main() {
    const randutv::idx n = 300;
    randutv::Matrix a(n, n);
    unsigned s = 12345u;
    for (randutv::idx j = 0; j < n; ++j)
        for (randutv::idx i = 0; i < n; ++i) {
            s = s * 1664525u + 1013904223u;
            a(i, j) = (static_cast<double>(s >> 8) / 16777216.0) - 0.5;
        }
    randutv::UTVConfig cfg;
    cfg.b = 64;
    cfg.q = 1;
    cfg.seed = 7;
    randutv::UTVResult r = randutv::randutv(a.view(), cfg);
    // residual
    double num = 0.0, den = 0.0, orth = 0.0;
    for (randutv::idx j = 0; j < n; ++j)
        for (randutv::idx i = 0; i < n; ++i) {
            double usv = 0.0;
            for (randutv::idx k = 0; k < n; ++k) {
                double tv = 0.0;
                for (randutv::idx l = k; l < n; ++l) tv += r.t(k, l) * r.v(j, l);
                usv += r.u(i, k) * tv;
            }
            num += (a(i, j) - usv) * (a(i, j) - usv);
            den += a(i, j) * a(i, j);
        }
    for (randutv::idx j = 0; j < n; ++j)
        for (randutv::idx i = 0; i < n; ++i) {
            double d = 0.0;
            for (randutv::idx k = 0; k < n; ++k) d += r.u(k, i) * r.u(k, j);
            d -= (i == j) ? 1.0 : 0.0;
            orth += d * d;
        }
    const double resid = std::sqrt(num / den), od = std::sqrt(orth);
    bool err_ok = false;
    try {
        randutv::UTVConfig bad = cfg;
        bad.q = -1;
        randutv::randutv(a.view(), bad);
    } catch (const randutv::ConfigError&) {
        err_ok = true;
    }
    // the public step API (randutv_blocked.hpp:41-72): one step by hand
    randutv::RngState rng(cfg.seed);
    randutv::StepTransform sv = randutv::build_v_alpha(a.view(), cfg.b, cfg.q, rng);
    bool step_ok = rng.pos == static_cast<std::uint64_t>(n * cfg.b) && sv.qr.rows() == n &&
                   sv.qr.cols() == cfg.b && sv.twy.rows() == cfg.b && sv.tau.size() == static_cast<size_t>(cfg.b);
    randutv::Matrix panel(n, cfg.b);
    for (randutv::idx j = 0; j < cfg.b; ++j)
        for (randutv::idx i = 0; i < n; ++i) panel(i, j) = a(i, j);
    randutv::StepTransform su = randutv::build_u_alpha(panel.view());
    for (randutv::idx j = 0; j < cfg.b; ++j) step_ok = step_ok && su.qr(j, j) == panel(j, j) && panel(j, j) >= 0.0;
    randutv::Matrix t22(n, n);
    for (randutv::idx j = 0; j < n; ++j)
        for (randutv::idx i = 0; i < n; ++i) t22(i, j) = (j < cfg.b) ? (i <= j ? panel(i, j) : 0.0) : a(i, j);
    randutv::BetaFactors bf = randutv::beta_stage(t22.view(), cfg.b);
    for (randutv::idx j = 0; j < cfg.b; ++j)
        for (randutv::idx i = 0; i < n; ++i)
            step_ok = step_ok && (i == j ? (t22(i, j) >= 0.0 && (j == 0 || t22(j - 1, j - 1) >= t22(i, j)))
                                         : t22(i, j) == 0.0);
    step_ok = step_ok && bf.u.rows() == cfg.b && bf.v.rows() == cfg.b;
    bool shape_err = false;
    try {
        randutv::beta_stage(t22.view(), n + 1);
    } catch (const randutv::ShapeError&) {
        shape_err = true;
    }
    std::printf("shim: resid=%.3e orth=%.3e config_error=%d step_api=%d shape_error=%d\n", resid, od,
                err_ok ? 1 : 0, step_ok ? 1 : 0, shape_err ? 1 : 0);
    return (resid < 1e-13 && od < 1e-12 && err_ok && step_ok && shape_err) ? 0 : 1;
}
