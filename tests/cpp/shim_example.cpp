// Reference-style caller compiled against the B200 drop-in header.
// Mirrors the reference's own usage (tests/test_randutv_blocked.cpp:40-78):
// factor, then check ||A - U T V'||_F / ||A||_F and U'U = I.
#include <cmath>
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
    std::printf("shim: resid=%.3e orth=%.3e config_error=%d\n", resid, od, err_ok ? 1 : 0);
    return (resid < 1e-13 && od < 1e-12 && err_ok) ? 0 : 1;
}
