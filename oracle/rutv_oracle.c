/*
 * rutv_oracle.c -- CPU restatement of the reference blocked randUTV path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product (paper_2104_05782_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links, calls or falls back to it.
 *
 * Every function restates one reference function from
 * /root/reference/proj (file:line cited at each definition) in plain C with the
 * reference's exact operation order.  Built with -ffp-contract=off (as the
 * reference is, proj/CMakeLists.txt:17-18) it reproduces the reference bit for
 * bit; tests/test_oracle_pin.py checks that against the compiled reference
 * (oracle/_ref) and against the committed golden vectors in tests/golden/.
 *
 * Storage: column-major doubles, element (i, j) at data[i + j*ld]
 * (proj/include/randutv/matrix.hpp:16-28).
 *
 * Status codes (mirrors include/rutv_b200.h):
 *   0 OK, 1 CONFIG, 2 SHAPE, 3 INDEX, 4 CONVERGENCE, 7 OOM, 9 INTERNAL
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx;

enum { ORA_OK = 0, ORA_CONFIG = 1, ORA_SHAPE = 2, ORA_INDEX = 3, ORA_CONVERGENCE = 4,
       ORA_OOM = 7, ORA_INTERNAL = 9 };

typedef struct {
    idx rows, cols, ld;
    double* data;
} View;

#define AT(v, i, j) ((v).data[(i) + (j) * (v).ld])

static View view_block(View v, idx i0, idx j0, idx nr, idx nc) {
    View out = {nr, nc, v.ld, v.data + i0 + j0 * v.ld};
    return out;
}

/* Owning allocation: zero-filled rows x cols with ld = rows (matrix.hpp:67-73). */
static View mat_new(idx rows, idx cols) {
    View m = {rows, cols, rows > 0 ? rows : 1, NULL};
    size_t cnt = (size_t)(rows > 0 ? rows : 0) * (size_t)(cols > 0 ? cols : 0);
    m.data = (double*)calloc(cnt ? cnt : 1, sizeof(double));
    return m;
}
static void mat_free(View* m) {
    free(m->data);
    m->data = NULL;
}
static View mat_identity(idx rows, idx cols) { /* matrix.hpp:77-82 */
    View m = mat_new(rows, cols);
    idx p = rows < cols ? rows : cols;
    for (idx k = 0; k < p; ++k) AT(m, k, k) = 1.0;
    return m;
}
static void copy_into(View dst, View src) { /* matrix.cpp:11-17 */
    for (idx j = 0; j < dst.cols; ++j)
        for (idx i = 0; i < dst.rows; ++i) AT(dst, i, j) = AT(src, i, j);
}
static View to_matrix(View a) { /* matrix.cpp:5-9 */
    View m = mat_new(a.rows, a.cols);
    copy_into(m, a);
    return m;
}

/* ------------------------------------------------------------------ RNG -- */
/* proj/src/rng.cpp:9-36 : splitmix64-style counter RNG + Box-Muller. */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

static uint64_t mix64(uint64_t z) { /* rng.cpp:11-18 */
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

uint64_t ora_word(uint64_t seed, uint64_t c) { return mix64(seed + (c + 1) * kGolden); } /* rng.cpp:22 */

double ora_uniform(uint64_t seed, uint64_t c) { /* rng.cpp:24-27 */
    return (double)((ora_word(seed, c) >> 11) + 1) * 0x1.0p-53;
}

double ora_normal_at(uint64_t seed, uint64_t d) { /* rng.cpp:29-36 */
    const uint64_t p = d >> 1;
    const double u1 = ora_uniform(seed, 2 * p);
    const double u2 = (double)(ora_word(seed, 2 * p + 1) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    return (d & 1) == 0 ? r * cos(th) : r * sin(th);
}

/* Deviates pos .. pos+count-1 of stream `seed` (generate_normal_random,
 * rng.cpp:44-53, consumes the stream in column-major order). */
void ora_normal_fill(uint64_t seed, uint64_t pos, double* out, idx count) {
    for (idx i = 0; i < count; ++i) out[i] = ora_normal_at(seed, pos + (uint64_t)i);
}

typedef struct {
    uint64_t seed, pos;
} Rng;

static void gen_normal(Rng* rng, View a) { /* rng.cpp:44-47 */
    /* normal_at is a pure function of (seed, position): columns in parallel,
     * same values as the reference's sequential pos++ walk */
    const uint64_t base = rng->pos;
#pragma omp parallel for schedule(static) if (a.rows * a.cols > 65536)
    for (idx j = 0; j < a.cols; ++j)
        for (idx i = 0; i < a.rows; ++i)
            AT(a, i, j) = ora_normal_at(rng->seed, base + (uint64_t)(i + j * a.rows));
    rng->pos = base + (uint64_t)(a.rows * a.cols);
}

/* ----------------------------------------------------------------- GEMM -- */
/* proj/src/gemm.cpp:21-75 with the contract of matrix_ops.hpp:9-18:
 * beta==0 writes exact zeros, then k-ascending accumulation of
 * op(A)(i,k) * fl(alpha * op(B)(k,j)), no FMA. */
static void gemm_v(double alpha, int ta, View a, int tb, View b, double beta, View c) {
    const idx m = c.rows, n = c.cols, kk = ta ? a.rows : a.cols;
    if (beta == 0.0) {
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < m; ++i) AT(c, i, j) = 0.0;
    } else if (beta != 1.0) {
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < m; ++i) AT(c, i, j) *= beta;
    }
    if (alpha == 0.0 || kk == 0) return;
    /* Output columns are independent and each keeps the reference's
     * k-ascending order: OpenMP over j is bit-identical to the serial loop. */
    const int par = (double)m * (double)n * (double)kk > 4e6;
    if (!ta) { /* gemm.cpp:40-55, axpy form */
#pragma omp parallel for schedule(static) if (par)
        for (idx j = 0; j < n; ++j)
            for (idx k = 0; k < kk; ++k) {
                const double t = alpha * (tb ? AT(b, j, k) : AT(b, k, j));
                const double* acol = a.data + k * a.ld;
                double* ccol = c.data + j * c.ld;
                for (idx i = 0; i < m; ++i) ccol[i] += acol[i] * t;
            }
    } else { /* gemm.cpp:56-74, dot form */
#pragma omp parallel for schedule(static) if (par)
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < m; ++i) {
                const double* acol = a.data + i * a.ld;
                double s = AT(c, i, j);
                if (!tb) {
                    const double* bcol = b.data + j * b.ld;
                    for (idx k = 0; k < kk; ++k) s += acol[k] * (alpha * bcol[k]);
                } else {
                    for (idx k = 0; k < kk; ++k) s += acol[k] * (alpha * AT(b, j, k));
                }
                AT(c, i, j) = s;
            }
    }
}

int ora_gemm(double alpha, int ta, const double* A, idx ar, idx ac, idx lda, int tb,
             const double* B, idx br, idx bc, idx ldb, double beta, double* C, idx m, idx n,
             idx ldc) {
    const idx opa_r = ta ? ac : ar, opa_c = ta ? ar : ac;
    const idx opb_r = tb ? bc : br, opb_c = tb ? br : bc;
    if (opa_c != opb_r || m != opa_r || n != opb_c) return ORA_SHAPE; /* gemm.cpp:11-17 */
    View a = {ar, ac, lda, (double*)A}, b = {br, bc, ldb, (double*)B}, c = {m, n, ldc, C};
    gemm_v(alpha, ta, a, tb, b, beta, c);
    return ORA_OK;
}

/* proj/src/matrix_ops.cpp:9-14 */
static double frobenius_norm(View a) {
    double s = 0.0;
    for (idx j = 0; j < a.cols; ++j)
        for (idx i = 0; i < a.rows; ++i) s += AT(a, i, j) * AT(a, i, j);
    return sqrt(s);
}

/* ----------------------------------------------------------- Householder -- */
typedef struct {
    double beta, tau;
} HouseStep;

/* proj/src/householder.cpp:20-34: beta >= 0 always; Parlett head for alpha>=0;
 * tau = 2 (pure sign flip) for a negative head with an all-zero tail. */
static HouseStep house(double alpha, double* tail, idx len, idx stride) {
    double sigma = 0.0;
    for (idx i = 0; i < len; ++i) {
        const double t = tail[i * stride];
        sigma += t * t;
    }
    HouseStep h;
    if (sigma == 0.0) {
        if (alpha >= 0.0) {
            h.beta = alpha;
            h.tau = 0.0;
        } else {
            h.beta = -alpha;
            h.tau = 2.0;
        }
        return h;
    }
    const double beta = sqrt(alpha * alpha + sigma);
    const double head = alpha >= 0.0 ? -sigma / (alpha + beta) : alpha - beta;
    for (idx i = 0; i < len; ++i) tail[i * stride] /= head;
    h.beta = beta;
    h.tau = -head / beta;
    return h;
}

/* proj/src/householder.cpp:48-67; tau has min(m,n) entries. */
static void hqr_inplace(View a, double* tau) {
    const idx m = a.rows, n = a.cols, p = m < n ? m : n;
    for (idx j = 0; j < p; ++j) {
        const idx len = m - j - 1;
        HouseStep h = house(AT(a, j, j), len > 0 ? &AT(a, j + 1, j) : NULL, len, 1);
        AT(a, j, j) = h.beta;
        tau[j] = h.tau;
        if (h.tau == 0.0) continue;
        /* trailing columns are independent (one dot + one axpy each) */
#pragma omp parallel for schedule(static) if ((m - j) * (n - j) > 131072)
        for (idx jj = j + 1; jj < n; ++jj) {
            double w = AT(a, j, jj);
            for (idx i = j + 1; i < m; ++i) w += AT(a, i, j) * AT(a, i, jj);
            w *= h.tau;
            AT(a, j, jj) -= w;
            for (idx i = j + 1; i < m; ++i) AT(a, i, jj) -= w * AT(a, i, j);
        }
    }
}

void ora_hqr_inplace(double* a, idx m, idx n, idx lda, double* tau) {
    View v = {m, n, lda, a};
    hqr_inplace(v, tau);
}

/* proj/src/householder.cpp:76-97: forward recurrence for Twy (p x p, zeroed). */
static void form_wy_t(View qr, const double* tau, idx p, View t) {
    const idx m = qr.rows;
    double* z = (double*)calloc((size_t)(p > 0 ? p : 1), sizeof(double));
    for (idx j = 0; j < p; ++j) {
        const double tj = tau[j];
        for (idx k = 0; k < j; ++k) {
            double s = AT(qr, j, k);
            for (idx i = j + 1; i < m; ++i) s += AT(qr, i, k) * AT(qr, i, j);
            z[k] = s;
        }
        for (idx k = 0; k < j; ++k) {
            double s = 0.0;
            for (idx l = k; l < j; ++l) s += AT(t, k, l) * z[l];
            AT(t, k, j) = -tj * s;
        }
        AT(t, j, j) = tj;
    }
    free(z);
}

void ora_form_wy_t(const double* qr, idx m, idx lda, const double* tau, idx p, double* t) {
    View q = {m, p, lda, (double*)qr}, tv = {p, p, p, t};
    memset(t, 0, sizeof(double) * (size_t)(p * p));
    form_wy_t(q, tau, p, tv);
}

/* proj/src/householder.cpp:37-44: dense unit-lower-trapezoidal W. */
static View make_w(View qr, idx p) {
    View w = mat_new(qr.rows, p);
    for (idx j = 0; j < p; ++j) {
        AT(w, j, j) = 1.0;
        for (idx i = j + 1; i < qr.rows; ++i) AT(w, i, j) = AT(qr, i, j);
    }
    return w;
}

/* householder.cpp:103-114  B <- Q' B = B - W (Twy' (W' B)) */
static void apply_qt_left(View qr, View twy, View b) {
    const idx p = twy.rows;
    if (p == 0 || b.cols == 0) return;
    View w = make_w(qr, p), z = mat_new(p, b.cols), z2 = mat_new(p, b.cols);
    gemm_v(1.0, 1, w, 0, b, 0.0, z);
    gemm_v(1.0, 1, twy, 0, z, 0.0, z2);
    gemm_v(-1.0, 0, w, 0, z2, 1.0, b);
    mat_free(&w); mat_free(&z); mat_free(&z2);
}

/* householder.cpp:116-127  B <- Q B = B - W (Twy (W' B)) */
static void apply_q_left(View qr, View twy, View b) {
    const idx p = twy.rows;
    if (p == 0 || b.cols == 0) return;
    View w = make_w(qr, p), z = mat_new(p, b.cols), z2 = mat_new(p, b.cols);
    gemm_v(1.0, 1, w, 0, b, 0.0, z);
    gemm_v(1.0, 0, twy, 0, z, 0.0, z2);
    gemm_v(-1.0, 0, w, 0, z2, 1.0, b);
    mat_free(&w); mat_free(&z); mat_free(&z2);
}

/* householder.cpp:129-140  B <- B Q = B - ((B W) Twy) W' */
static void apply_q_right(View qr, View twy, View b) {
    const idx p = twy.rows;
    if (p == 0 || b.rows == 0) return;
    View w = make_w(qr, p), z = mat_new(b.rows, p), z2 = mat_new(b.rows, p);
    gemm_v(1.0, 0, b, 0, w, 0.0, z);
    gemm_v(1.0, 0, z, 0, twy, 0.0, z2);
    gemm_v(-1.0, 0, z2, 1, w, 1.0, b);
    mat_free(&w); mat_free(&z); mat_free(&z2);
}

/* Public wrappers for kernel-level parity tests. */
void ora_apply_q_right(const double* qr, idx s, idx ldq, const double* twy, idx p, double* b,
                       idx rows, idx ldb) {
    View q = {s, p, ldq, (double*)qr}, t = {p, p, p, (double*)twy}, bv = {rows, s, ldb, b};
    apply_q_right(q, t, bv);
}
void ora_apply_qt_left(const double* qr, idx s, idx ldq, const double* twy, idx p, double* b,
                       idx cols, idx ldb) {
    View q = {s, p, ldq, (double*)qr}, t = {p, p, p, (double*)twy}, bv = {s, cols, ldb, b};
    apply_qt_left(q, t, bv);
}

/* householder.cpp:155-173: leading ncols columns of Q. */
static View form_q(View qr, const double* tau, idx nref, idx ncols) {
    const idx m = qr.rows;
    View x = mat_identity(m, ncols);
    for (idx j = nref - 1; j >= 0; --j) {
        const double tj = tau[j];
        if (tj == 0.0) continue;
#pragma omp parallel for schedule(static) if ((m - j) * ncols > 131072)
        for (idx c = 0; c < ncols; ++c) {
            double w = AT(x, j, c);
            for (idx i = j + 1; i < m; ++i) w += AT(qr, i, j) * AT(x, i, c);
            w *= tj;
            AT(x, j, c) -= w;
            for (idx i = j + 1; i < m; ++i) AT(x, i, c) -= w * AT(qr, i, j);
        }
    }
    return x;
}

/* ----------------------------------------------------------- Jacobi SVD -- */
typedef struct {
    View u;        /* rows(A) x p or square */
    double* sigma; /* min(m, n) */
    View v;
    double residual;
} Svd;

static void svd_free(Svd* s) {
    mat_free(&s->u);
    mat_free(&s->v);
    free(s->sigma);
    s->sigma = NULL;
}

/* Stable descending order of sig (std::stable_sort in jacobi_svd.cpp:118-122). */
static void stable_sort_desc(idx* perm, const double* sig, idx n) {
    /* insertion sort is stable; n <= a few thousand here */
    for (idx i = 0; i < n; ++i) perm[i] = i;
    for (idx i = 1; i < n; ++i) {
        idx x = perm[i];
        idx k = i - 1;
        while (k >= 0 && sig[x] > sig[perm[k]]) {
            perm[k + 1] = perm[k];
            --k;
        }
        perm[k + 1] = x;
    }
}

/* proj/src/jacobi_svd.cpp:198-240: deterministic orthonormal completion. */
static int try_candidate(View out, idx* have, double* u, const double* cand, double accept) {
    const idx k = out.rows;
    for (idx i = 0; i < k; ++i) u[i] = cand[i];
    for (int pass = 0; pass < 2; ++pass) {
        for (idx j = 0; j < *have; ++j) {
            double dot = 0.0;
            for (idx i = 0; i < k; ++i) dot += AT(out, i, j) * u[i];
            for (idx i = 0; i < k; ++i) u[i] -= dot * AT(out, i, j);
        }
    }
    double nrm = 0.0;
    for (idx i = 0; i < k; ++i) nrm += u[i] * u[i];
    nrm = sqrt(nrm);
    if (nrm <= accept) return 0;
    for (idx i = 0; i < k; ++i) AT(out, i, *have) = u[i] / nrm;
    ++*have;
    return 1;
}

static int complete_orthonormal(View q, View* out_p) {
    const idx k = q.rows, r = q.cols;
    if (r > k) return ORA_SHAPE;
    View out = mat_new(k, k);
    for (idx j = 0; j < r; ++j)
        for (idx i = 0; i < k; ++i) AT(out, i, j) = AT(q, i, j);
    idx have = r;
    double* cand = (double*)calloc((size_t)(k > 0 ? k : 1), sizeof(double));
    double* u = (double*)calloc((size_t)(k > 0 ? k : 1), sizeof(double));
    for (idx c = 0; c < k && have < k; ++c) {
        memset(cand, 0, sizeof(double) * (size_t)k);
        cand[c] = 1.0;
        try_candidate(out, &have, u, cand, 0.25);
    }
    Rng rng = {0xC0317E7Eu, 0};
    for (int guard = 0; have < k && guard < 1000; ++guard) {
        for (idx i = 0; i < k; ++i) cand[i] = ora_normal_at(rng.seed, rng.pos++);
        try_candidate(out, &have, u, cand, 1e-6);
    }
    free(cand);
    free(u);
    if (have < k) {
        mat_free(&out);
        return ORA_INTERNAL;
    }
    *out_p = out;
    return ORA_OK;
}

/* proj/src/jacobi_svd.cpp:39-148: one-sided cyclic Jacobi on a square block. */
static int svd_block(View a, double tol, int max_sweeps, Svd* out) {
    const idx n = a.rows;
    out->residual = 0.0;
    if (a.rows != a.cols) return ORA_SHAPE;
    View b = to_matrix(a);
    View v = mat_identity(n, n);
    const double nf = frobenius_norm(a);
    if (n == 0 || nf == 0.0) {
        out->u = mat_identity(n, n);
        out->sigma = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
        out->v = v;
        mat_free(&b);
        return ORA_OK;
    }
    const double eps = DBL_EPSILON;
    const double rel = tol > sqrt((double)n) * eps ? tol : sqrt((double)n) * eps;
    const double floor_col = 4.0 * (double)n * eps * nf;

    int converged = 0;
    for (int sweep = 0; sweep < max_sweeps && !converged; ++sweep) {
        int rotated = 0;
        for (idx p = 0; p < n - 1; ++p) {
            for (idx q = p + 1; q < n; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0; /* pair_state, jacobi_svd.cpp:24-35 */
                const double* cp = b.data + p * n;
                const double* cq = b.data + q * n;
                for (idx i = 0; i < n; ++i) {
                    al += cp[i] * cp[i];
                    be += cq[i] * cq[i];
                    ga += cp[i] * cq[i];
                }
                const double np = sqrt(al), nq = sqrt(be);
                if (np <= floor_col || nq <= floor_col) continue;
                if (fabs(ga) <= rel * np * nq) continue;
                rotated = 1;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t);
                const double sn = c * t;
                double* bp = b.data + p * n;
                double* bq = b.data + q * n;
                double* vp = v.data + p * n;
                double* vq = v.data + q * n;
                for (idx i = 0; i < n; ++i) {
                    const double x = bp[i], y = bq[i];
                    bp[i] = c * x - sn * y;
                    bq[i] = sn * x + c * y;
                }
                for (idx i = 0; i < n; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - sn * y;
                    vq[i] = sn * x + c * y;
                }
            }
        }
        converged = !rotated;
    }
    if (!converged) { /* jacobi_svd.cpp:97-109 */
        double worst = 0.0;
        for (idx p = 0; p < n - 1; ++p)
            for (idx q = p + 1; q < n; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
                const double* cp = b.data + p * n;
                const double* cq = b.data + q * n;
                for (idx i = 0; i < n; ++i) {
                    al += cp[i] * cp[i];
                    be += cq[i] * cq[i];
                    ga += cp[i] * cq[i];
                }
                const double np = sqrt(al), nq = sqrt(be);
                if (np <= floor_col || nq <= floor_col) continue;
                const double r = fabs(ga) / (np * nq);
                if (r > worst) worst = r;
            }
        out->residual = worst;
        mat_free(&b);
        mat_free(&v);
        return ORA_CONVERGENCE;
    }

    double* sig = (double*)calloc((size_t)n, sizeof(double));
    for (idx j = 0; j < n; ++j) {
        double s = 0.0;
        const double* cj = b.data + j * n;
        for (idx i = 0; i < n; ++i) s += cj[i] * cj[i];
        sig[j] = sqrt(s);
    }
    idx* perm = (idx*)calloc((size_t)n, sizeof(idx));
    stable_sort_desc(perm, sig, n);

    out->u = mat_new(n, n);
    out->v = mat_new(n, n);
    out->sigma = (double*)calloc((size_t)n, sizeof(double));
    idx kept = 0;
    for (idx t = 0; t < n; ++t) {
        const idx j = perm[t];
        const double s = sig[j];
        out->sigma[t] = s;
        for (idx i = 0; i < n; ++i) AT(out->v, i, t) = AT(v, i, j);
        if (s > floor_col) {
            for (idx i = 0; i < n; ++i) AT(out->u, i, t) = AT(b, i, j) / s;
            kept = t + 1;
        }
    }
    int rc = ORA_OK;
    if (kept < n) {
        View filled;
        rc = complete_orthonormal(view_block(out->u, 0, 0, n, kept), &filled);
        if (rc == ORA_OK) {
            for (idx t = kept; t < n; ++t)
                for (idx i = 0; i < n; ++i) AT(out->u, i, t) = AT(filled, i, t);
            mat_free(&filled);
        }
    }
    free(sig);
    free(perm);
    mat_free(&b);
    mat_free(&v);
    return rc;
}

/* proj/src/jacobi_svd.cpp:150-183: economic SVD, QR of the tall side first. */
static int svd_dense(View a, double tol, int max_sweeps, Svd* out) {
    const idx m = a.rows, n = a.cols;
    if (m == n) return svd_block(a, tol, max_sweeps, out);
    if (m > n) {
        View f = to_matrix(a);
        double* tau = (double*)calloc((size_t)n + 1, sizeof(double));
        hqr_inplace(f, tau);
        View r = mat_new(n, n);
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i <= j; ++i) AT(r, i, j) = AT(f, i, j);
        Svd inner;
        int rc = svd_block(r, tol, max_sweeps, &inner);
        mat_free(&r);
        if (rc != ORA_OK) {
            out->residual = inner.residual;
            mat_free(&f);
            free(tau);
            return rc;
        }
        View qe = form_q(f, tau, n, n);
        out->u = mat_new(m, n);
        gemm_v(1.0, 0, qe, 0, inner.u, 0.0, out->u);
        out->sigma = inner.sigma;
        out->v = inner.v;
        out->residual = 0.0;
        mat_free(&inner.u);
        mat_free(&qe);
        mat_free(&f);
        free(tau);
        return ORA_OK;
    }
    View at = mat_new(n, m);
    for (idx j = 0; j < n; ++j)
        for (idx i = 0; i < m; ++i) AT(at, j, i) = AT(a, i, j);
    double* tau = (double*)calloc((size_t)m + 1, sizeof(double));
    hqr_inplace(at, tau);
    View rt = mat_new(m, m);
    for (idx j = 0; j < m; ++j)
        for (idx i = 0; i <= j; ++i) AT(rt, j, i) = AT(at, i, j);
    Svd inner;
    int rc = svd_block(rt, tol, max_sweeps, &inner);
    mat_free(&rt);
    if (rc != ORA_OK) {
        out->residual = inner.residual;
        mat_free(&at);
        free(tau);
        return rc;
    }
    View qe = form_q(at, tau, m, m);
    out->u = inner.u;
    out->sigma = inner.sigma;
    out->v = mat_new(n, m);
    gemm_v(1.0, 0, qe, 0, inner.v, 0.0, out->v);
    out->residual = 0.0;
    mat_free(&inner.v);
    mat_free(&qe);
    mat_free(&at);
    free(tau);
    return ORA_OK;
}

/* proj/src/jacobi_svd.cpp:185-192: full square factors. */
static int svd_full(View a, Svd* out) {
    int rc = svd_dense(a, 1e-15, 30, out);
    if (rc != ORA_OK) return rc;
    if (a.rows > a.cols) {
        View full;
        rc = complete_orthonormal(out->u, &full);
        if (rc != ORA_OK) return rc;
        mat_free(&out->u);
        out->u = full;
    } else if (a.rows < a.cols) {
        View full;
        rc = complete_orthonormal(out->v, &full);
        if (rc != ORA_OK) return rc;
        mat_free(&out->v);
        out->v = full;
    }
    return ORA_OK;
}

/* Square one-sided Jacobi with explicit options; u, v are n x n (ld n). */
int ora_svd_block(const double* a, idx n, idx lda, double tol, int max_sweeps, double* u,
                  double* sigma, double* v, double* residual) {
    View av = {n, n, lda, (double*)a};
    Svd s;
    int rc = svd_block(av, tol, max_sweeps, &s);
    if (residual) *residual = s.residual;
    if (rc != ORA_OK) return rc;
    memcpy(u, s.u.data, sizeof(double) * (size_t)(n * n));
    memcpy(v, s.v.data, sizeof(double) * (size_t)(n * n));
    memcpy(sigma, s.sigma, sizeof(double) * (size_t)n);
    svd_free(&s);
    return ORA_OK;
}

/* svd_full for any m x n: u m x m, sigma min(m,n), v n x n. */
int ora_svd_full(const double* a, idx m, idx n, idx lda, double* u, double* sigma, double* v) {
    View av = {m, n, lda, (double*)a};
    Svd s;
    int rc = svd_full(av, &s);
    if (rc != ORA_OK) return rc;
    const idx p = m < n ? m : n;
    memcpy(u, s.u.data, sizeof(double) * (size_t)(m * m));
    memcpy(v, s.v.data, sizeof(double) * (size_t)(n * n));
    memcpy(sigma, s.sigma, sizeof(double) * (size_t)p);
    svd_free(&s);
    return ORA_OK;
}

/* ------------------------------------------------------- randUTV driver -- */
/* randutv_blocked.cpp:17-23: B <- B * M through a temporary. */
static void right_multiply(View b, View m) {
    if (b.rows == 0 || b.cols == 0) return;
    View tmp = mat_new(b.rows, m.cols);
    gemm_v(1.0, 0, b, 0, m, 0.0, tmp);
    copy_into(b, tmp);
    mat_free(&tmp);
}
/* randutv_blocked.cpp:25-30: B <- M' * B through a temporary. */
static void left_multiply_t(View b, View m) {
    if (b.rows == 0 || b.cols == 0) return;
    View tmp = mat_new(m.cols, b.cols);
    gemm_v(1.0, 1, m, 0, b, 0.0, tmp);
    copy_into(b, tmp);
    mat_free(&tmp);
}
/* randutv_blocked.cpp:32-37 */
static void write_rect_diag(View block, const double* sigma, idx p) {
    for (idx j = 0; j < block.cols; ++j)
        for (idx i = 0; i < block.rows; ++i) AT(block, i, j) = (i == j && i < p) ? sigma[i] : 0.0;
}

/* randutv_blocked.cpp:66-82: beta_stage. On success *bu is rt x rt, *bv bw x bw. */
static int beta_stage(View t22, idx bw, View* bu, View* bv, double* residual) {
    const idx rows22 = t22.rows, cols22 = t22.cols;
    if (bw < 1 || bw > cols22) return ORA_SHAPE;
    const idx rt = rows22 < bw ? rows22 : bw;
    View r = mat_new(rt, bw);
    for (idx j = 0; j < bw; ++j)
        for (idx i = 0; i <= j && i < rt; ++i) AT(r, i, j) = AT(t22, i, j);
    Svd s;
    int rc = svd_full(r, &s);
    mat_free(&r);
    if (rc != ORA_OK) {
        *residual = s.residual;
        return rc;
    }
    write_rect_diag(view_block(t22, 0, 0, rows22, bw), s.sigma, rt < bw ? rt : bw);
    if (cols22 > bw) left_multiply_t(view_block(t22, 0, bw, rt, cols22 - bw), s.u);
    free(s.sigma);
    *bu = s.u;
    *bv = s.v;
    return ORA_OK;
}

/* Total deviates the blocked driver draws: sum over full steps of rows_rem*b. */
int64_t ora_stream_length(idx m, idx n, idx b) {
    int64_t total = 0;
    for (idx i = 0;; ++i) {
        const idx r0 = i * b, rr = m - r0, cr = n - r0;
        if (rr <= 0 || cr <= 0 || cr <= b) break;
        total += rr * b;
    }
    return total;
}

static int randutv_impl(View a, idx b, int q, int build_u, int build_v, uint64_t seed,
                        int qr_prepass, int max_steps, View t, View u, View v, double* residual);

/* randutv_blocked.cpp:84-157.  t (m x n), u (m x m), v (n x n) are caller
 * storage (ld = rows); u / v may be NULL when their build flag is off.
 * max_steps < 0 runs to completion; otherwise stops after that many loop
 * iterations (the final ragged SVD counts as one), giving the reference's
 * exact first-k-step state. */
int ora_randutv(const double* a, idx m, idx n, idx lda, idx b, int q, int build_u, int build_v,
                uint64_t seed, int qr_prepass, int max_steps, double* t, double* u, double* v,
                double* residual) {
    View av = {m, n, lda, (double*)a};
    View tv = {m, n, m > 0 ? m : 1, t};
    View uv = {m, m, m > 0 ? m : 1, u};
    View vv = {n, n, n > 0 ? n : 1, v};
    double res = 0.0;
    int rc = randutv_impl(av, b, q, build_u, build_v, seed, qr_prepass, max_steps, tv, uv, vv,
                          &res);
    if (residual) *residual = res;
    return rc;
}

static int randutv_impl(View a, idx bb, int q, int build_u, int build_v, uint64_t seed,
                        int qr_prepass, int max_steps, View t, View uo, View vo,
                        double* residual) {
    if (bb < 1) return ORA_CONFIG; /* check_config, randutv_blocked.cpp:10-14 */
    if (q < 0) return ORA_CONFIG;
    const idx m = a.rows, n = a.cols;

    if (qr_prepass && m > n) { /* randutv_blocked.cpp:88-112 */
        View f = to_matrix(a);
        double* tau = (double*)calloc((size_t)n + 1, sizeof(double));
        hqr_inplace(f, tau);
        View r = mat_new(n, n);
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i <= j; ++i) AT(r, i, j) = AT(f, i, j);
        View it = mat_new(n, n), iu = mat_new(n, n), iv = mat_new(n, n);
        int rc = randutv_impl(r, bb, q, build_u, build_v, seed, 0, max_steps, it, iu, iv, residual);
        if (rc == ORA_OK) {
            for (idx j = 0; j < n; ++j)
                for (idx i = 0; i < m; ++i) AT(t, i, j) = i < n ? AT(it, i, j) : 0.0;
            if (build_u) {
                View e = mat_identity(m, m);
                for (idx j = 0; j < n; ++j)
                    for (idx i = 0; i < n; ++i) AT(e, i, j) = AT(iu, i, j);
                View twy = mat_new(n, n);
                form_wy_t(f, tau, n, twy);
                apply_q_left(f, twy, e);
                copy_into(uo, e);
                mat_free(&e);
                mat_free(&twy);
            }
            if (build_v) copy_into(vo, iv);
        }
        mat_free(&f); mat_free(&r); mat_free(&it); mat_free(&iu); mat_free(&iv);
        free(tau);
        return rc;
    }

    copy_into(t, a);
    if (build_u) {
        for (idx j = 0; j < m; ++j)
            for (idx i = 0; i < m; ++i) AT(uo, i, j) = i == j ? 1.0 : 0.0;
    }
    if (build_v) {
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < n; ++i) AT(vo, i, j) = i == j ? 1.0 : 0.0;
    }
    Rng rng = {seed, 0};
    int steps = 0;
    for (idx i = 0;; ++i) {
        const idx r0 = i * bb;
        const idx rows_rem = m - r0, cols_rem = n - r0;
        if (rows_rem <= 0 || cols_rem <= 0) break;
        if (max_steps >= 0 && steps >= max_steps) break;
        ++steps;
        View t22 = view_block(t, r0, r0, rows_rem, cols_rem);

        if (cols_rem <= bb) { /* :129-137 ragged tail */
            Svd s;
            int rc = svd_full(t22, &s);
            if (rc != ORA_OK) {
                *residual = s.residual;
                return rc;
            }
            write_rect_diag(t22, s.sigma, rows_rem < cols_rem ? rows_rem : cols_rem);
            if (r0 > 0) right_multiply(view_block(t, 0, r0, r0, cols_rem), s.v);
            if (build_u) right_multiply(view_block(uo, 0, r0, m, rows_rem), s.u);
            if (build_v) right_multiply(view_block(vo, 0, r0, n, cols_rem), s.v);
            svd_free(&s);
            break;
        }

        /* build_v_alpha, randutv_blocked.cpp:41-56 */
        View g = mat_new(rows_rem, bb);
        gen_normal(&rng, g);
        View y = mat_new(cols_rem, bb);
        gemm_v(1.0, 1, t22, 0, g, 0.0, y);
        View z = mat_new(rows_rem, bb);
        for (int it = 0; it < q; ++it) {
            gemm_v(1.0, 0, t22, 0, y, 0.0, z);
            gemm_v(1.0, 1, t22, 0, z, 0.0, y);
        }
        mat_free(&g);
        mat_free(&z);
        const idx pv = cols_rem < bb ? cols_rem : bb;
        double* tauv = (double*)calloc((size_t)pv + 1, sizeof(double));
        hqr_inplace(y, tauv);
        View twyv = mat_new(pv, pv);
        form_wy_t(y, tauv, pv, twyv);

        apply_q_right(y, twyv, t22); /* :140-143 */
        if (r0 > 0) apply_q_right(y, twyv, view_block(t, 0, r0, r0, cols_rem));
        if (build_v) apply_q_right(y, twyv, view_block(vo, 0, r0, n, cols_rem));
        mat_free(&y);
        mat_free(&twyv);
        free(tauv);

        /* build_u_alpha, randutv_blocked.cpp:58-64 */
        const idx bw = bb;
        View panel = view_block(t22, 0, 0, rows_rem, bw);
        const idx pu = rows_rem < bw ? rows_rem : bw;
        double* tauu = (double*)calloc((size_t)pu + 1, sizeof(double));
        hqr_inplace(panel, tauu);
        View twyu = mat_new(pu, pu);
        form_wy_t(panel, tauu, pu, twyu);
        View qru = to_matrix(panel);
        apply_qt_left(qru, twyu, view_block(t22, 0, bw, rows_rem, cols_rem - bw)); /* :147 */
        if (build_u) apply_q_right(qru, twyu, view_block(uo, 0, r0, m, rows_rem)); /* :148 */
        mat_free(&qru);
        mat_free(&twyu);
        free(tauu);

        View bu, bv; /* :150-154 */
        int rc = beta_stage(t22, bw, &bu, &bv, residual);
        if (rc != ORA_OK) return rc;
        const idx rt = bu.rows;
        if (r0 > 0) right_multiply(view_block(t, 0, r0, r0, bw), bv);
        if (build_u) right_multiply(view_block(uo, 0, r0, m, rt), bu);
        if (build_v) right_multiply(view_block(vo, 0, r0, n, bw), bv);
        mat_free(&bu);
        mat_free(&bv);
    }
    return ORA_OK;
}

/* ------------------------------------------------------ test matrices -- */
/* proj/src/metrics.cpp:90-93 */
void ora_gaussian_matrix(idx m, idx n, uint64_t seed, double* a) {
    Rng rng = {seed, 0};
    View av = {m, n, m > 0 ? m : 1, a};
    gen_normal(&rng, av);
}

/* proj/src/metrics.cpp:24-28 random_orthonormal + :95-110 geometric_matrix,
 * generalised to an explicit spectrum sigma[0..p-1] (sigma == NULL means
 * beta^j, accumulated as s *= beta exactly as the reference does). */
int ora_spectrum_matrix(idx m, idx n, double beta, const double* sigma, uint64_t seed, double* a) {
    if (sigma == NULL && !(beta > 0.0)) return ORA_CONFIG;
    const idx p = m < n ? m : n;
    View av = {m, n, m > 0 ? m : 1, a};
    if (p == 0) {
        for (idx j = 0; j < n; ++j)
            for (idx i = 0; i < m; ++i) AT(av, i, j) = 0.0;
        return ORA_OK;
    }
    Rng rng = {seed, 0};
    View g1 = mat_new(m, p);
    gen_normal(&rng, g1);
    double* tau1 = (double*)calloc((size_t)p, sizeof(double));
    hqr_inplace(g1, tau1);
    View u = form_q(g1, tau1, p, p);
    View g2 = mat_new(n, p);
    gen_normal(&rng, g2);
    double* tau2 = (double*)calloc((size_t)p, sizeof(double));
    hqr_inplace(g2, tau2);
    View v = form_q(g2, tau2, p, p);
    double s = 1.0;
    for (idx j = 0; j < p; ++j) {
        const double f = sigma ? sigma[j] : s;
#pragma omp parallel for schedule(static) if (m > 65536)
        for (idx i = 0; i < m; ++i) AT(u, i, j) *= f;
        s *= beta;
    }
    gemm_v(1.0, 0, u, 1, v, 0.0, av);
    mat_free(&g1); mat_free(&g2); mat_free(&u); mat_free(&v);
    free(tau1);
    free(tau2);
    return ORA_OK;
}

int ora_geometric_matrix(idx m, idx n, double beta, uint64_t seed, double* a) {
    return ora_spectrum_matrix(m, n, beta, NULL, seed, a);
}

/* Flop model of SURVEY.md section 8(a): 2MNK per reference gemm call (dense W)
 * plus 2k^2(m - k/3) per Householder QR; U and V built. */
double ora_flops(idx n, idx b, int q) {
    double f = 0.0;
    for (idx i = 0;; ++i) {
        const double r0 = (double)(i * b), s = (double)(n - i * b), bb = (double)b, nn = (double)n;
        if (s <= 0) break;
        if (s <= bb) {
            f += 2 * r0 * s * s + 4 * nn * s * s;
            break;
        }
        f += 2 * s * s * bb * (1 + 2 * q);
        f += 4 * s * s * bb + 2 * s * bb * bb;
        f += 4 * r0 * s * bb + 2 * r0 * bb * bb;
        f += 4 * nn * s * bb + 2 * nn * bb * bb;
        f += 4 * s * bb * (s - bb) + 2 * bb * bb * (s - bb);
        f += 4 * nn * s * bb + 2 * nn * bb * bb;
        f += 2 * bb * bb * (s - bb) + 2 * r0 * bb * bb + 4 * nn * bb * bb;
        f += 2 * 2 * bb * bb * (s - bb / 3);
    }
    return f;
}
