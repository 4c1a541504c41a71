/*
 * rutv_b200.h -- C ABI of the B200-native blocked randUTV (librutv_b200.so).
 *
 * Drop-in boundary for the reference's hot path
 *   randutv::UTVResult randutv::randutv(ConstMatrixView a, const UTVConfig& cfg)
 *   (/root/reference/proj/include/randutv/randutv_blocked.hpp:39,
 *    implementation proj/src/randutv_blocked.cpp:84-157)
 * and of the L1 kernels it is built from.  Plain pointers and sizes only; all
 * matrices are column-major FP64, element (i, j) at p[i + j*ld]
 * (proj/include/randutv/matrix.hpp:16-28).  No torch types cross this line.
 *
 * Every entry point returns an int status (rutv_code) and, when `st` is
 * non-NULL, fills it with the code, the Jacobi residual for
 * RUTV_ERR_CONVERGENCE, and a message.  The codes map one-to-one onto the
 * reference's exception classes (proj/include/randutv/errors.hpp:9-50):
 * ConfigError -> RUTV_ERR_CONFIG, ShapeError -> RUTV_ERR_SHAPE,
 * IndexError -> RUTV_ERR_INDEX, ConvergenceError{residual} -> RUTV_ERR_CONVERGENCE,
 * IoError -> RUTV_ERR_IO.
 * The C++ shim (include/randutv_b200/randutv.hpp) rethrows those types.
 */
#ifndef RUTV_B200_H
#define RUTV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RUTV_OK = 0,
    RUTV_ERR_CONFIG = 1,      /* b < 1, q < 0            (randutv_blocked.cpp:10-14) */
    RUTV_ERR_SHAPE = 2,       /* operand shape mismatch  (gemm.cpp:11-17)            */
    RUTV_ERR_INDEX = 3,       /* view out of range       (matrix.hpp:30-36)          */
    RUTV_ERR_CONVERGENCE = 4, /* Jacobi sweep cap hit    (jacobi_svd.cpp:97-109)     */
    RUTV_ERR_CUDA = 5,
    RUTV_ERR_NCCL = 6,
    RUTV_ERR_OOM = 7,
    RUTV_ERR_NOTIMPL = 8,
    RUTV_ERR_INTERNAL = 9,
    RUTV_ERR_IO = 10          /* IoError                 (errors.hpp:36, matrix_io.cpp) */
} rutv_code;

typedef struct {
    int32_t code;
    int32_t reserved;
    double residual; /* ConvergenceError::residual (errors.hpp:29-33) */
    char message[256];
} rutv_status;

/* Mirror of randutv::UTVConfig (randutv_blocked.hpp:11-20) plus device-side knobs. */
typedef struct {
    int64_t b;          /* block size, >= 1 (reference default 128)          */
    int32_t q;          /* power iterations, >= 0 (reference default 1)      */
    int32_t build_u;    /* 0: U is not formed (reference returns 0x0 U)      */
    int32_t build_v;
    int32_t qr_prepass; /* reference qr_prepass (m > n only)                 */
    uint64_t seed;      /* Gaussian sketch stream seed (RngState, rng.hpp:18) */
    int32_t device;     /* CUDA device ordinal                               */
    int32_t max_steps;  /* < 0: run to completion; else stop after k steps   */
    int32_t overlap;    /* 1: off-critical-path updates on a second stream  */
    int32_t reserved0;
    uint64_t stream;    /* cudaStream_t to run on (0: an internal stream)    */
    int32_t grid_p;     /* 2D block-cyclic process grid (block_cyclic.cpp:26-38): grid_p x grid_q  */
    int32_t grid_q;     /* GPUs; 1 x 1 = one GPU.  Host-pointer rutv_b200_factorize only (square). */
    int32_t grid_sim;   /* 1: run the grid's ranks as threads on o->device with an in-process      */
                        /*    exchange instead of NCCL (validation of the sharded path on 1 GPU)   */
    int32_t keep_workspace; /* 1: leave this call's device workspace cached in the library's     */
                            /*    pool (repeated calls of one size skip re-mapping it, e.g. 60 GB */
                            /*    at n = 50000); rutv_b200_release_workspace() returns it.  0:   */
                            /*    trimmed to RUTV_POOL_KEEP_MB (4 GB) when the call returns.      */
} rutv_opts;

/* Return every cached byte of the library's device pool on `device` to the driver. */
int rutv_b200_release_workspace(int device);

#define RUTV_NCCL_ID_BYTES 128

/* Fills the reference defaults: b=128, q=1, build_u=build_v=1, seed=0,
 * device=0, max_steps=-1, overlap=1. */
void rutv_b200_default_opts(rutv_opts* o);

/* Number of Gaussian deviates the blocked driver draws for an m x n input:
 * sum over full steps of rows_rem*b (randutv_blocked.cpp:41-44, 122-139). */
int64_t rutv_b200_stream_length(int64_t m, int64_t n, int64_t b);

/* Algorithmic flop count F(n, b, q) of SURVEY.md section 8(a) (U and V built). */
double rutv_b200_flops(int64_t n, int64_t b, int32_t q);

/*
 * randutv::randutv replacement.  HOST pointers.
 *   A (m x n, lda) is read only.
 *   G: NULL -> the sketch is drawn on the device from RngState(o->seed)
 *      (counter-based, same stream positions as the reference; libm-level
 *      ulp differences possible in log/sin/cos);
 *      non-NULL -> the first g_len deviates of the reference stream, i.e.
 *      G[d] = RngState(seed).normal_at(d); g_len must be >=
 *      rutv_b200_stream_length(m, n, b).  This is the bit-identical parity mode.
 *   T (m x n, ldt), U (m x m, ldu), V (n x n, ldv) are written; U / V may be
 *   NULL when build_u / build_v is 0.
 */
int rutv_b200_factorize(const rutv_opts* o, const double* A, int64_t m, int64_t n, int64_t lda,
                        const double* G, int64_t g_len, double* T, int64_t ldt, double* U,
                        int64_t ldu, double* V, int64_t ldv, rutv_status* st);

/* Same, DEVICE pointers (no host copies; for resident-input benchmarking).
 * A is read only; T/U/V are device buffers on o->device. */
int rutv_b200_factorize_device(const rutv_opts* o, const double* dA, int64_t m, int64_t n,
                               int64_t lda, const double* dG, int64_t g_len, double* dT,
                               int64_t ldt, double* dU, int64_t ldu, double* dV, int64_t ldv,
                               rutv_status* st);

/* Per-phase device timings (ms) of the last factorize call on this thread
 * when RUTV_PROFILE=1; returns the number of phases written (<= cap). */
int rutv_b200_last_profile(const char** names, double* ms, int cap);

/* Kernels this library launched since load (evidence for bench.py). */
uint64_t rutv_b200_launch_count(void);

/* Page-locked host staging buffers of exactly `bytes` (cudaHostAlloc, portable):
 * the host-pointer entry points copy at full PCIe/C2C bandwidth from them. */
int rutv_b200_host_alloc(size_t bytes, void** p, rutv_status* st);
int rutv_b200_host_free(void* p, rutv_status* st);
/* Asynchronous column-major copy of a rows x cols FP64 matrix between any two memory kinds
 * (cudaMemcpy2DAsync, cudaMemcpyDefault) on `stream` (the staging step of host-pointer
 * callers of the DEVICE-pointer entry points, e.g. rutv_b200_factorize_dist). */
int rutv_b200_copy_matrix_async(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                                int64_t cols, uint64_t stream, rutv_status* st);

/* GEMM-kernel totals of the last factorize call on this thread when
 * RUTV_GEMM_PROFILE=1 (CUDA events around every GEMM launch): algorithmic
 * flops (2MNK), device ms, launch count.  Returns 0 when no data. */
int rutv_b200_gemm_profile(double* flops, double* ms, int64_t* launches);

/* ---------------- L1 kernels (DEVICE pointers, stream 0 of o->device) ---------------- */

/* gemm (proj/src/gemm.cpp:21, contract matrix_ops.hpp:9-18):
 * C <- alpha op(A) op(B) + beta C; ta/tb: 0 = N, 1 = T. */
int rutv_b200_gemm(int device, double alpha, int ta, const double* A, int64_t ar, int64_t ac,
                   int64_t lda, int tb, const double* B, int64_t br, int64_t bc, int64_t ldb,
                   double beta, double* C, int64_t m, int64_t n, int64_t ldc, rutv_status* st);

/* hqr_inplace + form_wy_t (householder.cpp:48-97): packed QR of A (m x n) in
 * place, tau[min(m,n)], Twy (p x p, ldt) with p = min(m, n). */
int rutv_b200_hqr(int device, double* A, int64_t m, int64_t n, int64_t lda, double* tau,
                  double* twy, int64_t ldt, rutv_status* st);

/* apply_q_right (householder.cpp:129-140): B (rows x s) <- B Q, Q = I - W Twy W'. */
int rutv_b200_apply_q_right(int device, const double* qr, int64_t s, int64_t ldq,
                            const double* twy, int64_t p, int64_t ldt, double* B, int64_t rows,
                            int64_t ldb, rutv_status* st);
/* apply_qt_left (householder.cpp:103-114): B (s x cols) <- Q' B. */
int rutv_b200_apply_qt_left(int device, const double* qr, int64_t s, int64_t ldq,
                            const double* twy, int64_t p, int64_t ldt, double* B, int64_t cols,
                            int64_t ldb, rutv_status* st);

/* svd_block (jacobi_svd.cpp:39-148): one-sided Jacobi SVD of a square block.
 * U, V n x n (ld n), sigma[n] descending. */
int rutv_b200_svd_block(int device, const double* A, int64_t n, int64_t lda, double tol,
                        int max_sweeps, double* U, double* sigma, double* V, rutv_status* st);

/* generate_normal_random (rng.cpp:44-53): G (rows x cols, ldg) from stream
 * position pos, column-major. */
int rutv_b200_normal_fill(int device, uint64_t seed, uint64_t pos, double* G, int64_t rows,
                          int64_t cols, int64_t ldg, rutv_status* st);

/* ---------------- on-device test-matrix generators (metrics.cpp:90-110) ---------------- */

/* gaussian_matrix: A(i, j) = RngState(seed).normal_at(i + j*m). DEVICE pointer. */
int rutv_b200_gaussian_matrix(int device, int64_t m, int64_t n, uint64_t seed, double* A,
                              int64_t lda, rutv_status* st);

/* geometric_matrix / explicit spectrum: A = Q1 diag(sigma) Q2' with Haar Q1, Q2 built as
 * form_q(hqr(G)) from one RngState(seed) (G1 m x p first, then G2 n x p).
 * sigma: HOST array of min(m, n) values, or NULL for sigma_j = beta^j (accumulated
 * s *= beta as metrics.cpp:103-106 does).  A: DEVICE pointer. */
int rutv_b200_spectrum_matrix(int device, int64_t m, int64_t n, const double* sigma, double beta,
                              uint64_t seed, double* A, int64_t lda, rutv_status* st);

/* ---------------- sharded factorization on a P x Q grid of GPUs ----------------
 * The reference's distributed randUTV is ScaLAPACK over MPI on the 2D
 * block-cyclic layout of block_cyclic.cpp:26-38.  Here: one rank per GPU, T/U/V distributed
 * identically in b x b blocks, block (br, bc) on rank (br mod P)*Q + (bc mod Q), stored at
 * local block (br div P, bc div Q); collectives over NCCL (NVLink).
 *
 * Single process, host buffers: rutv_b200_factorize with o->grid_p * o->grid_q > 1 (one host
 * thread per GPU, devices 0 .. P*Q-1, an NCCL clique) -- the C++ drop-in's
 * UTVConfig{grid_p, grid_q} path.
 * One process per GPU (torchrun / MPI launchers): rank 0 makes an id with
 * rutv_b200_nccl_unique_id, ships it to every rank out of band, every rank calls
 * rutv_b200_dist_create and then rutv_b200_factorize_dist on its local blocks (DEVICE
 * pointers; local shape from rutv_b200_grid_local_shape).  Collective calls: every rank of
 * the grid must make them, in the same order. */
typedef struct rutv_dist_ctx rutv_dist_ctx;
int rutv_b200_grid_local_shape(int64_t n, int64_t b, int P, int Q, int rank, int64_t* rows, int64_t* cols);
/* full (n x n, ldf) <-> rank's local blocks (ldl); any memory kinds (cudaMemcpyDefault). */
int rutv_b200_grid_copy(int device, int64_t n, int64_t b, int P, int Q, int rank, double* full, int64_t ldf,
                        double* loc, int64_t ldl, int to_local, rutv_status* st);
int rutv_b200_nccl_unique_id(unsigned char* id, rutv_status* st);
int rutv_b200_dist_create(const unsigned char* id, int P, int Q, int rank, int device, rutv_dist_ctx** out,
                          rutv_status* st);
int rutv_b200_dist_destroy(rutv_dist_ctx* ctx, rutv_status* st);
/* A_loc (local rows x local cols) is read; T_loc / U_loc / V_loc written (in place, no copies,
 * when V_loc sits directly on top of T_loc: T_loc == V_loc + local rows, ldt == ldv).  G: the
 * full explicit stream on this device (parity mode) or NULL (device RNG, each rank draws its
 * own rows).  o->stream, o->overlap, o->max_steps honoured. */
int rutv_b200_factorize_dist(rutv_dist_ctx* ctx, const rutv_opts* o, int64_t n, const double* A_loc, int64_t lda,
                             const double* G, int64_t g_len, double* T_loc, int64_t ldt, double* U_loc, int64_t ldu,
                             double* V_loc, int64_t ldv, rutv_status* st);

/* RngState(seed).normal_at(d) evaluated on the host (rng.cpp:29-36), bit-identical to
 * the reference's stream; the drop-in header's RngState uses it. */
double rutv_b200_normal_at(uint64_t seed, uint64_t d);

/* ---------------- the reference's public step API (randutv_blocked.hpp:41-72) ----------------
 * One step of the blocked driver, stage by stage (what the reference's own first-k-step
 * harnesses call).  HOST-pointer entries mirror the C++ signatures; the *_device entries
 * take DEVICE pointers and run on `stream` (0: an internal stream).  All synchronous.
 *
 * build_v_alpha (randutv_blocked.cpp:40-55): Y = (T22' T22)^q T22' G, G (rows x b) the
 *   deviates pos .. pos + rows*b of RngState(seed) (or the explicit G, rows x b, ld rows),
 *   Y = QR in place with the house() convention.  Outputs: qr (cols x b, ld cols), tau
 *   (min(cols, b)), twy (p x p, ld p, p = min(cols, b)).  The caller advances its stream
 *   position by rows*b, as the reference's RngState& does.
 * build_u_alpha (randutv_blocked.cpp:57-63): the panel (rows x cols, ld) is factored in
 *   place; qr_copy (rows x cols, ld rows; may be NULL), tau (min), twy (p x p).
 * beta_stage (randutv_blocked.cpp:65-81): t22 (rows x cols, ld) is updated in place;
 *   U (rt x rt, ld rt), V (bw x bw, ld bw), rt = min(rows, bw).  bw outside [1, cols] ->
 *   RUTV_ERR_SHAPE; Jacobi sweep cap -> RUTV_ERR_CONVERGENCE. */
int rutv_b200_build_v_alpha(int device, const double* t22, int64_t rows, int64_t cols, int64_t ld, int64_t b, int q,
                            uint64_t seed, uint64_t pos, const double* G, double* qr, double* tau, double* twy,
                            rutv_status* st);
int rutv_b200_build_u_alpha(int device, double* panel, int64_t rows, int64_t cols, int64_t ld, double* qr_copy,
                            double* tau, double* twy, rutv_status* st);
int rutv_b200_beta_stage(int device, double* t22, int64_t rows, int64_t cols, int64_t ld, int64_t bw, double* U,
                         double* V, rutv_status* st);
int rutv_b200_build_v_alpha_device(int device, uint64_t stream, const double* t22, int64_t rows, int64_t cols,
                                   int64_t ld, int64_t b, int q, uint64_t seed, uint64_t pos, const double* G,
                                   double* qr, double* tau, double* twy, rutv_status* st);
int rutv_b200_build_u_alpha_device(int device, uint64_t stream, double* panel, int64_t rows, int64_t cols,
                                   int64_t ld, double* qr_copy, double* tau, double* twy, rutv_status* st);
int rutv_b200_beta_stage_device(int device, uint64_t stream, double* t22, int64_t rows, int64_t cols, int64_t ld,
                                int64_t bw, double* U, double* V, rutv_status* st);

/* ---------------- asynchronous building blocks (distributed driver) ----------------
 * Enqueue on the calling thread's current stream (rutv_b200_set_stream; 0 =
 * legacy default stream) and return without synchronising.  DEVICE pointers.
 * Used by paper_2104_05782_b200/dist.py to compose a step of
 * randutv_blocked.cpp:122-155 around NCCL collectives. */
void rutv_b200_set_stream(uint64_t stream);
int rutv_b200_gemm_async(double alpha, int ta, const double* A, int64_t ar, int64_t ac, int64_t lda, int tb,
                         const double* B, int64_t br, int64_t bc, int64_t ldb, double beta, double* C, int64_t m,
                         int64_t n, int64_t ldc, rutv_status* st);
/* hqr_inplace (householder.cpp:48-67).  Panels of >= 4608 rows (RUTV_CHOLQR_MIN_ROWS) factor their
 * 128-column sub-panels by Cholesky-QR2 + Householder reconstruction and read one safety flag per
 * sub-panel back from the device, i.e. synchronise the host with the current stream that many
 * times before returning; shorter panels stay fully asynchronous. */
int rutv_b200_hqr_async(double* A, int64_t m, int64_t n, int64_t lda, double* tau, rutv_status* st);
/* W (unit-lower), Twy and M = W Twy' of a packed QR (householder.cpp:37-44, 76-97). */
int rutv_b200_form_wy(const double* qr, int64_t s, int64_t ldq, const double* tau, int64_t p, double* W,
                      int64_t ldw, double* M, int64_t ldm, double* twy, int64_t ldt, rutv_status* st);
int rutv_b200_normal_fill_async(uint64_t seed, uint64_t pos, double* G, int64_t rows, int64_t cols, int64_t ldg,
                                rutv_status* st);
int rutv_b200_copy_async(double* dst, int64_t rows, int64_t cols, int64_t ldd, const double* src, int64_t lds,
                         rutv_status* st);
int rutv_b200_copy_upper_async(double* dst, int64_t rows, int64_t cols, int64_t ldd, const double* src, int64_t lds,
                               rutv_status* st);
int rutv_b200_identity_async(double* a, int64_t rows, int64_t cols, int64_t lda, rutv_status* st);
int rutv_b200_rect_diag_async(double* block, int64_t rows, int64_t cols, int64_t ld, const double* sigma, int64_t p,
                              rutv_status* st);
/* small rows [t*b, t*b+w) <-> big rows [(first + t*stride)*b, ...), t < count; scatter != 0 writes big. */
int rutv_b200_block_rows_async(double* small, int64_t lds_small, double* big, int64_t ld_big, int64_t big_rows,
                               int64_t cols, int64_t b, int64_t first, int64_t stride, int64_t count, int scatter,
                               rutv_status* st);
/* Batched svd_block over count square problems; status = device double[4*count]. */
int rutv_b200_svd_batch_async(int count, const int64_t* n, double* const* A, const int64_t* lda, double* const* U,
                              double* const* sigma, double* const* V, double* status, rutv_status* st);

/* ---------------- data format and quality metrics (io_metrics.cu) ----------------
 * .rutv files (proj/src/matrix_io.cpp:40-70): "RUTV", u64 LE rows, u64 LE cols,
 * column-major binary64 payload, no trailing bytes.  Replace
 * randutv::read_rutv / write_rutv (proj/include/randutv/matrix_io.hpp:12-13);
 * failures are RUTV_ERR_IO with the reference's IoError messages.
 * on_device != 0: `dst` / `src` are DEVICE pointers, streamed through pinned
 * double buffers (disk I/O overlaps the host<->device copies). */
int rutv_b200_rutv_dims(const char* path, int64_t* rows, int64_t* cols, rutv_status* st);
int rutv_b200_read_rutv(const char* path, double* dst, int64_t ld, int on_device, rutv_status* st);
int rutv_b200_write_rutv(const char* path, const double* src, int64_t rows, int64_t cols, int64_t ld, int on_device,
                         rutv_status* st);
/* randutv::lowrank_error (proj/src/metrics.cpp:32-46): ||A - U(:,0:k) T(0:k,:) V'|| of
 * DEVICE matrices, norm 0 = Frobenius (matrix_ops.cpp:9-14), 1 = spectral estimate
 * (matrix_ops.cpp:16-40; max_iter <= 0 selects the reference defaults 100, 1e-10).
 * k outside [0, min(m, n)] -> RUTV_ERR_INDEX.  *out is a HOST double. */
int rutv_b200_lowrank_error(int device, const double* A, int64_t lda, const double* T, int64_t ldt, const double* U,
                            int64_t ldu, const double* V, int64_t ldv, int64_t m, int64_t n, int64_t k, int norm,
                            int max_iter, double tol, double* out, rutv_status* st);

#ifdef __cplusplus
}
#endif

#endif /* RUTV_B200_H */
