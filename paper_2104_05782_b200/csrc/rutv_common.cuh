// rutv_common.cuh -- shared definitions for the B200 randUTV kernels.
//
// All matrices are column-major FP64 with an explicit leading dimension,
// element (i, j) at data[i + j*ld] -- the reference's storage contract
// (proj/include/randutv/matrix.hpp:16-28), kept so device views map 1:1 onto
// the reference's MatrixView sub-blocks.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rutv_b200.h"

namespace rutv {

// NVTX range for profilers (Nsight Systems / ncu --nvtx): free when no tool is attached.
// The factorization marks each step and phase (tracing).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kNumSMs = 148;  // B200; queried at runtime for sizing decisions

// Error carrying a rutv status code; thrown inside the library, mapped to the
// C-ABI status at the boundary (capi.cpp).
struct Error : std::runtime_error {
    int code;
    double residual;
    Error(int c, const std::string& msg, double r = 0.0)
        : std::runtime_error(msg), code(c), residual(r) {}
};

#define RUTV_CUDA(x)                                                                  \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            cudaGetLastError(); /* a failed API call must not poison the next launch check */ \
            throw ::rutv::Error(RUTV_ERR_CUDA, std::string("CUDA error ") +           \
                                                   cudaGetErrorString(e_) + " at " +  \
                                                   __FILE__ + ":" + std::to_string(__LINE__)); \
        }                                                                             \
    } while (0)

#define RUTV_CHECK_LAUNCH() RUTV_CUDA(cudaGetLastError())

// Non-owning device view (mirror of randutv::MatrixView, matrix.hpp:18-38).
struct DView {
    int64_t rows = 0, cols = 0, ld = 1;
    double* data = nullptr;
    DView() = default;
    DView(int64_t r, int64_t c, int64_t l, double* d) : rows(r), cols(c), ld(l), data(d) {}
    __host__ __device__ double* at(int64_t i, int64_t j) const { return data + i + j * ld; }
    DView block(int64_t i0, int64_t j0, int64_t nr, int64_t nc) const {
        if (i0 < 0 || j0 < 0 || nr < 0 || nc < 0 || i0 + nr > rows || j0 + nc > cols)
            throw Error(RUTV_ERR_INDEX, "device subview out of range");
        return DView(nr, nc, ld, data + i0 + j0 * ld);
    }
};

enum class Op { N = 0, T = 1 };

// Stream-ordered allocation from the LIBRARY's per-device pool (runtime.cu;
// never the device's default pool, which the host process owns).  Freed
// blocks stay cached for the rest of a call; pool_trim() at the end of every
// public call returns all but RUTV_POOL_KEEP_MB (default 4096) to the driver.
void* dev_alloc(size_t bytes, cudaStream_t st);
void pool_trim();
void pool_keep_this_call(bool keep);  // skip the trim that ends the current call (keep_workspace)
void pool_release(int device);

struct DevBuf {
    double* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(int64_t elems, cudaStream_t s) : st(s) {
        if (elems <= 0) elems = 1;
        p = static_cast<double*>(dev_alloc(static_cast<size_t>(elems) * 8, s));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

// Largest dynamic shared memory a kernel may request on this device, after its
// static __shared__ usage (cudaDevAttrMaxSharedMemoryPerBlockOptin - static).
inline int dyn_smem_cap(const void* kernel) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) return optin - 1024;
    return optin - static_cast<int>(fa.sharedSizeBytes);
}

// Runs `init` once per (current CUDA device, key), thread-safe.  Kernel
// attributes (dynamic shared-memory opt-in, non-portable cluster sizes) belong
// to a device context, so a process that uses device 0 and then device 1 must
// set them again; concurrent callers block until the first finishes.
void once_per_device(const void* key, const std::function<void()>& init);

// ---- kernels' host launchers (all asynchronous on `stream`) ----

// C <- alpha op(A) op(B) + beta C.  beta == 0 writes C without reading it, so
// stale NaN never leaks (matrix_ops.hpp:9-18).  Deterministic: split-K partials
// are reduced in a fixed order.  `work`/`work_elems` is scratch for split-K.
void gemm(cudaStream_t stream, double alpha, Op ta, const DView& a, Op tb, const DView& b,
          double beta, const DView& c, double* work, int64_t work_elems);
// Scratch (in doubles) the gemm launcher may want for this shape.
int64_t gemm_work_elems(int64_t m, int64_t n, int64_t k);
// Count of kernels launched by this library since process start (bench evidence).
uint64_t launch_count();
void note_launch(int n = 1);
// RUTV_GEMM_PROFILE=1: events around each gemm() between begin and end.
void gemm_profile_begin();
void gemm_profile_end();
int gemm_profile_get(double* flops, double* ms, int64_t* launches);

// G(i, j) = normal_at(seed, pos + i + j*rows)  (proj/src/rng.cpp:29-53).
void normal_fill(cudaStream_t stream, uint64_t seed, uint64_t pos, const DView& g);
// A rank's block-cyclic rows of a step's G (s x cols): g(lr, j) = G((first + (lr/b)*stride)*b
// + lr%b, j) with G(i, j) = normal_at(seed, pos + i + j*s) (rng.cu).
void normal_fill_cyclic(cudaStream_t stream, uint64_t seed, uint64_t pos, int64_t s, int64_t b, int64_t first,
                        int64_t stride, const DView& g);
// small rows [t*b, t*b + w_t) <-> big rows [(first + t*stride)*b, ...), t < count; scatter writes
// big (stream_api.cu) -- row-block gather / scatter of block-cyclic layouts.
void block_rows(cudaStream_t st, double* small, int64_t lds_small, double* big, int64_t ld_big, int64_t big_rows,
                int64_t cols, int64_t b, int64_t first, int64_t stride, int64_t count, bool scatter);

// Small elementwise kernels.
void set_identity(cudaStream_t stream, const DView& a);
void copy_view(cudaStream_t stream, const DView& dst, const DView& src);
// W (rows x p) = unit-lower-trapezoidal reflector matrix of packed QR
// (proj/src/householder.cpp:37-44).
void make_w(cudaStream_t stream, const DView& qr, int64_t p, const DView& w);
// block := rectangular diagonal of sigma, zeros elsewhere (randutv_blocked.cpp:32-37).
void write_rect_diag(cudaStream_t stream, const DView& block, const double* sigma, int64_t p);
// dst (rt x bw) = upper trapezoid of src, zeros below (randutv_blocked.cpp:73-75).
void copy_upper(cudaStream_t stream, const DView& dst, const DView& src);

// Householder panel QR (reference house() convention, householder.cpp:20-67)
// of an s x w panel in place; tau[0..min(s,w)).  `scratch` holds sub-panel
// workspace (see hqr_work_elems).
void hqr_panel(cudaStream_t stream, const DView& a, double* tau, double* twy, int64_t ldt,
               double* scratch, int64_t scratch_elems);
int64_t hqr_work_elems(int64_t s, int64_t w);
// The Householder kernels only (no Cholesky-QR2 fast path).
void hqr_panel_householder(cudaStream_t stream, const DView& a, double* tau, double* scratch,
                           int64_t scratch_elems);
// Twy from the Gram matrix of W and tau (householder.cpp:76-97).
void form_t(cudaStream_t stream, const double* gram, int64_t ldg, const double* tau, int64_t p,
            double* t, int64_t ldt);

// The same for p <= 128 by blocked inversion of diag(1/tau) + striu(G) (cholqr.cu).
void form_t_small(cudaStream_t stream, const double* gram, int64_t ldg, const double* tau, int64_t p,
                  double* t, int64_t ldt);
// Panel QR through Cholesky-QR2 + Householder reconstruction (cholqr.cu); false
// (panel untouched) when the fast path is not applicable or not safe.
bool qr_panel_fast(cudaStream_t stream, const DView& a, double* tau);
// Deferred mode of the fast path (the factorization driver): panels commit
// without a host check and OR their safety flags into *dflag (null: off).
void cholqr_set_deferred(int* dflag);
bool cholqr_deferred_enabled();
// Panels of at least this many rows take the fast path by default, in
// immediate mode: the safety flag is read back after each <= 128-column
// sub-panel (one host synchronisation of the panel's stream) and an unsafe
// sub-panel is redone by the Householder kernels.
bool cholqr_tall(int64_t s);

// One-sided Jacobi SVD of a square block (jacobi_svd.cpp:39-148).  Writes U, sigma, V
// (n x n, ld n).  Status (code, residual, kept, sweeps) is written to
// dev_status[0..3] on the device; the caller checks it after synchronising.
void svd_block(cudaStream_t stream, const DView& a, double* u, double* sigma, double* v,
               double* work, int64_t work_elems, double* dev_status, double tol, int max_sweeps);
// per-problem scratch (V spill + completion candidate); svd_block needs +16 more
int64_t svd_work_elems(int64_t n, int max_sweeps);

// One problem of a batched SVD launch (device-resident array of these).
struct SvdDesc {
    const double* A;
    int64_t lda;
    int n;
    int pad;
    double* U;       // n x n, ld n
    double* sigma;   // n
    double* V;       // n x n, ld n
    double* work;    // svd_work_elems(n) doubles
    double* status;  // 4 doubles: code, residual, kept, sweeps
};
// All problems in one launch (one CTA cluster each); nmax = max n.
void svd_batch(cudaStream_t stream, const SvdDesc* d_descs, int count, int nmax, double tol,
               int max_sweeps);

// Leading ncols columns of Q = H_1...H_p from packed qr (householder.cpp:155-173).
void form_q(cudaStream_t st, const DView& qr, const double* tau, int64_t p, const DView& x,
            double* scratch, int64_t scratch_elems);
int64_t form_q_work_elems(int64_t m, int64_t ncols);
// A = Q1 diag(sigma) Q2' with the reference's Haar construction (metrics.cpp:24-28, 95-110);
// sigma_dev has min(m, n) entries on the device.
void spectrum_matrix(cudaStream_t st, int64_t m, int64_t n, const double* sigma_dev, uint64_t seed,
                     const DView& a);

// Arguments of the single-GPU driver (randutv.cu); all pointers are device.
struct FactorArgs {
    int64_t b;
    int q;
    bool build_u, build_v;
    uint64_t seed;
    int max_steps;
    const double* dA;  // n x n, lda
    int64_t lda;
    const double* dG;  // host-stream G (parity mode) or null (device RNG)
    double* dT;
    int64_t ldt;
    double* dU;        // may be null when !build_u
    int64_t ldu;
    double* dV;        // may be null when !build_v
    int64_t ldv;
    bool overlap = true;  // second stream for the off-critical-path work
};
void factorize_device(cudaStream_t st, int device, int64_t n, const FactorArgs& fa);
// grouped.cu: in-place X_i <- X_i M_i (right) or X_i <- M_i' X_i (left) for many
// small square M_i (w <= small_mul_max_w()) in one launch.
struct SmallMulDesc {
    double* X;
    int64_t ldx;
    int64_t rows, cols;  // right: rows x w; left: w x cols
    const double* M;
    int64_t ldm;
    int w;
    int pad;
};
int small_mul_max_w();
struct RectDiagDesc {
    double* A;
    int64_t rows, cols, ld;
    const double* sigma;
    int64_t p;
};
void rect_diag_grouped(cudaStream_t st, const std::vector<RectDiagDesc>& descs, void* dev_scratch,
                       size_t scratch_bytes);
void small_mul_grouped(cudaStream_t st, bool left, const std::vector<SmallMulDesc>& descs, void* dev_scratch,
                       size_t scratch_bytes);
size_t small_mul_scratch_bytes(size_t ndesc, int64_t total_extent);

// General m x n (rect.cu): the reference loop on one stream, rectangular
// dense SVDs (svd_full) with orthonormal completion; qr_prepass for m > n.
void factorize_rect_device(cudaStream_t st, int device, int64_t m, int64_t n, const FactorArgs& fa);
void factorize_prepass_device(cudaStream_t st, int device, int64_t m, int64_t n, const FactorArgs& fa);
// Reference svd_full (jacobi_svd.cpp:185-192) of an m' x n' block: U m' x m', sigma
// min(m', n'), V n' x n' (ld = their row counts); Jacobi status (4 doubles) at dev_status.
void svd_full_device(cudaStream_t st, const DView& a, double* U, double* sigma, double* V, double* dev_status);
// The public step API (randutv_blocked.hpp:41-72) on device views (step_api.cu).
void build_v_alpha_device(cudaStream_t st, const DView& t22, int64_t b, int q, uint64_t seed, uint64_t pos,
                          const double* dG, double* qr, double* tau, double* twy);
void build_u_alpha_device(cudaStream_t st, const DView& panel, double* qr_copy, double* tau, double* twy);
void beta_stage_device(cudaStream_t st, const DView& t22, int64_t bw, double* U, double* V, double* dev_status);
// The sharded driver over a P x Q grid from HOST buffers (dist.cu; one thread per rank).
void factorize_grid_host(const rutv_opts* o, const double* A, int64_t n, int64_t lda, const double* G, int64_t glen,
                         double* T, int64_t ldt, double* U, int64_t ldu, double* V, int64_t ldv);
// X <- Q X with Q = H_1...H_p from packed qr (householder.cpp:116-127, blocked).
void apply_q_left_blocked(cudaStream_t st, const DView& qr, const double* tau, int64_t p, const DView& x,
                          double* scratch, int64_t scratch_elems);
int last_profile(const char** names, double* ms, int cap);

}  // namespace rutv
