// hqr.cu -- Householder panel QR on a thread-block cluster (sm_100a DSMEM).
//
// Restates hqr_inplace + house (proj/src/householder.cpp:20-67) with the
// reference's convention, which is NOT LAPACK's and is load-bearing for
// parity:
//   sigma = sum(tail^2); sigma == 0 -> (alpha >= 0: beta = alpha, tau = 0)
//                                      (alpha <  0: beta = -alpha, tau = 2)
//   else beta = sqrt(alpha^2 + sigma) >= 0,
//        head = alpha >= 0 ? -sigma/(alpha+beta) : alpha - beta   (Parlett),
//        v_tail = tail/head, tau = -head/beta.
//
// Layout: the s x w panel is split by rows over a cluster of CS CTAs; each CTA
// keeps its row chunk (all w columns) resident in shared memory for the whole
// factorisation.  Per column j there is ONE cluster barrier: every CTA
// computes its partial [sigma, x'a_{j+1}, ..., x'a_{w-1}] (x = unscaled tail
// of column j), all-gathers the partials into every CTA's shared memory over
// DSMEM, and reduces them in rank order (deterministic and identical in every
// CTA).  Then w_k = tau*(a(j,k) + d_k/head) -- algebraically the reference's
// w = tau*(a(j,k) + sum v_i a(i,k)) -- and the rank-1 update is local.
// Panels that do not fit the cluster's shared memory are factored in column
// sub-panels, the trailing columns updated with DMMA GEMMs (blocked
// right-looking, same reflectors).
#include <cooperative_groups.h>

#include <algorithm>

#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kQrThreads = 512;
int kSmemCap = 227 * 1024 - 1024;  // refined at first use (dyn_smem_cap)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kQrThreads, 1)
    hqr_cluster_kernel(double* A, int64_t lda, int s, int w, int p, int R, double* tau) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = static_cast<int>(cluster.num_blocks());
    const int rank = static_cast<int>(cluster.block_rank());
    extern __shared__ __align__(16) double sm[];
    double* chunk = sm;                                  // w * R, column c at chunk[c*R]
    double* msg = chunk + static_cast<size_t>(w) * R;    // [2][CS][w]
    double* hrow = msg + static_cast<size_t>(2) * CS * w;  // [2][w]
    double* red = hrow + static_cast<size_t>(2) * w;     // [w]
    double* wv = red + w;                                // [w]
    __shared__ double s_head, s_tau, s_beta;
    __shared__ int s_scale;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int r_beg = rank * R;
    const int r_cnt = max(0, min(s, r_beg + R) - r_beg);

    for (int idx = tid; idx < w * R; idx += blockDim.x) {
        const int c = idx / R, r = idx % R;
        chunk[idx] = r < r_cnt ? A[(r_beg + r) + static_cast<int64_t>(c) * lda] : 0.0;
    }
    cluster.sync();  // every CTA resident and loaded before any DSMEM traffic

    for (int j = 0; j < p; ++j) {
        const int par = j & 1;
        const int nk = w - j;  // message entries e = 0..nk-1 <-> column j+e (e = 0: sigma)
        const int i0 = max(0, j + 1 - r_beg);
        const double* xc = chunk + static_cast<size_t>(j) * R;

        // (A) partial dots of the unscaled tail x with columns j..w-1
        for (int e = warp; e < nk; e += nwarps) {
            const double* ac = chunk + static_cast<size_t>(j + e) * R;
            double acc = 0.0;
            for (int i = i0 + lane; i < r_cnt; i += 32) acc += xc[i] * ac[i];
            acc = warp_sum(acc);
            if (lane == 0) red[e] = acc;
        }
        __syncthreads();
        // (B) all-gather the partial vector (and, from the owner, row j)
        const bool owner = j >= r_beg && j < r_beg + r_cnt;
        for (int idx = tid; idx < CS * nk; idx += blockDim.x) {
            const int dst = idx / nk, e = idx - dst * nk;
            double* rmsg = cluster.map_shared_rank(msg, dst);
            rmsg[(par * CS + rank) * w + e] = red[e];
            if (owner) {
                double* rh = cluster.map_shared_rank(hrow, dst);
                rh[par * w + e] = chunk[static_cast<size_t>(j + e) * R + (j - r_beg)];
            }
        }
        cluster.sync();
        // (C) reduce in rank order
        for (int e = tid; e < nk; e += blockDim.x) {
            double acc = 0.0;
            for (int r = 0; r < CS; ++r) acc += msg[(par * CS + r) * w + e];
            red[e] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            const double sigma = red[0], alpha = hrow[par * w];
            double beta, tj, head = 1.0;
            int scale = 0;
            if (sigma == 0.0) {
                if (alpha >= 0.0) {
                    beta = alpha;
                    tj = 0.0;
                } else {
                    beta = -alpha;
                    tj = 2.0;
                }
            } else {
                beta = sqrt(alpha * alpha + sigma);
                head = alpha >= 0.0 ? -sigma / (alpha + beta) : alpha - beta;
                tj = -head / beta;
                scale = 1;
            }
            s_beta = beta;
            s_tau = tj;
            s_head = head;
            s_scale = scale;
            if (rank == 0) tau[j] = tj;
        }
        __syncthreads();
        const double head = s_head, tj = s_tau;
        const bool scale = s_scale != 0;
        double* xw = chunk + static_cast<size_t>(j) * R;
        if (scale)
            for (int i = i0 + tid; i < r_cnt; i += blockDim.x) xw[i] /= head;
        for (int e = 1 + tid; e < nk; e += blockDim.x)
            wv[e] = tj * (hrow[par * w + e] + (scale ? red[e] / head : red[e]));
        __syncthreads();
        if (owner && tid == 0) chunk[static_cast<size_t>(j) * R + (j - r_beg)] = s_beta;
        if (owner)
            for (int e = 1 + tid; e < nk; e += blockDim.x)
                chunk[static_cast<size_t>(j + e) * R + (j - r_beg)] -= wv[e];
        if (tj != 0.0) {
            const int rows = r_cnt - i0;
            if (rows > 0) {
                const int total = rows * (nk - 1);
                for (int idx = tid; idx < total; idx += blockDim.x) {
                    const int e = 1 + idx / rows, i = i0 + idx % rows;
                    chunk[static_cast<size_t>(j + e) * R + i] -= wv[e] * xw[i];
                }
            }
        }
        __syncthreads();
    }

    for (int idx = tid; idx < w * R; idx += blockDim.x) {
        const int c = idx / R, r = idx % R;
        if (r < r_cnt) A[(r_beg + r) + static_cast<int64_t>(c) * lda] = chunk[idx];
    }
    cluster.sync();  // no CTA exits while a peer may still write into it
}

size_t cluster_smem_bytes(int w, int R, int cs) {
    return (static_cast<size_t>(w) * R + static_cast<size_t>(2) * cs * w + 4 * static_cast<size_t>(w)) *
           sizeof(double);
}

int g_max_cluster = 0;  // largest cluster size the device accepted (probe once)

int max_cluster() {
    if (g_max_cluster) return g_max_cluster;
    kSmemCap = dyn_smem_cap(reinterpret_cast<const void*>(hqr_cluster_kernel));
    RUTV_CUDA(cudaFuncSetAttribute(hqr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RUTV_CUDA(cudaFuncSetAttribute(hqr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemCap));
    int best = 8;
    for (int cs : {16, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kQrThreads);
        cfg.dynamicSmemBytes = kSmemCap;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = cs;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, hqr_cluster_kernel, &cfg) == cudaSuccess &&
            nclusters > 0) {
            best = cs;
            break;
        }
        cudaGetLastError();
    }
    g_max_cluster = best;
    return best;
}

// Largest column count one cluster launch can hold for s rows.
int cluster_cols_capacity(int64_t s, int cs) {
    const int64_t R = (s + cs - 1) / cs;
    int64_t wmax = (kSmemCap - 1024) / (static_cast<int64_t>(sizeof(double)) * (R + 2 * cs + 4));
    return static_cast<int>(std::max<int64_t>(0, wmax));
}

void launch_cluster(cudaStream_t stream, const DView& a, double* tau) {
    const int s = static_cast<int>(a.rows), w = static_cast<int>(a.cols);
    const int p = std::min(s, w);
    const int cmax = max_cluster();
    // smallest cluster (>= 4 unless tiny) that holds the panel
    int cs = 1;
    const int64_t bytes = static_cast<int64_t>(s) * w * 8;
    while (cs < cmax && (bytes > static_cast<int64_t>(cs) * 120 * 1024 || cs < 4)) cs *= 2;
    if (bytes < 48 * 1024) cs = 1;
    while (cs <= cmax && cluster_cols_capacity(s, cs) < w) cs *= 2;
    if (cs > cmax) throw Error(RUTV_ERR_INTERNAL, "hqr: sub-panel exceeds cluster capacity");
    const int R = (s + cs - 1) / cs;
    const size_t smem = cluster_smem_bytes(w, R, cs);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kQrThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    RUTV_CUDA(cudaLaunchKernelEx(&cfg, hqr_cluster_kernel, a.data, a.ld, s, w, p, R, tau));
    note_launch();
}

}  // namespace

int64_t hqr_work_elems(int64_t s, int64_t w) {
    // W (s x nb) + Gram (nb x nb) + Tsub (nb x nb) + Z, Z2 (nb x w) + gemm split-K scratch
    const int64_t nb = std::min<int64_t>(w, 512);
    return s * nb + 2 * nb * nb + 2 * nb * w + gemm_work_elems(nb, w, s) +
           gemm_work_elems(nb, nb, s) + 1024;
}

void hqr_panel(cudaStream_t stream, const DView& a, double* tau, double* twy, int64_t ldt,
               double* scratch, int64_t scratch_elems) {
    const int64_t s = a.rows, w = a.cols, p = std::min(s, w);
    if (p == 0) return;
    const int cmax = max_cluster();
    const int cap = cluster_cols_capacity(s, cmax);
    if (cap < 1) throw Error(RUTV_ERR_NOTIMPL, "hqr: panel too tall for one cluster");
    if (cap >= w) {
        launch_cluster(stream, a, tau);
    } else {
        // Blocked right-looking: sub-panels of nb columns, trailing update
        // A_trail <- (I - W T W')' A_trail = A_trail - W T' (W' A_trail).
        const int64_t nb = std::max<int64_t>(1, (cap / 8) * 8 > 0 ? (cap / 8) * 8 : cap);
        double* W = scratch;
        double* Gm = W + s * nb;
        double* Ts = Gm + nb * nb;
        double* Z = Ts + nb * nb;
        double* Z2 = Z + nb * w;
        double* gw = Z2 + nb * w;
        const int64_t gw_elems = scratch_elems - (gw - scratch);
        for (int64_t j0 = 0; j0 < p; j0 += nb) {
            const int64_t jb = std::min(nb, p - j0);
            DView sub = a.block(j0, j0, s - j0, jb);
            launch_cluster(stream, sub, tau + j0);
            const int64_t rest = w - j0 - jb;
            if (rest <= 0) continue;
            DView trail = a.block(j0, j0 + jb, s - j0, rest);
            DView Wv(s - j0, jb, s - j0, W);
            make_w(stream, sub, jb, Wv);
            DView Gv(jb, jb, jb, Gm), Tv(jb, jb, jb, Ts);
            gemm(stream, 1.0, Op::T, Wv, Op::N, Wv, 0.0, Gv, gw, gw_elems);
            form_t(stream, Gm, jb, tau + j0, jb, Ts, jb);
            DView Zv(jb, rest, jb, Z), Z2v(jb, rest, jb, Z2);
            gemm(stream, 1.0, Op::T, Wv, Op::N, trail, 0.0, Zv, gw, gw_elems);
            gemm(stream, 1.0, Op::T, Tv, Op::N, Zv, 0.0, Z2v, gw, gw_elems);
            gemm(stream, -1.0, Op::N, Wv, Op::N, Z2v, 1.0, trail, gw, gw_elems);
        }
    }
    if (twy) {
        // Twy of the whole panel: Gram of W then the forward recurrence.
        if (scratch_elems < s * p + p * p) throw Error(RUTV_ERR_INTERNAL, "hqr: scratch too small");
        double* W = scratch;
        double* Gm = W + s * p;
        double* gw = Gm + p * p;
        DView Wv(s, p, s, W), Gv(p, p, p, Gm);
        make_w(stream, a, p, Wv);
        gemm(stream, 1.0, Op::T, Wv, Op::N, Wv, 0.0, Gv, gw, scratch_elems - (gw - scratch));
        form_t(stream, Gm, p, tau, p, twy, ldt);
    }
}

}  // namespace rutv
