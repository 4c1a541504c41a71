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
// keeps its row chunk (all w columns, column-major with an odd leading
// dimension so column-strided lane accesses are bank-conflict free) resident
// in shared memory for the whole factorisation.  Per column j:
//   every CTA's partial [sigma_j, x_j'a_{j+1}, ..., x_j'a_{w-1}]
//   (x_j = unscaled tail of column j) and the row owner's row j are
//   all-gathered with st.async remote stores that complete on each
//   receiver's mbarrier (transaction bytes) -- no cluster barrier, no
//   fences, one DSMEM hop per column; every CTA reduces in rank order
//   (identical results everywhere), warp 0 computes house(), and
//   w_k = tau (a(j,k) + d_k / head) -- algebraically the reference's
//   tau (a(j,k) + sum v_i a(i,k)).  Then a row pass scales the reflector (v = x / head, the reference's
//   division) and updates column j+1, and ONE fused pass over the trailing
//   columns applies a_k -= w_k v and, in the same sweep, accumulates the NEXT
//   column's partials x_{j+1}' a_k.  Lanes map to columns and loop over rows
//   (the reflector value is a shared-memory broadcast): no warp reductions in
//   the inner loop.  Reductions are in fixed rank order -> deterministic.
// Panels whose chunk does not fit the cluster's shared memory are factored in
// column sub-panels, the trailing columns updated with DMMA GEMMs (blocked
// right-looking, same reflectors).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "cluster_msg.cuh"
#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kQrThreads = 512;
constexpr int kQrWarps = kQrThreads / 32;
int kSmemCap = 227 * 1024 - 1024;  // refined at first use (dyn_smem_cap)

struct QrSmem {
    double* chunk;  // w columns x LD
    double* msg;    // [2][CS][w] partial vectors, all-gathered with st.async
    double* hrow;   // [2][w] head row (from the row owner)
    double* red;    // [w] reduced entries of the current column / combine scratch
    double* part;   // [16][w] per-row-group partials
    double* hs;     // [4] house scalars: beta, tau, head, scale
    uint64_t* bar;  // [2] mbarriers (one per message parity)
};

__device__ __forceinline__ QrSmem carve(double* sm, int w, int LD, int CS) {
    QrSmem s;
    s.chunk = sm;
    s.msg = s.chunk + static_cast<size_t>(w) * LD;
    s.hrow = s.msg + static_cast<size_t>(2) * CS * w;
    s.red = s.hrow + static_cast<size_t>(2) * w;
    s.part = s.red + w;
    s.hs = s.part + static_cast<size_t>(kQrWarps) * w;
    s.bar = reinterpret_cast<uint64_t*>(s.hs + 4);
    return s;
}

__device__ __forceinline__ int col_groups_log(int nk) {
    const int ncg = (nk + 31) >> 5;  // 32 columns (lanes) per group, rounded up to a power of two
    return ncg <= 1 ? 0 : ncg <= 2 ? 1 : ncg <= 4 ? 2 : ncg <= 8 ? 3 : 4;
}
__device__ __forceinline__ int row_groups(int nk) { return max(1, kQrWarps >> col_groups_log(nk)); }

// Fused pass.  Columns kc in [k0, w) (lanes <-> columns, 32 per column group,
// warps split into column groups x row groups).  When upd0, columns >= kupd
// get a -= w_kc * v_i on rows [iu, rc) (v = chunk column jv), with
// w_kc = tj * (hv[kc] + (scale ? dv[kc] / head : dv[kc])).  Every column's
// dot with the NEXT column (chunk column jn, rows [id, rc), id >= iu) is
// accumulated into part[rg][kc].
__device__ __forceinline__ void fused_pass(const QrSmem& S, int LD, int w, int k0, int kupd, int rc,
                                           bool upd0, int jv, int iu, const double* hv, const double* dv,
                                           double tj, double rh, bool scale, int jn, int id) {
    const int nk = w - k0;
    if (nk <= 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lcg = col_groups_log(nk);
    const int lnrg = max(0, 4 - lcg);  // log2(kQrWarps) = 4
    const int nrg = 1 << lnrg;
    const int rg = warp >> lcg, cg_ = warp & ((1 << lcg) - 1);
    if (rg >= nrg) return;
    const int kc = k0 + cg_ * 32 + lane;
    if (kc >= w) return;
    const bool upd = upd0 && kc >= kupd;
    const int lo = upd0 ? iu : id;
    const int span = max(0, rc - lo);
    const int per = (span + nrg - 1) >> lnrg;
    const int rb = lo + rg * per, re = min(rc, rb + per);
    double* col = S.chunk + static_cast<size_t>(kc) * LD;
    const double* ncol = S.chunk + static_cast<size_t>(jn) * LD;
    double acc0 = 0.0, acc1 = 0.0;
    if (upd) {
        const double* vcol = S.chunk + static_cast<size_t>(jv) * LD;
        const double d = dv[kc];
        const double wk = tj * (hv[kc] + (scale ? d * rh : d));
        int i = rb;
        const int e1 = min(re, id);
        for (; i < e1; ++i) col[i] -= wk * vcol[i];  // rows in [iu, id): update only
        double* cp = col + i;
        const double* vp = vcol + i;
        const double* np = ncol + i;
        const int cntr = re - i;
        int t = 0;
#pragma unroll 1
        for (; t + 3 < cntr; t += 4) {
            const double a0 = cp[t] - wk * vp[t];
            const double a1 = cp[t + 1] - wk * vp[t + 1];
            const double a2 = cp[t + 2] - wk * vp[t + 2];
            const double a3 = cp[t + 3] - wk * vp[t + 3];
            cp[t] = a0;
            cp[t + 1] = a1;
            cp[t + 2] = a2;
            cp[t + 3] = a3;
            acc0 += np[t] * a0 + np[t + 2] * a2;
            acc1 += np[t + 1] * a1 + np[t + 3] * a3;
        }
        for (; t < cntr; ++t) {
            const double a0 = cp[t] - wk * vp[t];
            cp[t] = a0;
            acc0 += np[t] * a0;
        }
    } else {
        int i = max(rb, id);
        for (; i + 3 < re; i += 4) {
            acc0 += ncol[i] * col[i] + ncol[i + 2] * col[i + 2];
            acc1 += ncol[i + 1] * col[i + 1] + ncol[i + 3] * col[i + 3];
        }
        for (; i < re; ++i) acc0 += ncol[i] * col[i];
    }
    S.part[static_cast<size_t>(rg) * w + kc] = acc0 + acc1;
}

__global__ void __launch_bounds__(kQrThreads, 1)
    hqr_cluster_kernel(double* A, int64_t lda, int s, int w, int p, int R, int LD, int lcs, double* tau) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = 1 << lcs;
    const int rank = static_cast<int>(cluster.block_rank());
    extern __shared__ __align__(16) double sm[];
    const QrSmem S = carve(sm, w, LD, CS);
    const int tid = threadIdx.x;
    const int r_beg = rank * R;
    const int rc = max(0, min(s, r_beg + R) - r_beg);  // my row count

    if (rc > 0)
        for (int idx = tid; idx < w * rc; idx += kQrThreads) {
            const int c = idx / rc, i = idx - c * rc;
            S.chunk[static_cast<size_t>(c) * LD + i] = A[(r_beg + i) + static_cast<int64_t>(c) * lda];
        }
    // message bytes for column c: CS partial vectors + the head row, (w - c) entries each
    auto msg_bytes = [&](int c) { return static_cast<uint32_t>((CS + 1) * (w - c) * 8); };
    if (tid == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        if (p > 0) mbar_arm(&S.bar[0], msg_bytes(0));
        if (p > 1) mbar_arm(&S.bar[1], msg_bytes(1));
    }
    cluster.sync();  // every CTA live, barriers initialised, before any remote traffic

    const uint32_t msg_a = smem_u32(S.msg), hrow_a = smem_u32(S.hrow);
    const uint32_t bar_a[2] = {smem_u32(&S.bar[0]), smem_u32(&S.bar[1])};

    // All-gather of column jn's partials (and the row owner's row jn) into
    // every CTA's msg/hrow slot of parity jn & 1, counted on its mbarrier.
    auto send = [&](int jn) {
        const int nk = w - jn, par = jn & 1;
        const int nrg = row_groups(nk);
        for (int e = tid; e < nk; e += kQrThreads) {
            double v = 0.0;
            for (int g = 0; g < nrg; ++g) v += S.part[static_cast<size_t>(g) * w + jn + e];
            S.red[e] = v;
        }
        __syncthreads();
        const bool owner = jn >= r_beg && jn < r_beg + rc;
        const int jl = jn - r_beg;
        for (int e = tid; e < nk; e += kQrThreads) {
            const double v = S.red[e];
            const double h = owner ? S.chunk[static_cast<size_t>(jn + e) * LD + jl] : 0.0;
            const uint32_t moff = msg_a + static_cast<uint32_t>(((par * CS + rank) * w + e) * 8);
            const uint32_t hoff = hrow_a + static_cast<uint32_t>((par * w + e) * 8);
            for (int dst = 0; dst < CS; ++dst) {
                const uint32_t rbar = mapa_u32(bar_a[par], dst);
                st_async_f64(mapa_u32(moff, dst), v, rbar);
                if (owner) st_async_f64(mapa_u32(hoff, dst), h, rbar);
            }
        }
    };

    if (p > 0) {  // initial partials for column 0 (dots over rows > 0)
        fused_pass(S, LD, w, 0, w, rc, false, 0, 0, nullptr, nullptr, 0.0, 1.0, false, 0, max(0, 1 - r_beg));
        __syncthreads();
        send(0);
    }

    for (int j = 0; j < p; ++j) {
        const int nk = w - j, par = j & 1;
        mbar_wait(&S.bar[par], static_cast<uint32_t>((j >> 1) & 1));
        const double* msgp = S.msg + static_cast<size_t>(par) * CS * w;
        const double* hv = S.hrow + static_cast<size_t>(par) * w;  // hv[e] = a(j, j+e)
        if (tid < 32) {  // house() scalars (householder.cpp:20-34), one warp
            double sigma = 0.0;
            for (int r = 0; r < CS; ++r) sigma += msgp[static_cast<size_t>(r) * w];
            const double alpha = hv[0];
            double beta, tj, head = 1.0, scale = 0.0;
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
                scale = 1.0;
            }
            if (tid == 0) {
                S.hs[0] = beta;
                S.hs[1] = tj;
                S.hs[2] = head;
                S.hs[3] = scale;
                if (rank == 0) tau[j] = tj;
                if (j + 2 < p) mbar_arm(&S.bar[par], msg_bytes(j + 2));  // next use of this slot
            }
        } else {
            for (int e = tid - 32 + 1; e < nk; e += kQrThreads - 32) {  // reduce d_{j+e} in rank order
                double d = 0.0;
                for (int r = 0; r < CS; ++r) d += msgp[static_cast<size_t>(r) * w + e];
                S.red[e] = d;
            }
        }
        __syncthreads();
        const double beta = S.hs[0], tj = S.hs[1], head = S.hs[2];
        const bool scale = S.hs[3] != 0.0;
        const double rh = 1.0 / head;  // w_k uses d_k * (1/head); v keeps the reference's division
        // row pass: scale the reflector, update column j+1 (rows > j) and row j
        const int iu = max(0, j + 1 - r_beg);
        double* xj = S.chunk + static_cast<size_t>(j) * LD;
        double* xn = S.chunk + static_cast<size_t>(j + 1) * LD;
        const bool upd_next = nk > 1 && tj != 0.0;
        const double w1 = nk > 1 ? tj * (hv[1] + (scale ? S.red[1] * rh : S.red[1])) : 0.0;
        for (int i = iu + tid; i < rc; i += kQrThreads) {
            const double v = scale ? xj[i] / head : xj[i];
            xj[i] = v;
            if (upd_next) xn[i] -= w1 * v;
        }
        const bool owner = j >= r_beg && j < r_beg + rc;
        if (owner) {
            const int jl = j - r_beg;
            if (tid == 0) xj[jl] = beta;
            if (tj != 0.0)
                for (int e = 1 + tid; e < nk; e += kQrThreads) {
                    const double d = S.red[e];
                    S.chunk[static_cast<size_t>(j + e) * LD + jl] -= tj * (hv[e] + (scale ? d * rh : d));
                }
        }
        __syncthreads();
        if (j + 1 >= w) break;
        // fused pass: update columns j+2.. and accumulate the next partials
        // x_{j+1}' a_k over rows > j+1 (k = j+1 gives the next sigma).
        fused_pass(S, LD, w, j + 1, j + 2, rc, tj != 0.0, j, iu, hv - j, S.red - j, tj, rh, scale, j + 1,
                   max(0, j + 2 - r_beg));
        __syncthreads();
        if (j + 1 < p) send(j + 1);
    }

    if (rc > 0)
        for (int idx = tid; idx < w * rc; idx += kQrThreads) {
            const int c = idx / rc, i = idx - c * rc;
            A[(r_beg + i) + static_cast<int64_t>(c) * lda] = S.chunk[static_cast<size_t>(c) * LD + i];
        }
    cluster.sync();  // no CTA exits while a peer may still write into it
}

size_t cluster_smem_bytes(int w, int LD, int cs) {
    return (static_cast<size_t>(w) * LD + static_cast<size_t>(2) * cs * w + 2 * static_cast<size_t>(w) +
            static_cast<size_t>(w) + static_cast<size_t>(kQrWarps) * w + 4 + 2) *
           sizeof(double);
}

int g_max_cluster = 0;  // largest cluster size the device accepted (probe once)

void max_cluster_device();

int max_cluster() {
    once_per_device(reinterpret_cast<const void*>(&g_max_cluster), [] { max_cluster_device(); });
    return g_max_cluster;
}

void max_cluster_device() {
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
}

inline int odd_ld(int64_t R) { return static_cast<int>(R | 1); }

// Largest column count one cluster launch of cs CTAs can hold for s rows.
int cluster_cols_capacity(int64_t s, int cs) {
    const int LD = odd_ld((s + cs - 1) / cs);
    int w = static_cast<int>(std::max<int64_t>(0, (kSmemCap - 512) / (8 * (LD + 2 + kQrWarps))));
    while (w > 0 && cluster_smem_bytes(w, LD, cs) > static_cast<size_t>(kSmemCap) - 512) --w;
    return w;
}

// Cluster size: enough CTAs for the chunk to fit, and roughly one CTA per 192
// rows (per-column work vs. the DSMEM all-gather, which grows with CS).
int pick_cluster(int64_t s, int64_t w, int cmax) {
    int cs = 1;
    while (cs < cmax && (s + cs - 1) / cs > 192) cs *= 2;
    while (cs < cmax && cluster_cols_capacity(s, cs) < w) cs *= 2;
    return cs;
}

void launch_cluster(cudaStream_t stream, const DView& a, double* tau, int cs) {
    const int s = static_cast<int>(a.rows), w = static_cast<int>(a.cols);
    const int p = std::min(s, w);
    const int R = (s + cs - 1) / cs;
    const int LD = odd_ld(R);
    const size_t smem = cluster_smem_bytes(w, LD, cs);
    if (smem > static_cast<size_t>(kSmemCap)) throw Error(RUTV_ERR_INTERNAL, "hqr: sub-panel exceeds cluster capacity");
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
    int lcs = 0;
    while ((1 << lcs) < cs) ++lcs;
    RUTV_CUDA(cudaLaunchKernelEx(&cfg, hqr_cluster_kernel, a.data, a.ld, s, w, p, R, LD, lcs, tau));
    note_launch();
}

}  // namespace

namespace {
// one blocked right-looking pass with sub-panels of at most nb columns
int64_t blocked_work_elems(int64_t s, int64_t w, int64_t nbmax) {
    // W (s x nb) + Gram (nb x nb) + Tsub (nb x nb) + Z, Z2 (nb x w) + gemm split-K scratch
    const int64_t nb = std::min<int64_t>(w, nbmax);
    return s * nb + 2 * nb * nb + 2 * nb * w + gemm_work_elems(nb, w, s) +
           gemm_work_elems(nb, nb, s) + 1024;
}
constexpr int64_t kFastCols = 128;  // sub-panel width of the Cholesky-QR2 path (cholqr.cu)
}  // namespace

int64_t hqr_work_elems(int64_t s, int64_t w) {
    // the Householder kernels' own blocking, plus (tall panels, cholqr_tall) the outer
    // loop over 128-column fast sub-panels whose fallback runs the former inside
    return blocked_work_elems(s, w, 512) + blocked_work_elems(s, std::min(w, kFastCols), 512);
}

// qr_reg.cu: micro-panel register kernel (preferred where its chunk fits)
int qr_reg_capacity(int64_t s, int cs);
int qr_reg_rows();
void qr_reg_launch(cudaStream_t stream, const DView& a, double* tau, int cs);

namespace {
bool reg_kernel_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RUTV_QR_KERNEL");
        return !(e && std::string(e) == "cluster");
    }();
    return on;
}
}  // namespace

namespace {
// Blocked right-looking panel QR: sub-panels of nb columns factored by `factor`,
// trailing update A_trail <- (I - W T W')' A_trail = A_trail - W T' (W' A_trail).
template <class Factor>
void blocked_panel(cudaStream_t stream, const DView& a, double* tau, int64_t nb, double* scratch,
                   int64_t scratch_elems, Factor factor) {
    const int64_t s = a.rows, w = a.cols, p = std::min(s, w);
    double* W = scratch;
    double* Gm = W + s * nb;
    double* Ts = Gm + nb * nb;
    double* Z = Ts + nb * nb;
    double* Z2 = Z + nb * w;
    double* gw = Z2 + nb * w;
    const int64_t gw_elems = scratch_elems - (gw - scratch);
    if (gw_elems < 0) throw Error(RUTV_ERR_INTERNAL, "hqr: scratch too small");
    for (int64_t j0 = 0; j0 < p; j0 += nb) {
        const int64_t jb = std::min(nb, p - j0);
        DView sub = a.block(j0, j0, s - j0, jb);
        factor(sub, tau + j0);
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
}  // namespace

void hqr_panel(cudaStream_t stream, const DView& a, double* tau, double* twy, int64_t ldt,
               double* scratch, int64_t scratch_elems) {
    const int64_t s = a.rows, w = a.cols, p = std::min(s, w);
    if (p == 0) return;
    if (w > kFastCols && cholqr_tall(s) && scratch_elems >= hqr_work_elems(s, w)) {
        // Tall panel: 128-column sub-panels by Cholesky-QR2 + Householder reconstruction
        // (level-3 work on every SM instead of one 16-CTA cluster streaming the panel
        // column by column), each falling back to the Householder kernels when unsafe.
        const int64_t outer = blocked_work_elems(s, w, 512);
        blocked_panel(stream, a, tau, kFastCols, scratch, outer, [&](const DView& sub, double* t) {
            if (!qr_panel_fast(stream, sub, t))
                hqr_panel_householder(stream, sub, t, scratch + outer, scratch_elems - outer);
        });
    } else if (!qr_panel_fast(stream, a, tau)) {
        hqr_panel_householder(stream, a, tau, scratch, scratch_elems);
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

void hqr_panel_householder(cudaStream_t stream, const DView& a, double* tau, double* scratch,
                           int64_t scratch_elems) {
    const int64_t s = a.rows, w = a.cols, p = std::min(s, w);
    if (p == 0) return;
    const int cmax = max_cluster();
    const bool use_reg = reg_kernel_enabled() && qr_reg_capacity(s, cmax) >= std::min<int64_t>(w, 16);
    auto pick_reg = [&](int64_t rows, int64_t cols) {
        int cs = 1;
        while (cs < cmax && (rows + cs - 1) / cs > qr_reg_rows()) cs *= 2;
        while (cs < cmax && qr_reg_capacity(rows, cs) < cols) cs *= 2;
        return cs;
    };
    auto launch = [&](const DView& sub, double* t) {
        if (use_reg)
            qr_reg_launch(stream, sub, t, pick_reg(sub.rows, sub.cols));
        else
            launch_cluster(stream, sub, t, pick_cluster(sub.rows, sub.cols, cmax));
    };
    int cap = use_reg ? qr_reg_capacity(s, cmax) : cluster_cols_capacity(s, cmax);
    if (cap < 1) throw Error(RUTV_ERR_NOTIMPL, "hqr: panel too tall for one cluster");
    if (use_reg && cap >= 16 && cap < w) cap = cap / 16 * 16;
    if (cap >= w && w <= 512) {
        launch(a, tau);
    } else {
        const int64_t nb = std::min<int64_t>(512, use_reg ? cap : std::max<int64_t>(1, (cap / 8) * 8 > 0 ? (cap / 8) * 8 : cap));
        blocked_panel(stream, a, tau, nb, scratch, scratch_elems, launch);
    }
}

}  // namespace rutv
