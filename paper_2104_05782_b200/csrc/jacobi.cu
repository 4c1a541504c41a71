// jacobi.cu -- one-sided Jacobi SVD of a square b x b block on a CTA cluster.
//
// Restates svd_block (proj/src/jacobi_svd.cpp:39-148) with the reference's
// acceptance semantics, reordered for parallelism:
//   * pair test: skip if ||b_p|| or ||b_q|| <= floor_col = 4 n eps ||A||_F,
//     or |b_p.b_q| <= rel ||b_p|| ||b_q||, rel = max(tol, sqrt(n) eps)
//     (jacobi_svd.cpp:55-72); rotation zeta/t/c/s exactly as :74-80;
//   * converged when a full sweep rotates nothing, ConvergenceError with the
//     worst remaining pair ratio after max_sweeps (:97-109);
//   * sigma_j = ||b_j||, stable descending sort, U = B/sigma above the floor,
//     deterministic orthonormal completion below it (:111-146, :198-240).
// The cyclic row ordering p<q of the reference is replaced by the round-robin
// (circle) tournament ordering: each sweep is n-1 rounds of n/2 disjoint
// pairs that are processed concurrently.  Rows of B (and V) are distributed
// over a cluster of CS CTAs, resident in shared memory; per round the pair
// partial sums (alpha, beta, gamma) are reduce-scattered to the pair's owner
// CTA over DSMEM, the owner decides the rotation, and broadcasts (c, s) back:
// two cluster barriers per round, O(n) DSMEM words per CTA.  Reductions are in
// fixed rank order, so every CTA takes bit-identical decisions.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kJThreads = 512;
int kJSmemCap = 227 * 1024 - 1024;  // refined at first use (dyn_smem_cap)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Round-robin pairing: N even players, round r in [0, N-1), pair pi in [0, N/2).
__device__ __forceinline__ void rr_pair(int N, int r, int pi, int& x, int& y) {
    auto pos = [&](int k) { return k == 0 ? 0 : 1 + ((k - 1 + r) % (N - 1)); };
    x = pos(pi);
    y = pos(N - 1 - pi);
}

struct JParams {
    const double* A;
    int64_t lda;
    int n, N, R, npairs;
    double* U;       // n x n, ld n
    double* sigma;   // n
    double* V;       // n x n, ld n
    double* vglob;   // per-CTA V chunks in global memory when not in smem (else null)
    double* gscr;    // global scratch: CS * max(n, 4) doubles
    double tol;
    int max_sweeps;
    double* status;  // [code, residual, kept, sweeps]
};

__global__ void __launch_bounds__(kJThreads, 1) jacobi_kernel(const JParams P) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = static_cast<int>(cluster.num_blocks());
    const int rank = static_cast<int>(cluster.block_rank());
    const int n = P.n, N = P.N, R = P.R, npairs = P.npairs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int slots = (npairs + CS - 1) / CS;  // pairs owned per CTA

    extern __shared__ __align__(16) double sm[];
    double* Bs = sm;                                     // n columns x R rows
    double* Vs = P.vglob ? P.vglob + static_cast<size_t>(rank) * n * R : Bs + static_cast<size_t>(n) * R;
    double* part = (P.vglob ? Bs + static_cast<size_t>(n) * R : Vs + static_cast<size_t>(n) * R);  // 3*npairs
    double* msg1 = part + 3 * npairs;                    // [CS][slots][3]
    double* dec = msg1 + 3 * CS * slots;                 // [npairs][3] = c, s, flag
    __shared__ int s_rot;
    __shared__ double s_nf;
    __shared__ double s_wp[kJThreads / 32];

    const int r_beg = rank * R;
    const int r_cnt = max(0, min(n, r_beg + R) - r_beg);

    // load rows, V := I rows; ||A||_F partial
    double fro = 0.0;
    for (int idx = tid; idx < n * R; idx += blockDim.x) {
        const int c = idx / R, r = idx % R;
        double v = 0.0;
        if (r < r_cnt) v = P.A[(r_beg + r) + static_cast<int64_t>(c) * P.lda];
        Bs[idx] = v;
        Vs[idx] = (r < r_cnt && r_beg + r == c) ? 1.0 : 0.0;
        fro += v * v;
    }
    fro = warp_sum(fro);
    if (lane == 0) s_wp[warp] = fro;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += s_wp[w];
        P.gscr[rank] = s;
    }
    cluster.sync();
    if (tid == 0) {
        double s = 0.0;
        for (int r = 0; r < CS; ++r) s += P.gscr[r];
        s_nf = sqrt(s);
    }
    __syncthreads();
    const double nf = s_nf;
    const double eps = DBL_EPSILON;
    const double rel = fmax(P.tol, sqrt(static_cast<double>(n)) * eps);
    const double floor_col = 4.0 * static_cast<double>(n) * eps * nf;

    if (n == 0 || nf == 0.0) {  // jacobi_svd.cpp:47-53: U = I, sigma = 0, V = I
        for (int idx = tid; idx < n * r_cnt; idx += blockDim.x) {
            const int c = idx / r_cnt, r = r_beg + idx % r_cnt;
            P.U[r + static_cast<int64_t>(c) * n] = r == c ? 1.0 : 0.0;
            P.V[r + static_cast<int64_t>(c) * n] = r == c ? 1.0 : 0.0;
        }
        if (rank == 0)
            for (int j = tid; j < n; j += blockDim.x) P.sigma[j] = 0.0;
        if (rank == 0 && tid == 0) {
            P.status[0] = 0.0;
            P.status[1] = 0.0;
            P.status[2] = n;
            P.status[3] = 0;
        }
        cluster.sync();
        return;
    }

    // One round: partial dots -> owner reduce/decide -> broadcast -> rotate.
    // check_only: no rotation; owners accumulate the worst ratio instead.
    auto round = [&](int r, bool check_only, double& worst) {
        for (int pi = warp; pi < npairs; pi += nwarps) {
            int x, y;
            rr_pair(N, r, pi, x, y);
            double a = 0.0, b = 0.0, g = 0.0;
            if (x < n && y < n) {
                const int p = min(x, y), q = max(x, y);
                const double* cp = Bs + static_cast<size_t>(p) * R;
                const double* cq = Bs + static_cast<size_t>(q) * R;
                for (int i = lane; i < r_cnt; i += 32) {
                    const double u = cp[i], v = cq[i];
                    a += u * u;
                    b += v * v;
                    g += u * v;
                }
                a = warp_sum(a);
                b = warp_sum(b);
                g = warp_sum(g);
            }
            if (lane == 0) {
                double* dst = CS > 1 ? cluster.map_shared_rank(msg1, pi % CS) : msg1;
                double* slot = dst + 3 * (rank * slots + pi / CS);
                slot[0] = a;
                slot[1] = b;
                slot[2] = g;
            }
        }
        if (CS > 1) cluster.sync(); else __syncthreads();
        // owner: pairs pi = rank + k*CS
        for (int k = tid; k < slots; k += blockDim.x) {
            const int pi = rank + k * CS;
            if (pi >= npairs) continue;
            int x, y;
            rr_pair(N, r, pi, x, y);
            double c = 1.0, s = 0.0, flag = 0.0;
            if (x < n && y < n) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int rr = 0; rr < CS; ++rr) {
                    const double* slot = msg1 + 3 * (rr * slots + k);
                    al += slot[0];
                    be += slot[1];
                    ga += slot[2];
                }
                const double np = sqrt(al), nq = sqrt(be);
                if (!(np <= floor_col || nq <= floor_col)) {
                    if (check_only) {
                        worst = fmax(worst, fabs(ga) / (np * nq));
                    } else if (!(fabs(ga) <= rel * np * nq)) {
                        const double zeta = (be - al) / (2.0 * ga);
                        const double t = (zeta >= 0.0 ? 1.0 : -1.0) /
                                         (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                        c = 1.0 / sqrt(1.0 + t * t);
                        s = c * t;
                        flag = 1.0;
                    }
                }
            }
            for (int d = 0; d < CS; ++d) {
                double* dd = (CS > 1 ? cluster.map_shared_rank(dec, d) : dec) + 3 * pi;
                dd[0] = c;
                dd[1] = s;
                dd[2] = flag;
            }
        }
        if (CS > 1) cluster.sync(); else __syncthreads();
        if (check_only) return;
        // rotate my rows of B and V: pair-major, rows fastest
        const int work = npairs * r_cnt;
        for (int idx = tid; idx < work; idx += blockDim.x) {
            const int pi = idx / r_cnt, i = idx - pi * r_cnt;
            const double* dd = dec + 3 * pi;
            if (dd[2] == 0.0) continue;
            int x, y;
            rr_pair(N, r, pi, x, y);
            const int p = min(x, y), q = max(x, y);
            const double c = dd[0], s = dd[1];
            double* bp = Bs + static_cast<size_t>(p) * R + i;
            double* bq = Bs + static_cast<size_t>(q) * R + i;
            const double u = *bp, v = *bq;
            *bp = c * u - s * v;
            *bq = s * u + c * v;
            double* vp = Vs + static_cast<size_t>(p) * R + i;
            double* vq = Vs + static_cast<size_t>(q) * R + i;
            const double vu = *vp, vv = *vq;
            *vp = c * vu - s * vv;
            *vq = s * vu + c * vv;
        }
        if (tid < npairs && dec[3 * tid + 2] != 0.0) s_rot = 1;
        __syncthreads();
    };

    bool converged = false;
    int sweep = 0;
    double dummy = 0.0;
    for (; sweep < P.max_sweeps && !converged; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int r = 0; r < N - 1; ++r) round(r, false, dummy);
        converged = s_rot == 0;
        __syncthreads();
    }
    if (!converged) {
        double worst = 0.0;
        for (int r = 0; r < N - 1; ++r) round(r, true, worst);
        // owners' local maxima -> global scratch -> max
        __shared__ double s_w[kJThreads / 32];
        double wmax = worst;
        for (int o = 16; o > 0; o >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        if (lane == 0) s_w[warp] = wmax;
        __syncthreads();
        if (tid == 0) {
            double m = 0.0;
            for (int w = 0; w < nwarps; ++w) m = fmax(m, s_w[w]);
            P.gscr[rank] = m;
        }
        cluster.sync();
        if (rank == 0 && tid == 0) {
            double m = 0.0;
            for (int r = 0; r < CS; ++r) m = fmax(m, P.gscr[r]);
            P.status[0] = RUTV_ERR_CONVERGENCE;
            P.status[1] = m;
            P.status[2] = n;
            P.status[3] = sweep;
        }
        cluster.sync();
        return;
    }

    // sigma_j = ||b_j||: partial column sums -> global scratch -> rank-order sum
    for (int c = warp; c < n; c += nwarps) {
        const double* cc = Bs + static_cast<size_t>(c) * R;
        double a = 0.0;
        for (int i = lane; i < r_cnt; i += 32) a += cc[i] * cc[i];
        a = warp_sum(a);
        if (lane == 0) P.gscr[static_cast<size_t>(rank) * n + c] = a;
    }
    cluster.sync();
    double* sig = part;  // reuse: n <= 3*npairs
    for (int c = tid; c < n; c += blockDim.x) {
        double a = 0.0;
        for (int r = 0; r < CS; ++r) a += P.gscr[static_cast<size_t>(r) * n + c];
        sig[c] = sqrt(a);
    }
    __syncthreads();
    // stable descending rank: t(j) = #{k: s_k > s_j} + #{k < j: s_k == s_j}
    int* dest = reinterpret_cast<int*>(msg1);  // n ints fit in 3*CS*slots doubles
    for (int j = tid; j < n; j += blockDim.x) {
        const double sj = sig[j];
        int t = 0;
        for (int k = 0; k < n; ++k) {
            const double sk = sig[k];
            t += (sk > sj) || (k < j && sk == sj);
        }
        dest[j] = t;
    }
    __syncthreads();
    for (int idx = tid; idx < n * r_cnt; idx += blockDim.x) {
        const int j = idx / r_cnt, i = idx - j * r_cnt;
        const int t = dest[j];
        const double s = sig[j];
        const int64_t row = r_beg + i;
        P.V[row + static_cast<int64_t>(t) * n] = Vs[static_cast<size_t>(j) * R + i];
        P.U[row + static_cast<int64_t>(t) * n] =
            s > floor_col ? Bs[static_cast<size_t>(j) * R + i] / s : 0.0;
    }
    if (rank == 0) {
        for (int j = tid; j < n; j += blockDim.x) P.sigma[dest[j]] = sig[j];
        if (tid == 0) {
            int kept = 0;
            for (int j = 0; j < n; ++j) kept += sig[j] > floor_col;
            P.status[0] = 0.0;
            P.status[1] = 0.0;
            P.status[2] = kept;
            P.status[3] = sweep;
        }
    }
    cluster.sync();
}

// complete_orthonormal (jacobi_svd.cpp:198-240) on U's columns kept..n-1: identity
// candidates in index order, two Gram-Schmidt passes, accept norm > 0.25.
// Rare path (rank-deficient blocks); one CTA, sequential over candidates.
__global__ void complete_kernel(double* U, int n, const double* status, double* cand) {
    const int kept = static_cast<int>(status[2]);
    if (status[0] != 0.0 || kept >= n) return;
    __shared__ double red[32];
    __shared__ double s_val;
    int have = kept;
    for (int c = 0; c < n && have < n; ++c) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) cand[i] = i == c ? 1.0 : 0.0;
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass)
            for (int j = 0; j < have; ++j) {
                double d = 0.0;
                for (int i = threadIdx.x; i < n; i += blockDim.x) d += U[i + static_cast<int64_t>(j) * n] * cand[i];
                d = warp_sum(d);
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
                __syncthreads();
                if (threadIdx.x == 0) {
                    double s = 0.0;
                    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
                    s_val = s;
                }
                __syncthreads();
                const double dot = s_val;
                for (int i = threadIdx.x; i < n; i += blockDim.x) cand[i] -= dot * U[i + static_cast<int64_t>(j) * n];
                __syncthreads();
            }
        double nn = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) nn += cand[i] * cand[i];
        nn = warp_sum(nn);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nn;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
            s_val = sqrt(s);
        }
        __syncthreads();
        const double nrm = s_val;
        if (nrm > 0.25) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) U[i + static_cast<int64_t>(have) * n] = cand[i] / nrm;
            ++have;
        }
        __syncthreads();
    }
}

int g_jmax_cluster = 0;

int jmax_cluster() {
    if (g_jmax_cluster) return g_jmax_cluster;
    kJSmemCap = dyn_smem_cap(reinterpret_cast<const void*>(jacobi_kernel));
    RUTV_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RUTV_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kJSmemCap));
    int best = 8;
    for (int cs : {16, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kJThreads);
        cfg.dynamicSmemBytes = kJSmemCap;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = cs;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, jacobi_kernel, &cfg) == cudaSuccess && nclusters > 0) {
            best = cs;
            break;
        }
        cudaGetLastError();
    }
    g_jmax_cluster = best;
    return best;
}

size_t jsmem(int n, int R, int cs, bool v_in_smem) {
    const int N = n + (n & 1), npairs = N / 2, slots = (npairs + cs - 1) / cs;
    return (static_cast<size_t>(n) * R * (v_in_smem ? 2 : 1) + 3 * npairs + 3 * cs * slots +
            3 * npairs) * sizeof(double);
}

}  // namespace

int64_t svd_work_elems(int64_t n, int /*max_sweeps*/) {
    // V chunks in global (worst case) + scratch + completion candidate
    return n * (n + 16) + 16 * std::max<int64_t>(n, 4) + n + 64;
}

void svd_block(cudaStream_t stream, const DView& a, double* u, double* sigma, double* v,
               double* work, int64_t work_elems, double* dev_status, double tol, int max_sweeps) {
    const int n = static_cast<int>(a.rows);
    if (a.rows != a.cols) throw Error(RUTV_ERR_SHAPE, "svd_block expects a square block");
    if (work_elems < svd_work_elems(n, max_sweeps)) throw Error(RUTV_ERR_INTERNAL, "svd scratch too small");
    const int cmax = jmax_cluster();
    int cs = 1;
    bool vsm = true;
    for (;;) {
        const int R = (n + cs - 1) / cs;
        if (jsmem(n, R, cs, true) <= static_cast<size_t>(kJSmemCap) - 1024) break;
        if (cs >= cmax) {
            vsm = false;
            break;
        }
        cs *= 2;
    }
    if (n == 0) cs = 1;
    const int R = std::max(1, (n + cs - 1) / cs);
    if (!vsm && jsmem(n, R, cs, false) > static_cast<size_t>(kJSmemCap) - 1024)
        throw Error(RUTV_ERR_NOTIMPL, "svd_block: block too large for one cluster");
    JParams P;
    P.A = a.data;
    P.lda = a.ld;
    P.n = n;
    P.N = n + (n & 1);
    P.R = R;
    P.npairs = P.N / 2;
    P.U = u;
    P.sigma = sigma;
    P.V = v;
    P.vglob = vsm ? nullptr : work;
    P.gscr = work + static_cast<int64_t>(n) * (n + 16);
    P.tol = tol;
    P.max_sweeps = max_sweeps;
    P.status = dev_status;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kJThreads);
    cfg.dynamicSmemBytes = jsmem(n, R, cs, vsm);
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    RUTV_CUDA(cudaLaunchKernelEx(&cfg, jacobi_kernel, P));
    note_launch();
    double* cand = P.gscr + 16 * std::max(n, 4);
    complete_kernel<<<1, 256, 0, stream>>>(u, n, dev_status, cand);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

}  // namespace rutv
