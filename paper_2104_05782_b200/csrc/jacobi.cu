// jacobi.cu -- batched one-sided Jacobi SVD of square blocks on CTA clusters.
//
// Restates svd_block (proj/src/jacobi_svd.cpp:39-148) with the reference's
// acceptance semantics, reordered for parallelism:
//   * pair test: skip if ||b_p|| or ||b_q|| <= floor_col = 4 n eps ||A||_F,
//     or |b_p.b_q| <= rel ||b_p|| ||b_q||, rel = max(tol, sqrt(n) eps)
//     (jacobi_svd.cpp:55-72); zeta / t / c / s exactly as :74-80;
//   * converged when a full sweep rotates nothing; ConvergenceError carrying
//     the worst remaining pair ratio after max_sweeps (:97-109);
//   * sigma_j = ||b_j||, stable descending sort, U = B / sigma above the floor,
//     deterministic orthonormal completion below it (:111-146, :198-240).
// The reference's cyclic p<q order becomes the round-robin (circle)
// tournament: a sweep is N-1 rounds of N/2 disjoint pairs processed at once.
//
// Layout: one cluster of CS CTAs per problem, many problems per launch (the
// driver batches every b x b block of a factorization into one launch).  The
// problem's rows are split over the cluster, B and V resident in shared
// memory (V in a global work buffer when it does not fit).  A pair is owned by
// a group of LPP = 8 lanes; each lane holds <= RPL rows of b_p, b_q in
// registers, the three partial dots are reduced inside the 8-lane group, and
// -- for CS > 1 -- exchanged over DSMEM (every CTA receives every pair's
// partials, sums them in rank order, and takes the identical decision).  Per
// round: one cluster barrier (or none for CS = 1) and one __syncthreads.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cfloat>
#include <vector>

#include "cluster_msg.cuh"
#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kJThreads = 512;
constexpr int kLPP = 8;                      // lanes per pair
constexpr int kPPW = 32 / kLPP;              // pairs per warp
constexpr int kPairsPerPass = kPPW * kJThreads / 32;  // 64

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Round-robin pairing: N even players, round r in [0, N-1), pair pi in [0, N/2).
__device__ __forceinline__ void rr_pair(int N, int r, int pi, int& p, int& q) {
    auto pos = [&](int k) {
        if (k == 0) return 0;
        int v = k - 1 + r;
        if (v >= N - 1) v -= N - 1;
        return 1 + v;
    };
    const int x = pos(pi), y = pos(N - 1 - pi);
    p = min(x, y);
    q = max(x, y);
}

__device__ long long* g_jtrace = nullptr;  // debug: RUTV_JAC_TRACE per-round clock64 of CTA 0

template <int RPL, bool VSM>
__global__ void __launch_bounds__(kJThreads, 1)
    jacobi_kernel(const SvdDesc* __restrict__ descs, int R, int vsm_unused, int rs, double tol, int max_sweeps) {
    constexpr bool vsm = VSM;  // V in shared memory: compile-time, so V accesses are LDS / STS
    (void)vsm_unused;
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = static_cast<int>(cluster.num_blocks());
    const int rank = static_cast<int>(cluster.block_rank());
    const SvdDesc d = descs[blockIdx.x / CS];
    const int n = d.n, N = n + (n & 1), npairs = N / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kJThreads / 32;
    const int grp = lane / kLPP, sl = lane % kLPP;
    const int r_beg = rank * R;
    const int r_cnt = max(0, min(n, r_beg + R) - r_beg);
    const int LB = R | 1;  // column stride of B / V: odd -> the 4 pair groups of a warp hit distinct banks

    extern __shared__ __align__(16) double sm[];
    double* Bs = sm;  // n columns x R rows
    double* Vs = vsm ? Bs + static_cast<size_t>(n) * LB : d.work + static_cast<size_t>(rank) * n * LB;
    double* xb = (vsm ? Vs : Bs) + static_cast<size_t>(n) * LB;  // [2][CS][npairs][3]
    const size_t xpar = static_cast<size_t>(CS) * npairs * 3;
    __shared__ int s_rot;
    __shared__ double s_red[32];

    // load my rows of B, V := I rows, ||A||_F partial
    double fro = 0.0;
    for (int c = 0; c < n; ++c)
        for (int i = tid; i < R; i += kJThreads) {
            double v = 0.0;
            if (i < r_cnt) v = d.A[(r_beg + i) + static_cast<int64_t>(c) * d.lda];
            Bs[static_cast<size_t>(c) * LB + i] = v;
            Vs[static_cast<size_t>(c) * LB + i] = (i < r_cnt && r_beg + i == c) ? 1.0 : 0.0;
            fro += v * v;
        }
    fro = warp_sum(fro);
    if (lane == 0) s_red[warp] = fro;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += s_red[w];
        if (CS > 1)
            for (int dst = 0; dst < CS; ++dst) cluster.map_shared_rank(xb, dst)[rank] = s;
        else
            xb[0] = s;
    }
    if (CS > 1) cluster.sync(); else __syncthreads();
    double nf2 = 0.0;
    for (int r = 0; r < CS; ++r) nf2 += xb[r];
    const double nf = sqrt(nf2);
    const double eps = DBL_EPSILON;
    const double rel = fmax(tol, sqrt(static_cast<double>(n)) * eps);
    const double floor_col = 4.0 * static_cast<double>(n) * eps * nf;
    if (CS > 1) cluster.sync(); else __syncthreads();  // xb reused below

    if (n == 0 || nf == 0.0) {  // jacobi_svd.cpp:47-53: U = I, sigma = 0, V = I
        for (int c = 0; c < n; ++c)
            for (int i = tid; i < r_cnt; i += kJThreads) {
                const int row = r_beg + i;
                d.U[row + static_cast<int64_t>(c) * n] = row == c ? 1.0 : 0.0;
                d.V[row + static_cast<int64_t>(c) * n] = row == c ? 1.0 : 0.0;
            }
        if (rank == 0)
            for (int j = tid; j < n; j += kJThreads) d.sigma[j] = 0.0;
        if (rank == 0 && tid == 0) {
            d.status[0] = 0.0;
            d.status[1] = 0.0;
            d.status[2] = n;
            d.status[3] = 0;
        }
        if (CS > 1) cluster.sync();
        return;
    }

    // One round.  mode 0: rotate; mode 1: check only (owners track the worst
    // remaining pair ratio).  All-gather exchange (rs == 0): every CTA gets every
    // pair's partials and decides itself -- one cluster barrier.  Reduce-scatter
    // (rs != 0, large clusters): pair pi's partials go to CTA pi % CS, which
    // decides and broadcasts (c, s, flag) -- two barriers, O(npairs) words.
    const int slots = (npairs + CS - 1) / CS;
    double* dec = xb + static_cast<size_t>(CS) * slots * 3;  // rs mode: [npairs][3]
    // all-gather mode: one mbarrier per round parity counts the peers' partials
    __shared__ __align__(8) uint64_t s_bar[2];
    const uint32_t bar0 = smem_u32(s_bar);
    const uint32_t xbytes = static_cast<uint32_t>((CS - 1) * npairs * 3 * 8);
    int gr = 0;  // rounds done (both sweeps and check-only rounds)
    if (!rs && CS > 1) {
        if (tid == 0) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_arm(&s_bar[0], xbytes);
            mbar_arm(&s_bar[1], xbytes);
        }
        cluster.sync();  // peers' barriers armed before any remote traffic
    }
    // zeta is formed before the skip tests (it only depends on the partials;
    // unused -- possibly inf -- when the pair is skipped), so its division
    // overlaps the two square roots; c = rsqrt(1 + t^2).
    auto decide = [&](double al, double be, double ga, double& c, double& s, double& ratio, bool want_ratio) -> bool {
        const double np = sqrt(al), nq = sqrt(be);
        const double zeta = (be - al) / (2.0 * ga);
        ratio = -1.0;
        if (np <= floor_col || nq <= floor_col) return false;
        const double pq = np * nq;
        if (want_ratio) ratio = fabs(ga) / pq;
        if (fabs(ga) <= rel * pq) return false;
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        c = rsqrt(1.0 + tt * tt);
        s = c * tt;
        return true;
    };
    auto rotate = [&](int p, int q, double c, double s) {
        double* bp = Bs + static_cast<size_t>(p) * LB;
        double* bq = Bs + static_cast<size_t>(q) * LB;
        double* vp = Vs + static_cast<size_t>(p) * LB;
        double* vq = Vs + static_cast<size_t>(q) * LB;
        // rows in chunks of 4: all loads of a chunk issue before its stores (the
        // pointers may alias as far as the compiler knows)
#pragma unroll
        for (int t0 = 0; t0 < RPL; t0 += 4) {
            double x[4], y[4], vx[4], vy[4];
#pragma unroll
            for (int u = 0; u < 4 && t0 + u < RPL; ++u) {
                const int i = sl + kLPP * (t0 + u);
                const bool ok = i < r_cnt;
                x[u] = ok ? bp[i] : 0.0;
                y[u] = ok ? bq[i] : 0.0;
                vx[u] = ok ? vp[i] : 0.0;
                vy[u] = ok ? vq[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4 && t0 + u < RPL; ++u) {
                const int i = sl + kLPP * (t0 + u);
                if (i < r_cnt) {
                    bp[i] = c * x[u] - s * y[u];
                    bq[i] = s * x[u] + c * y[u];
                    vp[i] = c * vx[u] - s * vy[u];
                    vq[i] = s * vx[u] + c * vy[u];
                }
            }
        }
    };
    long long* const jtr = (g_jtrace && blockIdx.x == 0 && tid == 0) ? g_jtrace : nullptr;
    auto round = [&](int r, int par, int mode, double& worst) -> bool {
        if (jtr && gr < 64) jtr[gr * 4 + 0] = clock64();
        // phase 1: partial dots of every pair over my rows
        for (int base = 0; base < npairs; base += kPairsPerPass) {
            const int pi = base + warp * kPPW + grp;
            int p = 0, q = 0;
            const bool ok = pi < npairs;
            if (ok) rr_pair(N, r, pi, p, q);
            double a = 0.0, b = 0.0, g = 0.0;
            if (ok && q < n) {
                const double* cp = Bs + static_cast<size_t>(p) * LB;
                const double* cq = Bs + static_cast<size_t>(q) * LB;
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    const int i = sl + kLPP * t;
                    if (i < r_cnt) {
                        const double u = cp[i], v = cq[i];
                        a += u * u;
                        b += v * v;
                        g += u * v;
                    }
                }
            }
#pragma unroll
            for (int o = kLPP / 2; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
                g += __shfl_xor_sync(0xffffffffu, g, o);
            }
            if (!ok) continue;
            if (rs) {
                if (sl == 0) {
                    double* slot = cluster.map_shared_rank(xb, pi % CS) +
                                   (static_cast<size_t>(rank) * slots + pi / CS) * 3;
                    slot[0] = a;
                    slot[1] = b;
                    slot[2] = g;
                }
            } else if (sl < 3) {
                // lane sl owns value sl of the pair: written locally, and sent to
                // every peer with st.async completing on its mbarrier `par`
                const double val = sl == 0 ? a : (sl == 1 ? b : g);
                double* slot = xb + par * xpar + (static_cast<size_t>(rank) * npairs + pi) * 3 + sl;
                *slot = val;
                if (CS > 1) {
                    const uint32_t la = smem_u32(slot), lb = bar0 + 8 * par;
                    for (int dst = 0; dst < CS; ++dst)
                        if (dst != rank) st_async_f64(mapa_u32(la, dst), val, mapa_u32(lb, dst));
                }
            }
        }
        if (rs) {
            cluster.sync();
        } else {
            __syncthreads();  // local partials visible to the deciders
            if (jtr && gr < 64) jtr[gr * 4 + 1] = clock64();
            if (CS > 1 && tid < npairs) {
                mbar_wait(&s_bar[par], static_cast<uint32_t>((gr >> 1) & 1));
                if (tid == 0) mbar_arm(&s_bar[par], xbytes);  // round gr + 2
            }
            if (jtr && gr < 64) jtr[gr * 4 + 2] = clock64();
        }
        bool any = false;
        if (rs) {
            // owners reduce their pairs in rank order and broadcast the decision
            for (int k = tid; k < slots; k += kJThreads) {
                const int pi = rank + k * CS;
                if (pi >= npairs) continue;
                int p, q;
                rr_pair(N, r, pi, p, q);
                double c = 1.0, s = 0.0, flag = 0.0, ratio = -1.0;
                if (q < n) {
                    double al = 0.0, be = 0.0, ga = 0.0;
                    for (int rr = 0; rr < CS; ++rr) {
                        const double* slot = xb + (static_cast<size_t>(rr) * slots + k) * 3;
                        al += slot[0];
                        be += slot[1];
                        ga += slot[2];
                    }
                    if (decide(al, be, ga, c, s, ratio, mode == 1) && mode == 0) flag = 1.0;
                    if (mode == 1 && ratio >= 0.0) worst = fmax(worst, ratio);
                }
                for (int dst = 0; dst < CS; ++dst) {
                    double* dd = cluster.map_shared_rank(dec, dst) + 3 * pi;
                    dd[0] = c;
                    dd[1] = s;
                    dd[2] = flag;
                }
            }
            cluster.sync();
            if (mode == 0)
                for (int base = 0; base < npairs; base += kPairsPerPass) {
                    const int pi = base + warp * kPPW + grp;
                    if (pi >= npairs) continue;
                    const double* dd = dec + 3 * pi;
                    if (dd[2] == 0.0) continue;
                    int p, q;
                    rr_pair(N, r, pi, p, q);
                    any = true;
                    rotate(p, q, dd[0], dd[1]);
                }
        } else {
            // one thread per pair decides (sums the CS partials in rank order:
            // bit-identical decisions in every CTA), the 8-lane groups rotate
            double* decl = xb + 2 * xpar;  // [npairs][3]
            for (int pi = tid; pi < npairs; pi += kJThreads) {
                int p, q;
                rr_pair(N, r, pi, p, q);
                double c = 1.0, s = 0.0, flag = 0.0, ratio = -1.0;
                if (q < n) {
                    double al = 0.0, be = 0.0, ga = 0.0;
                    for (int rr = 0; rr < CS; ++rr) {
                        const double* slot = xb + par * xpar + (static_cast<size_t>(rr) * npairs + pi) * 3;
                        al += slot[0];
                        be += slot[1];
                        ga += slot[2];
                    }
                    if (decide(al, be, ga, c, s, ratio, mode == 1) && mode == 0) flag = 1.0;
                    if (mode == 1 && ratio >= 0.0) worst = fmax(worst, ratio);
                }
                decl[3 * pi] = c;
                decl[3 * pi + 1] = s;
                decl[3 * pi + 2] = flag;
            }
            __syncthreads();
            if (mode == 0)
                for (int base = 0; base < npairs; base += kPairsPerPass) {
                    const int pi = base + warp * kPPW + grp;
                    if (pi >= npairs) continue;
                    const double* dd = decl + 3 * pi;
                    if (dd[2] == 0.0) continue;
                    int p, q;
                    rr_pair(N, r, pi, p, q);
                    any = true;
                    rotate(p, q, dd[0], dd[1]);
                }
        }
        if (jtr && gr < 64) jtr[gr * 4 + 3] = clock64();
        __syncthreads();
        ++gr;
        return any;
    };

    bool converged = false;
    int sweep = 0;
    int par = 0;
    double worst = 0.0;
    for (; sweep < max_sweeps && !converged; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int r = 0; r < N - 1; ++r, par ^= 1)
            if (round(r, par, 0, worst)) s_rot = 1;
        __syncthreads();
        converged = s_rot == 0;
        __syncthreads();
    }

    if (!converged) {  // residual: worst remaining pair ratio (jacobi_svd.cpp:97-109)
        for (int r = 0; r < N - 1; ++r, par ^= 1) round(r, par, 1, worst);
        for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        if (lane == 0) s_red[warp] = worst;
        __syncthreads();
        if (tid == 0) {
            double m = 0.0;
            for (int w = 0; w < nwarps; ++w) m = fmax(m, s_red[w]);
            if (CS > 1) cluster.map_shared_rank(xb, 0)[rank] = m;
            else xb[0] = m;
        }
        if (CS > 1) cluster.sync(); else __syncthreads();
        if (rank == 0 && tid == 0) {
            double m = 0.0;
            for (int r = 0; r < CS; ++r) m = fmax(m, xb[r]);
            d.status[0] = RUTV_ERR_CONVERGENCE;
            d.status[1] = m;
            d.status[2] = n;
            d.status[3] = sweep;
        }
        if (CS > 1) cluster.sync();
        return;
    }

    // sigma_j = ||b_j||: partial column sums, all-gathered, summed in rank order.
    if (CS > 1) cluster.sync();  // every CTA done reading xb
    for (int c = warp; c < n; c += nwarps) {
        const double* cc = Bs + static_cast<size_t>(c) * LB;
        double a = 0.0;
        for (int i = lane; i < r_cnt; i += 32) a += cc[i] * cc[i];
        a = warp_sum(a);
        if (lane < CS) {
            double* dst = CS > 1 ? cluster.map_shared_rank(xb, lane) : xb;
            dst[static_cast<size_t>(rank) * n + c] = a;
        }
    }
    if (CS > 1) cluster.sync(); else __syncthreads();
    __shared__ double s_sig[1024];
    __shared__ int s_dest[1024];
    for (int c = tid; c < n; c += kJThreads) {
        double a = 0.0;
        for (int r = 0; r < CS; ++r) a += xb[static_cast<size_t>(r) * n + c];
        s_sig[c] = sqrt(a);
    }
    __syncthreads();
    for (int j = tid; j < n; j += kJThreads) {  // stable descending rank
        const double sj = s_sig[j];
        int t = 0;
        for (int k = 0; k < n; ++k) {
            const double sk = s_sig[k];
            t += (sk > sj) || (k < j && sk == sj);
        }
        s_dest[j] = t;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        const int t = s_dest[j];
        const double s = s_sig[j];
        for (int i = tid; i < r_cnt; i += kJThreads) {
            const int64_t row = r_beg + i;
            d.V[row + static_cast<int64_t>(t) * n] = Vs[static_cast<size_t>(j) * LB + i];
            d.U[row + static_cast<int64_t>(t) * n] =
                s > floor_col ? Bs[static_cast<size_t>(j) * LB + i] / s : 0.0;
        }
    }
    if (rank == 0) {
        for (int j = tid; j < n; j += kJThreads) d.sigma[s_dest[j]] = s_sig[j];
        if (tid == 0) {
            int kept = 0;
            for (int j = 0; j < n; ++j) kept += s_sig[j] > floor_col;
            d.status[0] = 0.0;
            d.status[1] = 0.0;
            d.status[2] = kept;
            d.status[3] = sweep;
        }
    }
    if (CS > 1) cluster.sync();
}

// complete_orthonormal (jacobi_svd.cpp:198-240) on U's columns kept..n-1: identity
// candidates in index order, two Gram-Schmidt passes, accept norm > 0.25.
// Rare path (rank-deficient blocks); one CTA per problem, early exit otherwise.
__global__ void complete_kernel(const SvdDesc* __restrict__ descs) {
    const SvdDesc d = descs[blockIdx.x];
    const int n = d.n;
    const int kept = static_cast<int>(d.status[2]);
    if (d.status[0] != 0.0 || kept >= n) return;
    double* U = d.U;
    double* cand = d.work + static_cast<size_t>(n) * (n + 16);
    __shared__ double red[32];
    __shared__ double s_val;
    const int nw = blockDim.x >> 5;
    auto block_sum = [&](double v) {
        v = warp_sum(v);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += red[w];
            s_val = s;
        }
        __syncthreads();
        const double r = s_val;
        __syncthreads();
        return r;
    };
    int have = kept;
    for (int c = 0; c < n && have < n; ++c) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) cand[i] = i == c ? 1.0 : 0.0;
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass)
            for (int j = 0; j < have; ++j) {
                double dd = 0.0;
                for (int i = threadIdx.x; i < n; i += blockDim.x) dd += U[i + static_cast<int64_t>(j) * n] * cand[i];
                const double dot = block_sum(dd);
                for (int i = threadIdx.x; i < n; i += blockDim.x) cand[i] -= dot * U[i + static_cast<int64_t>(j) * n];
                __syncthreads();
            }
        double nn = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) nn += cand[i] * cand[i];
        const double nrm = sqrt(block_sum(nn));
        if (nrm > 0.25) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) U[i + static_cast<int64_t>(have) * n] = cand[i] / nrm;
            ++have;
        }
        __syncthreads();
    }
}

struct JCfg {
    int cs, R, vsm, rpl;
    size_t smem;
};

int g_jcap = 0, g_jmax_cluster = 0;

void jinit_device();

template <int RPL, bool VSM>
void prep_kernel() {
    auto k = jacobi_kernel<RPL, VSM>;
    RUTV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    RUTV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, g_jcap));
}

template <int RPL>
void launch_j(cudaLaunchConfig_t& cfg, int vsm, const SvdDesc* d, int R, int rs, double tol, int max_sweeps) {
    if (vsm)
        RUTV_CUDA(cudaLaunchKernelEx(&cfg, jacobi_kernel<RPL, true>, d, R, vsm, rs, tol, max_sweeps));
    else
        RUTV_CUDA(cudaLaunchKernelEx(&cfg, jacobi_kernel<RPL, false>, d, R, vsm, rs, tol, max_sweeps));
}

void jinit() {
    once_per_device(reinterpret_cast<const void*>(&g_jcap), [] { jinit_device(); });
}

void jinit_device() {
    g_jcap = dyn_smem_cap(reinterpret_cast<const void*>(jacobi_kernel<16, true>));
    prep_kernel<2, true>();
    prep_kernel<4, true>();
    prep_kernel<8, true>();
    prep_kernel<16, true>();
    prep_kernel<2, false>();
    prep_kernel<4, false>();
    prep_kernel<8, false>();
    prep_kernel<16, false>();
    g_jmax_cluster = 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kJThreads);
    cfg.dynamicSmemBytes = g_jcap;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 16;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, jacobi_kernel<16, true>, &cfg) == cudaSuccess && ncl > 0)
        g_jmax_cluster = 16;
    cudaGetLastError();
}

bool use_rs(int n, int cs) { return cs >= 8 && n > 256; }

size_t jsmem_bytes(int n, int R, int cs, bool vsm) {
    const int npairs = (n + (n & 1)) / 2;
    const size_t slots = (static_cast<size_t>(npairs) + cs - 1) / cs;
    const size_t xg = use_rs(n, cs) ? static_cast<size_t>(cs) * slots * 3 + 3 * static_cast<size_t>(npairs)
                                    : 2 * static_cast<size_t>(cs) * npairs * 3 + 3 * static_cast<size_t>(npairs);
    const size_t x = std::max<size_t>(xg, static_cast<size_t>(cs) * n + 8);
    return (static_cast<size_t>(n) * (R | 1) * (vsm ? 2 : 1) + x) * sizeof(double);
}

JCfg choose(int n, int count = 1) {
    jinit();
    const size_t cap = static_cast<size_t>(g_jcap) - 512;
    JCfg c{1, std::max(n, 1), 1, 16, 0};
    static const int force_cs = [] {  // tuning knob: RUTV_JACOBI_CS=k starts the search at k CTAs
        const char* e = std::getenv("RUTV_JACOBI_CS");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    for (int cs = force_cs;; cs *= 2) {
        const int R = std::max(1, (n + cs - 1) / cs);
        if (R <= kLPP * 16 && jsmem_bytes(n, R, cs, true) <= cap) {
            c = {cs, R, 1, 0, jsmem_bytes(n, R, cs, true)};
            break;
        }
        if (cs >= g_jmax_cluster) {
            const int R2 = std::max(1, (n + g_jmax_cluster - 1) / g_jmax_cluster);
            if (R2 > kLPP * 16 || jsmem_bytes(n, R2, g_jmax_cluster, false) > cap)
                throw Error(RUTV_ERR_NOTIMPL, "svd_block: block too large for one cluster");
            c = {g_jmax_cluster, R2, 0, 0, jsmem_bytes(n, R2, g_jmax_cluster, false)};
            break;
        }
    }
    // Each round streams the CTA's rows of B and V through shared memory, so
    // time per round scales with the rows per CTA: spread a problem over more
    // CTAs while the whole batch still fits in one wave of SMs -- down to 32
    // rows per CTA; below that the per-round DSMEM exchange dominates (B200,
    // n = 128 batches: 4 CTAs 3.2 ms, 8 CTAs 4.3 ms, 1-2 CTAs 4.7 ms).
    static const int cs_cap = [] {  // tuning knob: RUTV_JACOBI_CSMAX=k caps the widening at k CTAs
        const char* e = std::getenv("RUTV_JACOBI_CSMAX");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : 1 << 30;
    }();
    while (c.vsm && c.cs * 2 <= std::min(g_jmax_cluster, cs_cap) && static_cast<int64_t>(count) * c.cs * 2 <= kNumSMs &&
           (n + 2 * c.cs - 1) / (2 * c.cs) >= 32 && !use_rs(n, c.cs * 2)) {
        const int cs = c.cs * 2, R = (n + cs - 1) / cs;
        c = {cs, R, 1, 0, jsmem_bytes(n, R, cs, true)};
    }
    const int rpl = (c.R + kLPP - 1) / kLPP;
    c.rpl = rpl <= 2 ? 2 : rpl <= 4 ? 4 : rpl <= 8 ? 8 : 16;
    return c;
}

}  // namespace

// V spill (CS x n x (R | 1) <= n (n + 16)) + completion candidate
int64_t svd_blk_work_elems(int64_t n);
bool svd_blk_applicable(int nmax);
void svd_batch_blk(cudaStream_t stream, const SvdDesc* d_descs, int count, int nmax, double tol, int max_sweeps);

int64_t svd_work_elems(int64_t n, int /*max_sweeps*/) {
    return std::max<int64_t>(n * (n + 16) + n + 64, svd_blk_work_elems(n));
}

void svd_batch(cudaStream_t stream, const SvdDesc* d_descs, int count, int nmax, double tol,
               int max_sweeps) {
    if (count <= 0) return;
    if (svd_blk_applicable(nmax)) {  // blocks up to 512 wide: the column-distributed kernel (jacobi_blk.cu)
        svd_batch_blk(stream, d_descs, count, nmax, tol, max_sweeps);
        complete_kernel<<<count, 256, 0, stream>>>(d_descs);
        note_launch();
        RUTV_CHECK_LAUNCH();
        return;
    }
    const JCfg c = choose(nmax, count);
    const int rs = use_rs(nmax, c.cs) ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * c.cs));
    cfg.blockDim = dim3(kJThreads);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = c.cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    static const bool jtrace = std::getenv("RUTV_JAC_TRACE") != nullptr;
    long long* dtr = nullptr;
    if (jtrace) {
        RUTV_CUDA(cudaMalloc(&dtr, 64 * 4 * sizeof(long long)));
        RUTV_CUDA(cudaMemset(dtr, 0, 64 * 4 * sizeof(long long)));
        RUTV_CUDA(cudaMemcpyToSymbol(g_jtrace, &dtr, sizeof(dtr)));
    }
    struct TraceOut {
        long long* p;
        int cs;
        ~TraceOut() {
            if (!p) return;
            long long h[256];
            cudaDeviceSynchronize();
            cudaMemcpy(h, p, sizeof(h), cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "jacobi trace cs=%d (cycles: dots+send, wait, decide+rotate, next)\n", cs);
            for (int r = 0; r + 1 < 16; ++r)
                std::fprintf(stderr, "  round %2d: %6lld %6lld %6lld %6lld\n", r, h[r * 4 + 1] - h[r * 4], h[r * 4 + 2] - h[r * 4 + 1],
                             h[r * 4 + 3] - h[r * 4 + 2], h[(r + 1) * 4] - h[r * 4 + 3]);
            long long* z = nullptr;
            cudaMemcpyToSymbol(g_jtrace, &z, sizeof(z));
            cudaFree(p);
        }
    } tro{dtr, c.cs};
    switch (c.rpl) {
        case 2: launch_j<2>(cfg, c.vsm, d_descs, c.R, rs, tol, max_sweeps); break;
        case 4: launch_j<4>(cfg, c.vsm, d_descs, c.R, rs, tol, max_sweeps); break;
        case 8: launch_j<8>(cfg, c.vsm, d_descs, c.R, rs, tol, max_sweeps); break;
        default: launch_j<16>(cfg, c.vsm, d_descs, c.R, rs, tol, max_sweeps); break;
    }
    note_launch();
    complete_kernel<<<count, 256, 0, stream>>>(d_descs);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

void svd_block(cudaStream_t stream, const DView& a, double* u, double* sigma, double* v,
               double* work, int64_t work_elems, double* dev_status, double tol, int max_sweeps) {
    const int n = static_cast<int>(a.rows);
    if (a.rows != a.cols) throw Error(RUTV_ERR_SHAPE, "svd_block expects a square block");
    if (work_elems < svd_work_elems(n, max_sweeps) + 16)
        throw Error(RUTV_ERR_INTERNAL, "svd scratch too small");
    SvdDesc h{a.data, a.ld, n, 0, u, sigma, v, work, dev_status};
    // descriptor lives at the end of the work buffer (stream-ordered copy)
    SvdDesc* dd = reinterpret_cast<SvdDesc*>(work + svd_work_elems(n, max_sweeps));
    static_assert(sizeof(SvdDesc) <= 16 * sizeof(double), "descriptor slot");
    RUTV_CUDA(cudaMemcpyAsync(dd, &h, sizeof h, cudaMemcpyHostToDevice, stream));
    // pageable source: cudaMemcpyAsync stages `h` before returning
    svd_batch(stream, dd, 1, n, tol, max_sweeps);
}

}  // namespace rutv
