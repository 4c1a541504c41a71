// jacobi_blk.cu -- batched one-sided Jacobi SVD with COLUMN-distributed blocks (n <= 512).
//
// Same algorithm contract as jacobi.cu (reference proj/src/jacobi_svd.cpp:39-148: one-sided
// Jacobi on the columns of a square block, thresholds rel = max(tol, sqrt(n) eps) and
// floor = 4 n eps ||A||_F, a sweep without rotations ends the iteration, max_sweeps ->
// ConvergenceError with the worst remaining pair ratio, stable descending sort, U = b / sigma),
// different data distribution.  jacobi.cu splits the ROWS of a block over the CTAs of a cluster,
// so every pair's three dot products cross the cluster every round (one DSMEM exchange + two CTA
// barriers per round, ~5 K cycles for n = 128).  Here the block's columns are cut into NB = 2 CS
// column blocks of 16; a CTA holds TWO column blocks (32 whole columns of B and of V) in shared
// memory and one HALF-WARP owns a pair: dots, decision and rotation are warp-local (shuffles
// only; the two pairs of a warp share every instruction -- with a full warp per pair the round was
// bound by the SM's shuffle and FP64 issue rates, 2.5 K cycles, all 32 lanes repeating one pair's
// square roots and divisions), a round costs one CTA barrier, and the cluster only meets when the
// column blocks are re-paired:
//   super-round sr of a sweep: CTA c takes the block pair rr_pair(NB, sr, c) of a round-robin
//   tournament over the blocks; the first super-round rotates all 31 x 16 pairs of its 32
//   columns, the others only the 16 x 16 cross pairs -- 31 + (NB - 2) 16 = N - 1 rounds per
//   sweep, every column pair exactly once.
// Between super-rounds the blocks live in a global master copy (the problem's work buffer, L2
// resident): store both blocks, fence, cluster barrier, load the next two.  V never enters shared
// memory: the rotations of a super-round are accumulated in a 32 x 32 matrix J (two rows per lane
// instead of n / 16), and V(:, my 32 columns) <- V(:, my 32 columns) J is applied to the master copy
// once per super-round -- half the shared-memory traffic of a round (which bounds it), and blocks
// up to 512 wide fit (32 columns of B: 131 KB).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "cluster_msg.cuh"
#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kBT = 256;  // threads: 8 warps x 2 half-warps = the 16 pairs of a local round
constexpr int kBW = 16;   // columns per block
constexpr int kHL = 16;   // lanes per pair

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double hsum(double v) {  // over the 16 lanes of a half-warp
#pragma unroll
    for (int o = kHL / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// round-robin pairing of N (even) players: round r in [0, N - 1), pair pi in [0, N / 2)
__device__ __forceinline__ void rrp(int N, int r, int pi, int& p, int& q) {
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

// jacobi_svd.cpp:60-85: skip tests and the rotation (c, s) of a pair from its three dots.  The
// skip tests in squared form (no square roots: ||b|| <= floor <=> ||b||^2 <= floor^2,
// |g| <= rel ||p|| ||q|| <=> g^2 <= rel^2 a b) come first, so a pair that does not rotate costs
// a few multiplies; the rotation itself is the reference's formula.
__device__ __forceinline__ bool jskip(double al, double be, double ga, double rel2, double floor2) {
    return al <= floor2 || be <= floor2 || ga * ga <= rel2 * (al * be);
}
__device__ __forceinline__ void jrot(double al, double be, double ga, double& c, double& s) {
    const double zeta = (be - al) / (2.0 * ga);
    const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    c = rsqrt(1.0 + tt * tt);
    s = c * tt;
}

__device__ long long* g_jbtrace = nullptr;  // debug: RUTV_JAC_TRACE per-round clock64 of CTA 0, warp 0

template <int RPT>  // rows per lane of a pair: n <= 16 RPT
__global__ void __launch_bounds__(kBT, 1)
    jacobi_blk_kernel(const SvdDesc* __restrict__ descs, int NB, int ldb, double tol, int max_sweeps) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = NB / 2;
    const int rank = static_cast<int>(cluster.block_rank());
    const SvdDesc d = descs[blockIdx.x / CS];
    const int n = d.n, NP = NB * kBW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) double sm[];
    constexpr int LJ = 2 * kBW + 1;
    double* Bs = sm;                                           // 32 columns x ldb
    double* Js = sm + static_cast<size_t>(2 * kBW) * ldb;      // J (32 x 32, column c at Js + c LJ)
    // the round body addresses shared memory from one opaque register (no special-register reads
    // rematerialised per round, see qr_reg.cu)
    uint32_t bs_a;
    asm volatile("mov.u32 %0, %1;" : "=r"(bs_a) : "r"(smem_u32(sm)));
    const uint32_t js_a = bs_a + 8u * static_cast<uint32_t>(2 * kBW * ldb);
    __shared__ double s_red[32];
    // global master copies and cluster-wide scratch (the problem's work buffer)
    double* Bm = d.work;
    double* Vm = Bm + static_cast<size_t>(n) * NP;
    double* sig = Vm + static_cast<size_t>(n) * NP;       // NP
    double* aux = sig + NP;                               // [0, 16): per-CTA partials; then 2 int flags
    int* gflag = reinterpret_cast<int*>(aux + 16);
    auto csync = [&] {
        __threadfence();
        if (CS > 1) cluster.sync(); else __syncthreads();
    };

    // masters: B := A (zero padding columns), V := I; ||A||_F
    double fro = 0.0;
    for (int64_t idx = static_cast<int64_t>(rank) * kBT + tid; idx < static_cast<int64_t>(n) * NP;
         idx += static_cast<int64_t>(CS) * kBT) {
        const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
        const double v = j < n ? d.A[i + static_cast<int64_t>(j) * d.lda] : 0.0;
        Bm[idx] = v;
        Vm[idx] = i == j ? 1.0 : 0.0;
        fro += v * v;
    }
    fro = wsum(fro);
    if (lane == 0) s_red[warp] = fro;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kBT / 32; ++w) s += s_red[w];
        aux[rank] = s;
        if (rank == 0) {
            gflag[0] = 0;
            gflag[1] = 0;
        }
    }
    csync();
    double nf2 = 0.0;
    for (int r = 0; r < CS; ++r) nf2 += __ldcg(aux + r);  // other CTAs' stores: read at L2
    const double nf = sqrt(nf2);
    const double eps = DBL_EPSILON;
    const double rel = fmax(tol, sqrt(static_cast<double>(n)) * eps);
    const double floor_col = 4.0 * static_cast<double>(n) * eps * nf;
    const double rel2 = rel * rel, floor2 = floor_col * floor_col;
    const int hl = lane & (kHL - 1), ph = lane >> 4;  // lane within the pair, which pair of the warp

    if (n == 0 || nf == 0.0) {  // jacobi_svd.cpp:47-53: U = I, sigma = 0, V = I
        for (int64_t idx = static_cast<int64_t>(rank) * kBT + tid; idx < static_cast<int64_t>(n) * n;
             idx += static_cast<int64_t>(CS) * kBT) {
            const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
            d.U[idx] = i == j ? 1.0 : 0.0;
            d.V[idx] = i == j ? 1.0 : 0.0;
        }
        if (rank == 0) {
            for (int j = tid; j < n; j += kBT) d.sigma[j] = 0.0;
            if (tid == 0) {
                d.status[0] = 0.0;
                d.status[1] = 0.0;
                d.status[2] = n;
                d.status[3] = 0;
            }
        }
        if (CS > 1) cluster.sync();
        return;
    }

    // my two blocks <-> shared memory (block b's 16 columns -> local columns 16 h .. 16 h + 15):
    // warp w moves local columns w and w + 16, lanes along the rows (coalesced), every load of the
    // warp's 4 RPT in flight before the first store
    constexpr int RL = (RPT + 1) / 2;  // rows per lane when all 32 lanes run along a column
    auto load_blocks = [&](int b0, int b1) {
        double vb[4][RL];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int col = warp + 8 * h;  // local column; block b0 holds 0..15, b1 16..31
            const int64_t g = (static_cast<int64_t>(col < kBW ? b0 : b1) * kBW + (col & (kBW - 1))) * n;
#pragma unroll
            for (int t = 0; t < RL; ++t) {
                const int i = lane + 32 * t;
                vb[h][t] = i < n ? __ldcg(Bm + g + i) : 0.0;
            }
        }
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int t = 0; t < RL; ++t) {
                const int i = lane + 32 * t;
                if (i < n) Bs[(warp + 8 * h) * ldb + i] = vb[h][t];
            }
        for (int e = tid; e < 2 * kBW * 2 * kBW; e += kBT) Js[(e >> 5) * LJ + (e & 31)] = (e >> 5) == (e & 31) ? 1.0 : 0.0;
        __syncthreads();
    };
    // B blocks back to the master; V(:, my 32 columns) <- V(:, my 32 columns) J on the master (a row
    // of V per thread: 32 coalesced loads, 32 x 32 fmas against J from shared memory, 32 stores)
    auto store_blocks = [&](int b0, int b1, bool rotated) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int col = warp + 8 * h;
            const int64_t g = (static_cast<int64_t>(col < kBW ? b0 : b1) * kBW + (col & (kBW - 1))) * n;
#pragma unroll
            for (int t = 0; t < RL; ++t) {
                const int i = lane + 32 * t;
                if (i < n) __stcg(Bm + g + i, Bs[col * ldb + i]);
            }
        }
        if (!rotated) return;  // J = I
        for (int i = tid; i < n; i += kBT) {
            double v[2 * kBW];
#pragma unroll
            for (int k = 0; k < 2 * kBW; ++k)
                v[k] = __ldcg(Vm + (static_cast<int64_t>(k < kBW ? b0 : b1) * kBW + (k & (kBW - 1))) * n + i);
#pragma unroll 2
            for (int c = 0; c < 2 * kBW; ++c) {
                const double* jc = Js + c * LJ;
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int k = 0; k < 2 * kBW; k += 2) {
                    a0 = __fma_rn(v[k], jc[k], a0);
                    a1 = __fma_rn(v[k + 1], jc[k + 1], a1);
                }
                __stcg(Vm + (static_cast<int64_t>(c < kBW ? b0 : b1) * kBW + (c & (kBW - 1))) * n + i, a0 + a1);
            }
        }
    };
    long long* const jtr = (g_jbtrace && blockIdx.x == 0 && tid == 0) ? g_jbtrace : nullptr;
    int gr = 0;  // rounds done (trace index)
    // one sweep: every column pair once; rotate (mode 0) or only track the worst ratio (mode 1)
    auto sweep_once = [&](int mode, double& worst) -> bool {
        bool rot = false;
        const int nsr = NB - 1;
        for (int sr = 0; sr < nsr; ++sr) {
            int b0, b1;
            rrp(NB, sr, rank, b0, b1);
            load_blocks(b0, b1);
            bool rot_sr = false;  // some pair of this super-round rotated (J != I)
            const int nrounds = sr == 0 ? 2 * kBW - 1 : kBW;
            for (int r = 0; r < nrounds; ++r) {
                const int pi = 2 * warp + ph;  // this half-warp's pair of the round
                int lp, lq;
                if (sr == 0) {
                    rrp(2 * kBW, r, pi, lp, lq);
                } else {
                    lp = pi;
                    lq = kBW + ((pi + r) & (kBW - 1));
                }
                if (jtr && gr < 48) jtr[gr * 6 + 0] = clock64();
                const uint32_t bp = bs_a + 8u * static_cast<uint32_t>(lp * ldb + hl);
                const uint32_t bq = bs_a + 8u * static_cast<uint32_t>(lq * ldb + hl);
                double x[RPT], y[RPT];
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int t = 0; t < RPT; ++t) {
                    const bool in = hl + kHL * t < n;
                    x[t] = in ? lds_f64(bp + 8u * (kHL * t)) : 0.0;
                    y[t] = in ? lds_f64(bq + 8u * (kHL * t)) : 0.0;
                    al += x[t] * x[t];
                    be += y[t] * y[t];
                    ga += x[t] * y[t];
                }
                al = hsum(al);
                be = hsum(be);
                ga = hsum(ga);
                if (jtr && gr < 48) jtr[gr * 6 + 1] = clock64();
                const bool skip = jskip(al, be, ga, rel2, floor2);
                if (mode == 1) {
                    if (!(al <= floor2 || be <= floor2)) worst = fmax(worst, fabs(ga) / sqrt(al * be));
                } else if (__any_sync(0xffffffffu, !skip)) {
                    double c = 1.0, s = 0.0;
                    jrot(al, be, ga, c, s);
                    if (jtr && gr < 48) jtr[gr * 6 + 2] = clock64();
                    if (!skip) {
                        rot = true;
                        rot_sr = true;
#pragma unroll
                        for (int t = 0; t < RPT; ++t) {
                            if (hl + kHL * t < n) {
                                sts_f64(bp + 8u * (kHL * t), c * x[t] - s * y[t]);
                                sts_f64(bq + 8u * (kHL * t), s * x[t] + c * y[t]);
                            }
                        }
                        const uint32_t jp = js_a + 8u * static_cast<uint32_t>(lp * LJ + hl);
                        const uint32_t jq = js_a + 8u * static_cast<uint32_t>(lq * LJ + hl);
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const double vx = lds_f64(jp + 8u * (kHL * t)), vy = lds_f64(jq + 8u * (kHL * t));
                            sts_f64(jp + 8u * (kHL * t), c * vx - s * vy);
                            sts_f64(jq + 8u * (kHL * t), s * vx + c * vy);
                        }
                    }
                }
                if (jtr && gr < 48) jtr[gr * 6 + 3] = clock64();
                __syncthreads();
                if (jtr && gr < 48) jtr[gr * 6 + 4] = clock64();
                ++gr;
            }
            if (mode == 0) {
                const bool srot = __syncthreads_or(rot_sr ? 1 : 0) != 0;
                store_blocks(b0, b1, srot);
            }
            csync();
            if (jtr && gr < 48) jtr[gr * 6 + 5] = clock64();
        }
        return rot;
    };

    bool converged = false;
    int sweep = 0;
    double worst = 0.0;
    for (; sweep < max_sweeps && !converged; ++sweep) {
        const bool rot = sweep_once(0, worst);
        // cluster-wide OR of "some pair rotated" through a global flag, two flags alternating
        const int any = __syncthreads_or(rot ? 1 : 0);
        if (tid == 0 && any) atomicOr(&gflag[sweep & 1], 1);
        csync();
        const int f = *reinterpret_cast<volatile int*>(&gflag[sweep & 1]);
        if (rank == 0 && tid == 0) gflag[(sweep + 1) & 1] = 0;
        converged = f == 0;
        csync();
    }

    if (!converged) {  // residual: worst remaining pair ratio (jacobi_svd.cpp:97-109)
        sweep_once(1, worst);
        worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, 16));
        if (lane == 0) s_red[warp] = worst;
        __syncthreads();
        if (tid == 0) {
            double m = 0.0;
            for (int w = 0; w < kBT / 32; ++w) m = fmax(m, s_red[w]);
            aux[rank] = m;
        }
        csync();
        if (rank == 0 && tid == 0) {
            double m = 0.0;
            for (int r = 0; r < CS; ++r) m = fmax(m, __ldcg(aux + r));
            d.status[0] = RUTV_ERR_CONVERGENCE;
            d.status[1] = m;
            d.status[2] = n;
            d.status[3] = sweep;
        }
        if (CS > 1) cluster.sync();
        return;
    }

    // sigma_j = ||b_j||: CTA c takes blocks 2c, 2c + 1 (four columns per warp)
    load_blocks(2 * rank, 2 * rank + 1);
    for (int col = warp; col < 2 * kBW; col += kBT / 32) {
        const double* b = Bs + col * ldb;
        double a = 0.0;
        for (int i = lane; i < n; i += 32) a += b[i] * b[i];
        a = wsum(a);
        if (lane == 0) sig[2 * rank * kBW + col] = sqrt(a);
    }
    csync();
    // stable descending rank of each of my columns among the n real ones, then write out
    __shared__ int s_dest[2 * kBW];
    __shared__ double s_sig[2 * kBW];
    if (tid < 2 * kBW) {
        const int j = 2 * rank * kBW + tid;
        int t = -1;
        double sj = 0.0;
        if (j < n) {
            sj = __ldcg(sig + j);
            t = 0;
            for (int k = 0; k < n; ++k) {
                const double sk = __ldcg(sig + k);
                t += (sk > sj) || (k < j && sk == sj);
            }
        }
        s_dest[tid] = t;
        s_sig[tid] = sj;
    }
    __syncthreads();
    for (int col = 0; col < 2 * kBW; ++col) {
        const int t = s_dest[col];
        if (t < 0) continue;
        const double s = s_sig[col];
        for (int i = tid; i < n; i += kBT) {
            d.V[i + static_cast<int64_t>(t) * n] = __ldcg(Vm + (static_cast<int64_t>(2 * rank) * kBW + col) * n + i);
            d.U[i + static_cast<int64_t>(t) * n] = s > floor_col ? Bs[col * ldb + i] / s : 0.0;
        }
        if (tid == 0) d.sigma[t] = s;
    }
    if (rank == 0 && tid == 0) {
        int kept = 0;
        for (int j = 0; j < n; ++j) kept += __ldcg(sig + j) > floor_col;
        d.status[0] = 0.0;
        d.status[1] = 0.0;
        d.status[2] = kept;
        d.status[3] = sweep;
    }
    if (CS > 1) cluster.sync();
}

int blk_nb(int n) { return n <= 32 ? 2 : n <= 64 ? 4 : n <= 128 ? 8 : n <= 256 ? 16 : 32; }

template <int RPT>
void launch_blk(cudaStream_t stream, const SvdDesc* d, int count, int NB, int ldb, size_t smem, double tol,
                int max_sweeps) {
    auto k = jacobi_blk_kernel<RPT>;
    once_per_device(reinterpret_cast<const void*>(k), [k] {
        RUTV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));  // 16 CTAs at n = 512
        RUTV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       dyn_smem_cap(reinterpret_cast<const void*>(k))));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(count * (NB / 2)));
    cfg.blockDim = dim3(kBT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = static_cast<unsigned>(NB / 2);
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    static const bool jtrace = std::getenv("RUTV_JAC_TRACE") != nullptr;
    long long* dtr = nullptr;
    if (jtrace) {
        RUTV_CUDA(cudaMalloc(&dtr, 49 * 6 * sizeof(long long)));
        RUTV_CUDA(cudaMemset(dtr, 0, 49 * 6 * sizeof(long long)));
        RUTV_CUDA(cudaMemcpyToSymbol(g_jbtrace, &dtr, sizeof(dtr)));
    }
    RUTV_CUDA(cudaLaunchKernelEx(&cfg, k, d, NB, ldb, tol, max_sweeps));
    if (jtrace) {
        long long h[49 * 6];
        RUTV_CUDA(cudaStreamSynchronize(stream));
        RUTV_CUDA(cudaMemcpy(h, dtr, sizeof(h), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "jacobi_blk trace NB=%d (cycles: dots, decide, rotate, barrier; exchange after the super-round)\n", NB);
        for (int r = 0; r < 48; ++r)
            std::fprintf(stderr, "  round %2d: %6lld %6lld %6lld %6lld   %6lld\n", r, h[r * 6 + 1] - h[r * 6], h[r * 6 + 2] - h[r * 6 + 1],
                         h[r * 6 + 3] - h[r * 6 + 2], h[r * 6 + 4] - h[r * 6 + 3], h[r * 6 + 5] ? h[r * 6 + 5] - h[(r - 1) * 6 + 4] : 0LL);
        long long* z = nullptr;
        RUTV_CUDA(cudaMemcpyToSymbol(g_jbtrace, &z, sizeof(z)));
        cudaFree(dtr);
    }
}

}  // namespace

// Work doubles the column-distributed kernel needs for an n x n problem inside a batch whose
// largest block is <= 512 wide: two n x 512 master copies, sigma, scratch (jacobi.cu adds its own).
int64_t svd_blk_work_elems(int64_t n) { return n <= 512 ? 2 * n * 512 + 512 + 64 : 0; }

// nmax <= 512 and not disabled (RUTV_JACOBI=rows selects the row-distributed kernel of jacobi.cu)
bool svd_blk_applicable(int nmax) {
    static const bool off = [] {
        const char* e = std::getenv("RUTV_JACOBI");
        return e && std::strcmp(e, "rows") == 0;
    }();
    return !off && nmax >= 1 && nmax <= 512;
}

void svd_batch_blk(cudaStream_t stream, const SvdDesc* d_descs, int count, int nmax, double tol, int max_sweeps) {
    const int NB = blk_nb(nmax);
    const int rpt = (nmax + kHL - 1) / kHL;
    const int RPT = rpt <= 2 ? 2 : rpt <= 4 ? 4 : rpt <= 8 ? 8 : rpt <= 16 ? 16 : 32;
    const int ldb = kHL * RPT + 1;
    const size_t smem = (static_cast<size_t>(2 * kBW) * ldb + static_cast<size_t>(2 * kBW) * (2 * kBW + 1)) * sizeof(double);
    switch (RPT) {
        case 2: launch_blk<2>(stream, d_descs, count, NB, ldb, smem, tol, max_sweeps); break;
        case 4: launch_blk<4>(stream, d_descs, count, NB, ldb, smem, tol, max_sweeps); break;
        case 8: launch_blk<8>(stream, d_descs, count, NB, ldb, smem, tol, max_sweeps); break;
        case 16: launch_blk<16>(stream, d_descs, count, NB, ldb, smem, tol, max_sweeps); break;
        default: launch_blk<32>(stream, d_descs, count, NB, ldb, smem, tol, max_sweeps); break;
    }
    note_launch();
    RUTV_CHECK_LAUNCH();
}

}  // namespace rutv
