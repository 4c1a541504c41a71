// gemm_f64.cu -- FP64 tensor-core GEMM for sm_100a (warp-level DMMA).
//
// Replaces the reference's single scalar gemm (proj/src/gemm.cpp:21-75,
// contract proj/include/randutv/matrix_ops.hpp:9-18), which carries 95% of
// the reference's wall time.  On sm_100a the only FP64
// tensor path is the legacy warp-level mma.sync .f64 (ptxas rejects
// tcgen05.mma kind::f64); every PTX shape lowers to SASS DMMA.8x8x4 and all
// reach the same measured peak (profiles/r01_dmma_peak.jsonl: 37.1 TF/s), so
// the kernel issues m16n8k4 and spends its effort on feeding it:
//   * cp.async multistage shared-memory pipeline (3 stages), 16-byte chunks
//     when operands are 16-byte aligned, 8-byte otherwise (odd b / ld);
//   * smem tiles stored in the operand's contiguous global direction with a
//     +4-double pad so every fragment load is bank-conflict free for all four
//     transpose combinations;
//   * main tile 128 x 64, 4 warps of 64 x 32, BK = 16, two CTAs per SM: one
//     CTA's k-tile barrier and epilogue hide behind the other's DMMAs; with
//     beta != 0 the C tile is staged through shared memory by cp.async (all
//     loads in flight at once) instead of per-element register loads;
//   * 64 x 64 tiles (4 warps of 32 x 32, C prefetched into registers) with a
//     deterministic split-K for the skinny K = s products (one side = b);
//   * split-K partials are summed in a fixed order by a separate kernel, so
//     results are bit-reproducible run to run.
// Measured (tools/gemm_bench.py, tools/gemm_c5.py; DESIGN.md GEMM table): 34.5 TF/s
// at 8192^3 (93 % of the DMMA peak; cuBLAS's sm_80 d884 kernel 35.5), 33.3 at the
// config-5 rank-512 update 50000^2 x 512 (cuBLAS 27.8), 35.1 at the config-5 sketch
// 50000 x 512 x 50000 (cuBLAS 36.2), 25.0 at the rank-128 update 4000^2 x 128.
// Tried and measured slower: 128 x 128 tiles on one CTA per SM (29.4 at the config-5
// update), 4 pipeline stages, red.global.add epilogues for beta = 1.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_count() { return g_launches.load(); }
void note_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

// Optional per-launch GEMM timing (RUTV_GEMM_PROFILE=1): CUDA events on the
// launching stream around every gemm() call, algorithmic flops 2MNK.
namespace {
struct GemmProf {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // pairs
    double flops_acc = 0.0;
    double flops = 0.0, ms = 0.0;
    int64_t launches = 0;
};
thread_local GemmProf g_gp;
}  // namespace

void gemm_profile_begin() {
    const char* e = std::getenv("RUTV_GEMM_PROFILE");
    g_gp.on = e && std::strcmp(e, "0") != 0;
    g_gp.ev.clear();
    g_gp.flops_acc = 0.0;
}

void gemm_profile_end() {
    if (!g_gp.on) return;
    if (!g_gp.ev.empty()) cudaEventSynchronize(g_gp.ev.back());
    double ms = 0.0;
    for (size_t i = 0; i + 1 < g_gp.ev.size(); i += 2) {
        float t = 0.f;
        cudaEventElapsedTime(&t, g_gp.ev[i], g_gp.ev[i + 1]);
        ms += t;
    }
    for (auto e : g_gp.ev) cudaEventDestroy(e);
    g_gp.flops = g_gp.flops_acc;
    g_gp.ms = ms;
    g_gp.launches = static_cast<int64_t>(g_gp.ev.size() / 2);
    g_gp.ev.clear();
    g_gp.on = false;
}

int gemm_profile_get(double* flops, double* ms, int64_t* launches) {
    if (flops) *flops = g_gp.flops;
    if (ms) *ms = g_gp.ms;
    if (launches) *launches = g_gp.launches;
    return g_gp.launches > 0 ? 1 : 0;
}

namespace {
struct ProfScope {
    cudaStream_t st;
    bool on;
    ProfScope(cudaStream_t s, double flops) : st(s), on(g_gp.on) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        g_gp.ev.push_back(e);
        g_gp.flops_acc += flops;
    }
    ~ProfScope() {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        g_gp.ev.push_back(e);
    }
};
}  // namespace

struct GemmParams {
    int64_t M, N, K;
    const double* A;
    int64_t lda;
    const double* B;
    int64_t ldb;
    double* C;
    int64_t ldc;
    double alpha, beta;
    double* work;
    int64_t kchunk;
    int splits;
    int cvec;  // C 16-byte aligned with an even ldc: 16-byte cp.async for the C tile
    // Tile rasterisation: blockIdx.x runs over groups of `group_m` tile rows, the
    // tile rows of a group fastest, so the CTAs resident at one time cover a compact
    // group_m x (wave / group_m) block of output tiles and their A and B k-slabs
    // are shared through L2 instead of re-streamed from HBM (at config 5 an
    // M-fastest raster re-reads a 205 MB panel once per 64-column tile).
    int tiles_m, tiles_n, group_m;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_16x8x4(double* c, const double* a, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(b));
}

template <int BM, int BN, int BK, bool TA, bool TB>
struct SmemGeom {
    static constexpr int A_LD = TA ? (BK + 4) : (BM + 4);
    static constexpr int A_SZ = TA ? BM * A_LD : BK * A_LD;
    static constexpr int B_LD = TB ? (BN + 4) : (BK + 4);
    static constexpr int B_SZ = TB ? BK * B_LD : BN * B_LD;
    static constexpr int C_LD = BM + 4;  // (2 C_LD) mod 16 == 8: conflict-free fragment reads
    static constexpr int C_SZ = BN * C_LD;
};

// Large warp tiles read C in the epilogue through shared memory (see below).
template <int WM, int WN>
constexpr bool gemm_prefetch_c() { return (WM / 16) * (WN / 8) * 4 <= 32; }

// Resident CTAs per SM the tile is built for: 4-warp tiles run two CTAs per SM
// so one CTA's k-tile barrier and epilogue hide behind the other's DMMAs.
template <int BM, int BN, int WM, int WN>
constexpr int gemm_min_blocks() { return (BM / WM) * (BN / WN) <= 4 ? 2 : 1; }

template <int BM, int BN, int BK, int WM, int WN, int ST, bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, (gemm_min_blocks<BM, BN, WM, WN>()))
    dgemm_kernel(const GemmParams p) {
    constexpr int NWM = BM / WM, NWN = BN / WN, NT = NWM * NWN * 32;
    constexpr int MI = WM / 16, NI = WN / 8;
    using G = SmemGeom<BM, BN, BK, TA, TB>;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + ST * G::A_SZ;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % NWM, wn = warp / NWM;
    const int g = lane >> 2, t = lane & 3;
    int64_t m0, n0;
    {
        const int per_group = p.group_m * p.tiles_n;
        const int grp = static_cast<int>(blockIdx.x) / per_group;
        const int first = grp * p.group_m;
        const int gsz = min(p.group_m, p.tiles_m - first);
        const int r = static_cast<int>(blockIdx.x) - grp * per_group;
        m0 = static_cast<int64_t>(first + r % gsz) * BM;
        n0 = static_cast<int64_t>(r / gsz) * BN;
    }
    const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * p.kchunk;
    const int64_t kend = min(p.K, kbeg + p.kchunk);
    const int KT = kend > kbeg ? static_cast<int>((kend - kbeg + BK - 1) / BK) : 0;
    const int64_t M = p.M, N = p.N;

    auto load_tile = [&](int stage, int64_t k0) {
        double* as = As + stage * G::A_SZ;
        double* bs = Bs + stage * G::B_SZ;
        if constexpr (!TA) {  // op(A)(m,k) = A[m + k*lda]; smem as[k][m]
            if constexpr (VEC) {
                for (int c = tid; c < BK * BM / 2; c += NT) {
                    const int k = c / (BM / 2), mm = (c % (BM / 2)) * 2;
                    const int64_t gm = m0 + mm, gk = k0 + k;
                    int bytes = 0;
                    const double* src = p.A;
                    if (gk < kend && gm < M) {
                        bytes = gm + 1 < M ? 16 : 8;
                        src = p.A + gm + gk * p.lda;
                    }
                    cp_async16(as + k * G::A_LD + mm, src, bytes);
                }
            } else {
                for (int c = tid; c < BK * BM; c += NT) {
                    const int k = c / BM, mm = c % BM;
                    const int64_t gm = m0 + mm, gk = k0 + k;
                    const bool ok = gk < kend && gm < M;
                    cp_async8(as + k * G::A_LD + mm, ok ? p.A + gm + gk * p.lda : p.A, ok ? 8 : 0);
                }
            }
        } else {  // op(A)(m,k) = A[k + m*lda]; smem as[m][k]
            if constexpr (VEC) {
                for (int c = tid; c < BM * BK / 2; c += NT) {
                    const int mm = c / (BK / 2), kk = (c % (BK / 2)) * 2;
                    const int64_t gm = m0 + mm, gk = k0 + kk;
                    int bytes = 0;
                    const double* src = p.A;
                    if (gk < kend && gm < M) {
                        bytes = gk + 1 < kend ? 16 : 8;
                        src = p.A + gk + gm * p.lda;
                    }
                    cp_async16(as + mm * G::A_LD + kk, src, bytes);
                }
            } else {
                for (int c = tid; c < BM * BK; c += NT) {
                    const int mm = c / BK, kk = c % BK;
                    const int64_t gm = m0 + mm, gk = k0 + kk;
                    const bool ok = gk < kend && gm < M;
                    cp_async8(as + mm * G::A_LD + kk, ok ? p.A + gk + gm * p.lda : p.A, ok ? 8 : 0);
                }
            }
        }
        if constexpr (!TB) {  // op(B)(k,n) = B[k + n*ldb]; smem bs[n][k]
            if constexpr (VEC) {
                for (int c = tid; c < BN * BK / 2; c += NT) {
                    const int nn = c / (BK / 2), kk = (c % (BK / 2)) * 2;
                    const int64_t gn = n0 + nn, gk = k0 + kk;
                    int bytes = 0;
                    const double* src = p.B;
                    if (gk < kend && gn < N) {
                        bytes = gk + 1 < kend ? 16 : 8;
                        src = p.B + gk + gn * p.ldb;
                    }
                    cp_async16(bs + nn * G::B_LD + kk, src, bytes);
                }
            } else {
                for (int c = tid; c < BN * BK; c += NT) {
                    const int nn = c / BK, kk = c % BK;
                    const int64_t gn = n0 + nn, gk = k0 + kk;
                    const bool ok = gk < kend && gn < N;
                    cp_async8(bs + nn * G::B_LD + kk, ok ? p.B + gk + gn * p.ldb : p.B, ok ? 8 : 0);
                }
            }
        } else {  // op(B)(k,n) = B[n + k*ldb]; smem bs[k][n]
            if constexpr (VEC) {
                for (int c = tid; c < BK * BN / 2; c += NT) {
                    const int k = c / (BN / 2), nn = (c % (BN / 2)) * 2;
                    const int64_t gn = n0 + nn, gk = k0 + k;
                    int bytes = 0;
                    const double* src = p.B;
                    if (gk < kend && gn < N) {
                        bytes = gn + 1 < N ? 16 : 8;
                        src = p.B + gn + gk * p.ldb;
                    }
                    cp_async16(bs + k * G::B_LD + nn, src, bytes);
                }
            } else {
                for (int c = tid; c < BK * BN; c += NT) {
                    const int k = c / BN, nn = c % BN;
                    const int64_t gn = n0 + nn, gk = k0 + k;
                    const bool ok = gk < kend && gn < N;
                    cp_async8(bs + k * G::B_LD + nn, ok ? p.B + gn + gk * p.ldb : p.B, ok ? 8 : 0);
                }
            }
        }
    };

    double acc[MI][NI][4];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;

    // beta != 0: prefetch this thread's C fragment now so the epilogue's
    // read-modify-write does not serialise on global-load latency (the
    // rank-b updates have K = b, a mainloop of only a few k-tiles).
    // (Large warp tiles would need 2x the accumulator registers for it: they
    // read C in the epilogue and rely on the second resident CTA instead.)
    constexpr bool PRE = gemm_prefetch_c<WM, WN>();
    const bool direct = p.splits == 1;
    const bool use_c = direct && p.beta != 0.0;
    double cpre[PRE ? MI : 1][PRE ? NI : 1][4];
    if constexpr (PRE) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int64_t m = m0 + wm * WM + mi * 16 + g + (r >= 2 ? 8 : 0);
                    const int64_t n = n0 + wn * WN + ni * 8 + 2 * t + (r & 1);
                    cpre[mi][ni][r] = (use_c && m < M && n < N) ? __ldg(p.C + m + n * p.ldc) : 0.0;
                }
    }

    // Fast loads (16-byte path), full k-tiles.  Thread `tid` owns chunks
    // c = tid + i*NT of each operand tile.  With NT a multiple of the chunk-row
    // width, chunk i sits at the thread's first chunk plus i fixed rows (k rows
    // for an m-contiguous tile, m rows for a k-contiguous one), so one base
    // pointer, one global and one shared stride describe all of them: a k-tile
    // is a pointer bump and ACH + BCH cp.async (the per-chunk pointer tables of
    // the previous version held ~48 registers the fragment double buffer needs).
    // The generic load_tile keeps the partial last tile and unaligned operands.
    constexpr int ACW = TA ? BK / 2 : BM / 2;  // 16-byte chunks per tile row (k-contiguous: per m row)
    constexpr int BCW = TB ? BN / 2 : BK / 2;
    static_assert(NT % ACW == 0 && NT % BCW == 0, "chunk rows must tile the CTA");
    constexpr int ARS = NT / ACW, BRS = NT / BCW;  // rows advanced per chunk index
    constexpr int ACH = VEC ? (BK * BM / 2 + NT - 1) / NT : 1;
    constexpr int BCH = VEC ? (BK * BN / 2 + NT - 1) / NT : 1;
    const int a_r0 = tid / ACW, a_c0 = (tid % ACW) * 2;  // (row, col) of chunk 0 in the smem tile
    const int b_r0 = tid / BCW, b_c0 = (tid % BCW) * 2;
    // A: TA -> rows are m, cols k (as[m][k]); !TA -> rows are k, cols m (as[k][m])
    const int64_t a_gm0 = m0 + (TA ? a_r0 : a_c0), a_gk0 = kbeg + (TA ? a_c0 : a_r0);
    const int64_t b_gn0 = n0 + (TB ? b_c0 : b_r0), b_gk0 = kbeg + (TB ? b_r0 : b_c0);
    const double* a_base = p.A + (TA ? a_gk0 + a_gm0 * p.lda : a_gm0 + a_gk0 * p.lda);
    const double* b_base = p.B + (TB ? b_gn0 + b_gk0 * p.ldb : b_gk0 + b_gn0 * p.ldb);
    const int64_t a_gs = static_cast<int64_t>(ARS) * p.lda, b_gs = static_cast<int64_t>(BRS) * p.ldb;
    const int a_so = a_r0 * G::A_LD + a_c0, b_so = b_r0 * G::B_LD + b_c0;
    // m-contiguous A / n-contiguous B: every chunk has the same m (n) pair -> one byte count
    const int a_bytes = a_gm0 < M ? (a_gm0 + 1 < M ? 16 : 8) : 0;
    const int b_bytes = b_gn0 < N ? (b_gn0 + 1 < N ? 16 : 8) : 0;
    const int64_t astep = TA ? BK : BK * p.lda, bstep = TB ? BK * p.ldb : BK;
    // Large warp tiles (registers to spare, 16 DMMAs per k-step) keep a table of
    // per-chunk pointers -- measured 2 % faster there (8192^3: 34.4 vs 33.8 TF/s);
    // small warp tiles use the compact plan and spend the registers on the
    // fragment double buffer (4000 x 128 x 4000: 28.9 vs 26.6 TF/s).
    constexpr bool TABLE = !(MI * NI <= 8);
    const double* agp[TABLE ? ACH : 1];
    const double* bgp[TABLE ? BCH : 1];
    int aby[TABLE ? ACH : 1], bby[TABLE ? BCH : 1];
    if constexpr (TABLE && VEC) {
#pragma unroll
        for (int i = 0; i < ACH; ++i) {
            const int64_t gm = a_gm0 + (TA ? i * ARS : 0);
            const bool ok = tid + i * NT < BK * BM / 2 && gm < M;
            aby[i] = !ok ? 0 : (!TA && gm + 1 >= M ? 8 : 16);
            agp[i] = ok ? a_base + i * a_gs : p.A;
        }
#pragma unroll
        for (int i = 0; i < BCH; ++i) {
            const int64_t gn = b_gn0 + (TB ? 0 : i * BRS);
            const bool ok = tid + i * NT < BK * BN / 2 && gn < N;
            bby[i] = !ok ? 0 : (TB && gn + 1 >= N ? 8 : 16);
            bgp[i] = ok ? b_base + i * b_gs : p.B;
        }
    }
    auto load = [&](int stage, int kt) {
        const int64_t k0 = kbeg + static_cast<int64_t>(kt) * BK;
        if (VEC && k0 + BK <= kend) {
            double* as = As + stage * G::A_SZ;
            double* bs = Bs + stage * G::B_SZ;
            if constexpr (TABLE) {
#pragma unroll
                for (int i = 0; i < ACH; ++i)
                    if (BK * BM / 2 % NT == 0 || tid + i * NT < BK * BM / 2)
                        cp_async16(as + a_so + i * ARS * G::A_LD, aby[i] ? agp[i] + kt * astep : p.A, aby[i]);
#pragma unroll
                for (int i = 0; i < BCH; ++i)
                    if (BK * BN / 2 % NT == 0 || tid + i * NT < BK * BN / 2)
                        cp_async16(bs + b_so + i * BRS * G::B_LD, bby[i] ? bgp[i] + kt * bstep : p.B, bby[i]);
            } else {
                const double* ab = a_base + kt * astep;
                const double* bb = b_base + kt * bstep;
#pragma unroll
                for (int i = 0; i < ACH; ++i)
                    if (BK * BM / 2 % NT == 0 || tid + i * NT < BK * BM / 2) {
                        // k-contiguous A: chunk i covers m row a_gm0 + i*ARS (all of its k in range)
                        const int by = TA ? (a_gm0 + i * ARS < M ? 16 : 0) : a_bytes;
                        cp_async16(as + a_so + i * ARS * G::A_LD, by ? ab + i * a_gs : p.A, by);
                    }
#pragma unroll
                for (int i = 0; i < BCH; ++i)
                    if (BK * BN / 2 % NT == 0 || tid + i * NT < BK * BN / 2) {
                        const int by = TB ? b_bytes : (b_gn0 + i * BRS < N ? 16 : 0);
                        cp_async16(bs + b_so + i * BRS * G::B_LD, by ? bb + i * b_gs : p.B, by);
                    }
            }
        } else {
            load_tile(stage, k0);
        }
    };
    for (int s = 0; s < ST - 1; ++s) {
        if (s < KT) load(s, s);
        cp_async_commit();
    }
    // Fragments are double-buffered across the four k-steps of a tile: the
    // shared-memory loads of step kk+4 are in flight while the DMMAs of step kk
    // issue (short-scoreboard stalls were the largest non-math stall).
    // (small warp tiles only: the 64 x 32 warp tile's 16 independent DMMAs per
    // k-step already hide the shared-memory latency, and its registers are tight)
    constexpr bool FDB = MI * NI <= 8;
    double af[FDB ? 2 : 1][MI][2], bf[FDB ? 2 : 1][NI];
    int rd = 0, wr = ST - 1;  // stage read this iteration / written by its prefetch
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        const int nk = kt + ST - 1;
        if (nk < KT) load(wr, nk);
        cp_async_commit();
        wr = wr + 1 == ST ? 0 : wr + 1;
        const double* as = As + rd * G::A_SZ;
        const double* bs = Bs + rd * G::B_SZ;
        rd = rd + 1 == ST ? 0 : rd + 1;
        auto frag = [&](int buf, int kk) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int mr = wm * WM + mi * 16 + g + 8 * h, kc = kk + t;
                    af[buf][mi][h] = TA ? as[mr * G::A_LD + kc] : as[kc * G::A_LD + mr];
                }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const int nc = wn * WN + ni * 8 + g, kr = kk + t;
                bf[buf][ni] = TB ? bs[kr * G::B_LD + nc] : bs[nc * G::B_LD + kr];
            }
        };
        if constexpr (FDB) {
            frag(0, 0);
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                const int cur = (kk / 4) & 1;
                if (kk + 4 < BK) frag(cur ^ 1, kk + 4);
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) dmma_16x8x4(acc[mi][ni], af[cur][mi], bf[cur][ni]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                frag(0, kk);
#pragma unroll
                for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) dmma_16x8x4(acc[mi][ni], af[0][mi], bf[0][ni]);
            }
        }
    }
    cp_async_wait<0>();

    double* wbase = p.work + static_cast<int64_t>(blockIdx.z) * M * N;
    // beta != 0 without the register prefetch: the C tile is staged through
    // shared memory (the pipeline stages are free now) with every cp.async in
    // flight at once -- register pressure would otherwise make the compiler
    // serialise one HBM round trip per element.  The second resident CTA of
    // the SM keeps the DMMA pipe busy meanwhile.
    if constexpr (!PRE) {
        if (use_c) {
            __syncthreads();  // every warp is done with the last k-tile
            double* cs = smem;
            if (p.cvec) {
                for (int c = tid; c < BN * (BM / 2); c += NT) {
                    const int nn = c / (BM / 2), mm = (c % (BM / 2)) * 2;
                    const int64_t gm = m0 + mm, gn = n0 + nn;
                    int bytes = 0;
                    const double* src = p.C;
                    if (gn < N && gm < M) {
                        bytes = gm + 1 < M ? 16 : 8;
                        src = p.C + gm + gn * p.ldc;
                    }
                    cp_async16(cs + nn * G::C_LD + mm, src, bytes);
                }
            } else {
                for (int c = tid; c < BN * BM; c += NT) {
                    const int nn = c / BM, mm = c % BM;
                    const int64_t gm = m0 + mm, gn = n0 + nn;
                    const bool ok = gn < N && gm < M;
                    cp_async8(cs + nn * G::C_LD + mm, ok ? p.C + gm + gn * p.ldc : p.C, ok ? 8 : 0);
                }
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int ml = wm * WM + mi * 16 + g + (r >= 2 ? 8 : 0);
                        const int nl = wn * WN + ni * 8 + 2 * t + (r & 1);
                        acc[mi][ni][r] = p.alpha * acc[mi][ni][r] + p.beta * cs[nl * G::C_LD + ml];
                    }
        } else if (direct) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[mi][ni][r] *= p.alpha;
        }
    } else if (direct) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    double v = p.alpha * acc[mi][ni][r];
                    if (use_c) v += p.beta * cpre[mi][ni][r];
                    acc[mi][ni][r] = v;
                }
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t m = m0 + wm * WM + mi * 16 + g + (r >= 2 ? 8 : 0);
                const int64_t n = n0 + wn * WN + ni * 8 + 2 * t + (r & 1);
                if (m < M && n < N) {
                    if (direct)
                        p.C[m + n * p.ldc] = acc[mi][ni][r];
                    else
                        wbase[m + n * M] = acc[mi][ni][r];
                }
            }
}

__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const double* __restrict__ work,
                                     double* C, int64_t ldc, double alpha, double beta) {
    const int64_t total = M * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int sp = 0; sp < splits; ++sp) s += work[sp * total + i];
        const int64_t m = i % M, n = i / M;
        double* cp = C + m + n * ldc;
        double v = alpha * s;
        if (beta != 0.0) v += beta * *cp;
        *cp = v;
    }
}

__global__ void scale_kernel(int64_t M, int64_t N, double* C, int64_t ldc, double beta) {
    const int64_t total = M * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = i % M, n = i / M;
        double* cp = C + m + n * ldc;
        *cp = beta == 0.0 ? 0.0 : beta * *cp;
    }
}

namespace {

// Rows of tiles per raster group (GemmParams::group_m).  Among the CTAs resident at
// once (two per SM), A k-slab traffic scales with the tile rows they cover and B
// with the tile columns: balance BM * rows = BN * cols, rows * cols = the wave; when
// the product is narrow (N = b: few tile columns) take every column and as many
// rows as fill the wave.  RUTV_GEMM_RASTER=0 restores the plain M-fastest raster.
int raster_group(int tiles_m, int tiles_n, int bm, int bn) {
    static const bool on = [] {
        const char* e = std::getenv("RUTV_GEMM_RASTER");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (!on) return std::max(tiles_m, 1);
    const double wave = 2.0 * kNumSMs;
    int gm = static_cast<int>(std::lround(std::sqrt(wave * bn / bm)));
    if (static_cast<double>(tiles_n) * gm < wave) gm = static_cast<int>(std::ceil(wave / tiles_n));
    return std::max(1, std::min(gm, tiles_m));
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool TA, bool TB, bool VEC>
void launch_cfg(cudaStream_t stream, const GemmParams& pin, int gx, int gy, int gz) {
    GemmParams p = pin;
    p.tiles_m = gx;
    p.tiles_n = gy;
    p.group_m = raster_group(gx, gy, BM, BN);
    using G = SmemGeom<BM, BN, BK, TA, TB>;
    constexpr int stages = ST * (G::A_SZ + G::B_SZ);
    constexpr int smem = (gemm_prefetch_c<WM, WN>() || stages >= G::C_SZ ? stages : G::C_SZ) *
                         static_cast<int>(sizeof(double));
    constexpr int nt = (BM / WM) * (BN / WN) * 32;
    auto kern = dgemm_kernel<BM, BN, BK, WM, WN, ST, TA, TB, VEC>;
    // per instantiation and per device (the opt-in is a property of the device context)
    once_per_device(reinterpret_cast<const void*>(kern), [kern] {
        RUTV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    });
    kern<<<dim3(static_cast<unsigned>(static_cast<int64_t>(gx) * gy), 1, gz), nt, smem, stream>>>(p);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

template <int BM, int BN, int BK, int WM, int WN, int ST>
void dispatch(cudaStream_t stream, const GemmParams& p, bool ta, bool tb, bool vec, int gz) {
    const int gx = static_cast<int>((p.M + BM - 1) / BM), gy = static_cast<int>((p.N + BN - 1) / BN);
#define RUTV_G(TA_, TB_, V_) \
    launch_cfg<BM, BN, BK, WM, WN, ST, TA_, TB_, V_>(stream, p, gx, gy, gz)
    if (vec) {
        if (!ta && !tb) RUTV_G(false, false, true);
        else if (!ta && tb) RUTV_G(false, true, true);
        else if (ta && !tb) RUTV_G(true, false, true);
        else RUTV_G(true, true, true);
    } else {
        if (!ta && !tb) RUTV_G(false, false, false);
        else if (!ta && tb) RUTV_G(false, true, false);
        else if (ta && !tb) RUTV_G(true, false, false);
        else RUTV_G(true, true, false);
    }
#undef RUTV_G
}

inline bool aligned16(const void* ptr, int64_t ld) {
    return (reinterpret_cast<uintptr_t>(ptr) % 16 == 0) && (ld % 2 == 0);
}

constexpr int kBK = 16;

// Tile config + split-K plan.  Large 128x128 tiles (8 warps, 1 CTA/SM) when
// the output tiles -- times a split-K factor for long K -- fill about one
// wave of 148 SMs; otherwise 64x64 tiles (several CTAs/SM) with split-K.
struct GemmPlan {
    bool large;  // 128 x 64 tiles (4 warps, 2 CTAs/SM); else 64 x 64 (legacy plan only)
    int splits;
};

int gemm_plan_mode() {  // RUTV_GEMM_PLAN=1: the 64 x 64 split-K plan for every short-tile product
    static int m = [] {
        const char* e = std::getenv("RUTV_GEMM_PLAN");
        return e ? std::atoi(e) : 0;
    }();
    return m;
}

// Tile + deterministic split-K plan.  128 x 64 tiles run two CTAs per SM
// (296 slots).  Enough tiles (>= 3 waves) or a short K (the rank-b updates):
// no split.  Otherwise (the K = s sketch / projection products, m or n = b)
// split K so the launch fills about two waves, each split at least 256 deep.
// Split count for `tiles` output tiles over K: minimise a wave model --
// ceil(tiles * sp / slots) waves of CTAs that each run K / sp deep (DMMA time
// at half an SM, plus a fixed prologue / epilogue cost), plus the split-K
// reduction's HBM traffic (sp partial M x N planes read, C written).
int choose_splits(int64_t M, int64_t N, int64_t K, int64_t tiles, int64_t tile_flops_per_k, int64_t slots,
                  int64_t maxsp) {
    const double clk = 1.965e9, sm_rate = 127.6 / 2.0;  // flop/clk for one of two resident CTAs
    double best = 1e300;
    int bsp = 1;
    for (int64_t sp = 1; sp <= maxsp; ++sp) {
        const double chunk = static_cast<double>((K + sp - 1) / sp);
        const double waves = static_cast<double>((tiles * sp + slots - 1) / slots);
        const double t_cta = chunk * static_cast<double>(tile_flops_per_k) / sm_rate / clk + 2.0e-6;
        const double t_red = sp > 1 ? static_cast<double>(sp + 2) * M * N * 8.0 / 6.0e12 + 3.0e-6 : 0.0;
        const double t = waves * t_cta + t_red;
        if (t < best * 0.98) {  // more splits only for a clear win
            best = t;
            bsp = static_cast<int>(sp);
        }
    }
    return bsp;
}

// Tile + deterministic split-K plan.  128 x 64 tiles run two CTAs per SM
// (296 slots).  Enough tiles (>= 3 waves) or a short K (the rank-b updates):
// no split.  Otherwise (the K = s sketch / projection products, m or n = b)
// split K by the wave model above.
GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int64_t work_elems) {
    auto cap = [&](int64_t sp) {
        if (M * N > 0) sp = std::min<int64_t>(sp, work_elems / (M * N));
        return static_cast<int>(std::max<int64_t>(sp, 1));
    };
    const int64_t slots = 2 * kNumSMs;
    // Skinny products (one side <= 128, i.e. n x b with b <= 128): 64 x 64
    // tiles (measured 22 vs 18.8 TF/s for 128 x 64 at 4000 x 128 x 4000).
    if (gemm_plan_mode() == 1 || (std::min(M, N) <= 128 && K >= 512)) {
        const int64_t ts = ((M + 63) / 64) * ((N + 63) / 64);
        if (K < 512) return {false, 1};
        return {false, cap(choose_splits(M, N, K, ts, 64 * 64 * 2, slots, std::min<int64_t>(K / 128, 32)))};
    }
    const int64_t tb = ((M + 127) / 128) * ((N + 63) / 64);
    if (K < 1024 && tb < slots) return {false, 1};  // small late-step updates: more, smaller tiles
    if (K < 1024 || (tb >= 3 * slots && K < 4096)) return {true, 1};
    // long K: the wave model also fixes the quantisation of mid-size grids
    // (e.g. 940 tiles = 3.2 waves of 296 at config 4's sketch)
    return {true, cap(choose_splits(M, N, K, tb, 128 * 64 * 2, slots, std::min<int64_t>(K / 256, 32)))};
}

}  // namespace

int64_t gemm_work_elems(int64_t m, int64_t n, int64_t k) {
    const GemmPlan pl = plan_gemm(m, n, k, INT64_MAX / 4);
    return pl.splits > 1 ? pl.splits * m * n : 0;
}

void gemm(cudaStream_t stream, double alpha, Op ta, const DView& a, Op tb, const DView& b,
          double beta, const DView& c, double* work, int64_t work_elems) {
    const int64_t opa_r = ta == Op::N ? a.rows : a.cols, opa_c = ta == Op::N ? a.cols : a.rows;
    const int64_t opb_r = tb == Op::N ? b.rows : b.cols, opb_c = tb == Op::N ? b.cols : b.rows;
    if (opa_c != opb_r || c.rows != opa_r || c.cols != opb_c)
        throw Error(RUTV_ERR_SHAPE, "gemm shapes op(A)=" + std::to_string(opa_r) + "x" +
                                        std::to_string(opa_c) + " op(B)=" + std::to_string(opb_r) +
                                        "x" + std::to_string(opb_c) + " C=" +
                                        std::to_string(c.rows) + "x" + std::to_string(c.cols));
    const int64_t M = c.rows, N = c.cols, K = opa_c;
    if (M == 0 || N == 0) return;
    if (K == 0 || alpha == 0.0) {
        if (beta != 1.0) {
            scale_kernel<<<std::min<int64_t>((M * N + 255) / 256, 4 * kNumSMs), 256, 0, stream>>>(
                M, N, c.data, c.ld, beta);
            note_launch();
            RUTV_CHECK_LAUNCH();
        }
        return;
    }
    ProfScope prof(stream, 2.0 * static_cast<double>(M) * N * K);
    GemmParams p{M, N, K, a.data, a.ld, b.data, b.ld, c.data, c.ld, alpha, beta, work, K, 1,
                 aligned16(c.data, c.ld) ? 1 : 0};
    const bool vec = aligned16(a.data, a.ld) && aligned16(b.data, b.ld);
    const bool tA = ta == Op::T, tB = tb == Op::T;
    const GemmPlan pl = plan_gemm(M, N, K, work ? work_elems : 0);
    int splits = work ? pl.splits : 1;
    if (splits > 1) {
        int64_t kc = (K + splits - 1) / splits;
        kc = (kc + kBK - 1) / kBK * kBK;
        splits = static_cast<int>((K + kc - 1) / kc);
        p.kchunk = kc;
        p.splits = splits;
    }
    if (pl.large) {
        static int cfg = [] {
            const char* e = std::getenv("RUTV_GEMM_CFG");
            return e ? std::atoi(e) : 4;
        }();
        // cfg 4 (128 x 64, 4 warps of 64 x 32, BK = 16, 3 stages, 2 CTAs/SM,
        // C staged through shared memory) measured best on B200 for every step
        // shape (tools/gemm_bench.py: 32.5 TF/s at 8192^3, 21.7 at K = 128,
        // 30.5 at 20000^2 x 512) over cfg 2 (128 x 128, 16 warps) and cfg 3.
        if (cfg == 2)
            dispatch<128, 128, 32, 32, 32, 3>(stream, p, tA, tB, vec, splits);
        else if (cfg == 3)
            dispatch<64, 128, 16, 32, 64, 3>(stream, p, tA, tB, vec, splits);
        else
            dispatch<128, 64, 16, 64, 32, 3>(stream, p, tA, tB, vec, splits);
    } else {
        dispatch<64, 64, kBK, 32, 32, 3>(stream, p, tA, tB, vec, splits);
    }
    if (splits > 1) {
        const int64_t total = M * N;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs));
        splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(M, N, splits, work, c.data, c.ld, alpha,
                                                         beta);
        note_launch();
        RUTV_CHECK_LAUNCH();
    }
}

}  // namespace rutv
