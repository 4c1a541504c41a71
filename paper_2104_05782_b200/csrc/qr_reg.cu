// qr_reg.cu -- Householder panel QR on a thread-block cluster, micro-panels in
// registers (sm_100a DSMEM + DMMA).
//
// Same arithmetic contract as qr_cluster.cu: the reference's house() convention
// (proj/src/householder.cpp:20-34, beta >= 0, Parlett head, tau = 2 sign flip,
// tau = 0 skip) and hqr_inplace's left-to-right reflector order
// (householder.cpp:48-67); outputs are the packed R / unit-lower V and tau.
//
// Why a second kernel: the one-level kernel streams every trailing column of
// the panel through shared memory once per column (3 loads + 1 store per
// element per column), which makes a 128-column panel shared-memory-bandwidth
// and latency bound at 3.5-9 us per column.  Here the panel is processed in
// micro-panels of KB = 16 columns:
//
//   * the s x w panel is split by rows over CS CTAs (one cluster); each CTA
//     keeps its row chunk resident in shared memory (odd leading dimension);
//   * the current micro-panel lives in REGISTERS: thread t owns local rows
//     t, t + 512, ... and all 16 columns of them.  Per column j the thread
//     scales its reflector entry, applies the reflector to its 15 other
//     columns and accumulates its share of the next column's dot products --
//     no shared-memory traffic at all;
//   * the 16 partial dots (and the owner's head row) are reduced by a warp
//     butterfly, then across warps, then all-gathered over the cluster with
//     st.async remote stores completing on the receivers' mbarriers (one DSMEM
//     hop per column); every CTA sums the CS partials in rank order, so all
//     CTAs hold bit-identical house() scalars;
//   * after each micro-panel the trailing columns of the panel receive the
//     block reflector, Q' A_t = A_t - V T' (V' A_t): V'[V | A_t] is formed with
//     warp-level DMMA (mma.sync m16n8k4 f64), reduce-scattered and all-gathered
//     over the cluster (deterministic rank order), T comes from the Gram
//     matrix V'V and tau by the forward recurrence of form_wy_t
//     (householder.cpp:69-97), and the rank-16 update is again DMMA.
//
// Rows per thread MR = 1 or 2 (chunk rows R <= 1024); taller chunks use the
// one-level kernel.
//
// Micro-panel fast path ("CQ", default on; RUTV_QR_CQ=0 disables).  The column
// loop above costs one cluster-wide exchange per column (~2.5 K cycles each).
// A full 16-column micro-panel X (rows >= j0) with a well-conditioned Gram
// matrix is instead factored with TWO exchanges, by Cholesky-QR2 and
// Householder reconstruction (cholqr.cu's scheme at micro-panel granularity,
// entirely in shared memory / registers):
//   G = X'X (DMMA partials, all-gathered)        -> R1 = chol(G) in one warp
//   X1 = X R1^-1 (per-row forward substitution in registers)
//   E = X1'X1 - I (second exchange, with the 16 x 16 head block of X1)
//   R2 = I + U1, U1 = striu(E) + diag(E)/2 (|E| <= 1e-9: the series is exact
//   to 1e-18), Q = X1 (I - U1), R = R2 R1
//   I - Q(head) = L U (one warp)  ->  V = [L; -Q(below) U^-1], tau = diag(U)
// which are the reference's reflectors (beta >= 0 makes the thin QR unique) up
// to rounding.  Every CTA forms bit-identical G / E (fixed summation order), so
// the safety decisions are uniform across the cluster: Cholesky breakdown or
// min/max diag(R1) < 1e-3 -> the micro-panel takes the column loop with its
// registers untouched; |E| > 1e-9 or an LU pivot |tau_j| < 0.25 (a reflector
// near the identity, e.g. tau = 0) -> X is restored as X1 R1 and the column
// loop runs.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "cluster_msg.cuh"
#include "small_chains.cuh"
#include "rutv_common.cuh"

namespace cg = cooperative_groups;

namespace rutv {

namespace {

constexpr int kT = 512;       // threads per CTA
constexpr int kWarps = kT / 32;
constexpr int KB = 16;        // micro-panel width
constexpr int kMsg = 2 * KB;  // per-column message: 16 partial dots + 16 head-row entries
constexpr int kNG = KB * (KB + 1) / 2;  // packed upper triangle of a 16 x 16 Gram matrix
constexpr int kCqMat = KB * KB;         // one 16 x 16 matrix
constexpr int kCqDoubles = 5 * kCqMat + 2 * kNG + 2 * KB + 2;  // rmat, rfin, lumat, q1in, q1 staging, 2 Gram staging, rdinv, udinv, flags
constexpr unsigned kFull = 0xffffffffu;

struct RegSmem {
    double* chunk;  // w x LD, column-major
    double* msg;    // [2][CS][kMsg]
    double* rsb;    // [CS][KB][nsmax] reduce-scatter inbox; also the CQ hop-1 inbox [CS][kNG]
    double* gin2;   // [CS][kNG] CQ hop-2 inbox
    double* cq;     // CQ small matrices (kCqDoubles)
    double* zg;     // [KB][ncol] all-gathered V'[V | A_t], then -T'Z in place
    double* part;   // per-warp partials: column dots [kWarps][KB]; block [ksplit][KB][ncol]
    double* tmat;   // [KB][KB] T, row-major
    double* taus;   // [KB]
    double* hsend;  // [KB] head row of the next column (row owner only)
    uint64_t* bar;  // [6]: column parity 0/1, reduce-scatter, all-gather, CQ hop 1, CQ hop 2
};

__host__ __device__ inline int ns_max(int w, int cs) { return (KB + w + cs - 1) / cs; }
__host__ __device__ inline int part_elems(int w) { return KB * std::max(kWarps * 8, KB + w); }

// The hop-1 inbox of the CQ path shares the reduce-scatter inbox: a peer enters the block
// phase of micro-panel m only after every CTA's hop-2 message of m (sent after that CTA read
// its hop-1 inbox), and sends hop 1 of m + 1 only after the all-gather of block phase m, which
// every CTA feeds after consuming its reduce-scatter inbox.
__host__ __device__ inline int rs_elems(int w, int cs) { return std::max(cs * KB * ns_max(w, cs), cs * kNG); }
// even, so the buffers behind the chunk stay 16-byte aligned (16-byte remote stores)
__host__ __device__ inline size_t chunk_elems(int w, int LD) { return (static_cast<size_t>(w) * LD + 1) & ~static_cast<size_t>(1); }

__host__ __device__ inline size_t reg_smem_doubles(int w, int LD, int cs) {
    return static_cast<size_t>(chunk_elems(w, LD)) + 2 * cs * kMsg + static_cast<size_t>(rs_elems(w, cs)) + cs * kNG +
           kCqDoubles + static_cast<size_t>(KB) * (KB + w) + part_elems(w) + KB * KB + 2 * KB + 6;
}

__device__ __forceinline__ RegSmem carve(double* sm, int w, int LD, int CS) {
    RegSmem S;
    S.chunk = sm;
    S.msg = S.chunk + chunk_elems(w, LD);
    S.rsb = S.msg + 2 * CS * kMsg;
    S.gin2 = S.rsb + rs_elems(w, CS);
    S.cq = S.gin2 + CS * kNG;
    S.zg = S.cq + kCqDoubles;
    S.part = S.zg + static_cast<size_t>(KB) * (KB + w);
    S.tmat = S.part + part_elems(w);
    S.taus = S.tmat + KB * KB;
    S.hsend = S.taus + KB;
    S.bar = reinterpret_cast<uint64_t*>(S.hsend + KB);
    return S;
}

__device__ __forceinline__ void dmma(double* c, double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// Reflector entry V(li, c) of the micro-panel starting at global column j0:
// unit lower trapezoidal (1 on the diagonal, 0 above, 0 for c >= kb).
__device__ __forceinline__ double vent(uint32_t chunk_a, int LD, int li, int rc, int gi, int j0, int c, int kb) {
    if (li >= rc || c >= kb) return 0.0;
    const int j = j0 + c;
    if (gi > j) return lds_f64(chunk_a + 8u * static_cast<uint32_t>(j * LD + li));
    return gi == j ? 1.0 : 0.0;
}

// Debug ablation mask (RUTV_QR_ABLATE, timing experiments only -- results are
// wrong when set): 1 = skip block phases, 2 = trivial house(), 4 = skip the
// warp butterfly.
__device__ int g_qr_ablate = 0;

template <int MR>
__global__ void __launch_bounds__(kT, 1)
    hqr_reg_kernel(double* A, int64_t lda, int s, int w, int p, int R, int LD, double* tau, long long* trace,
                   int cq_mode) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = static_cast<int>(cluster.num_blocks());
    const int rank = static_cast<int>(cluster.block_rank());
    extern __shared__ __align__(16) double sm[];
    const RegSmem S = carve(sm, w, LD, CS);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int r_beg = rank * R;
    const int rc = max(0, min(s, r_beg + R) - r_beg);
    const int nwact = max(1, min(kWarps, (rc + 31) >> 5));  // warps owning rows (warp 0 always)

    // Every shared-memory region by its 32-bit shared-window address, derived from ONE opaque
    // register (sm_a) plus the carve offsets.  A generic pointer access -- or a rematerialised
    // smem_u32() -- costs an S2R SR_CgaCtaId + LEA in a cluster kernel, and this kernel's phases
    // are single-warp latency chains: ptxas put those reads INSIDE the one-warp Cholesky / LU loops
    // (5.2 K -> 7.8 K cycles per chain) until the addresses became opaque to it.
    uint32_t sm_a;
    asm volatile("mov.u32 %0, %1;" : "=r"(sm_a) : "r"(smem_u32(sm)));
    auto addr = [&](const void* q) {
        return sm_a + static_cast<uint32_t>(reinterpret_cast<const char*>(q) - reinterpret_cast<const char*>(sm));
    };
    const uint32_t msg_a = addr(S.msg);
    const uint32_t part_a = addr(S.part), hsend_a = addr(S.hsend), chunk_a = sm_a;
    const uint32_t bar0 = addr(S.bar);  // mbarrier b at bar0 + 8 b
    const uint32_t rsb_a = addr(S.rsb), gin2_a = addr(S.gin2), zg_a = addr(S.zg), tmat_a = addr(S.tmat);
    const uint32_t taus_a = addr(S.taus), cqb_a = addr(S.cq);

    for (int idx = tid; idx < w * rc; idx += kT) {
        const int c = idx / rc, i = idx - c * rc;
        S.chunk[static_cast<size_t>(c) * LD + i] = A[(r_beg + i) + static_cast<int64_t>(c) * lda];
    }
    // number of block phases: micro-panels with trailing columns beyond their register tile
    int nphase = 0;
    for (int j0 = 0; j0 < p; j0 += KB) nphase += (j0 + min(KB, w - j0) < w) ? 1 : 0;
    const uint32_t col_bytes = static_cast<uint32_t>(CS * kMsg * 8);
    auto rs_bytes = [&](int j0) {
        const int kt = min(KB, w - j0), ncol = KB + w - j0 - kt, ns = (ncol + CS - 1) / CS;
        const int mine = max(0, min(ncol, (rank + 1) * ns) - rank * ns);
        return static_cast<uint32_t>(CS * KB * mine * 8);
    };
    auto ag_bytes = [&](int j0) {
        const int kt = min(KB, w - j0);
        return static_cast<uint32_t>(KB * (KB + w - j0 - kt) * 8);
    };
    auto next_phase_j0 = [&](int j0) {  // first micro-panel after j0 with a block phase, or -1
        for (int jj = j0 + KB; jj < p; jj += KB)
            if (jj + min(KB, w - jj) < w) return jj;
        return -1;
    };
    // CQ exchanges: hop 1 = CS packed Gram partials; hop 2 = the same plus the 16 x 16 head block
    const uint32_t hop1_bytes = static_cast<uint32_t>(CS * kNG * 8);
    const uint32_t hop2_bytes = static_cast<uint32_t>((CS * kNG + kCqMat) * 8);
    if (tid == 0) {
        for (int b = 0; b < 6; ++b) mbar_init(&S.bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        // The column barriers 0/1 are armed per micro-panel (only the micro-panels that take
        // the column loop use them); the CQ barriers once here and again after every
        // completed wait.  A message may land before its barrier is armed: the phase only
        // completes with the arming thread's own arrival.
        if (cq_mode) {
            mbar_arm_a(bar0 + 8u * 4, hop1_bytes);
            mbar_arm_a(bar0 + 8u * 5, hop2_bytes);
        }
        const int f = (0 + min(KB, w) < w && p > 0) ? 0 : next_phase_j0(0);
        if (nphase > 0 && f >= 0) {
            mbar_arm_a(bar0 + 8u * 2, rs_bytes(f));
            mbar_arm_a(bar0 + 8u * 3, ag_bytes(f));
        }
    }
    cluster.sync();  // every CTA live, barriers initialised, before any remote traffic

    // Reduce the 16 per-thread partial dots over the row-owning warps and
    // all-gather them, with the head row of column jn, to every CTA's message
    // slot jn & 1.  Called by the nwact row-owning warps only (named barrier).
    const int ablate = g_qr_ablate;
    auto col_send = [&](double (&vals)[KB], int jn) {
        // butterfly reduce-scatter: after it lane l holds the sum of index l >> 1
#pragma unroll
        for (int lvl = 0; lvl < 4; ++lvl) {
            if (ablate & 4) break;
            const int o = 16 >> lvl, n = (KB / 2) >> lvl;
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < n; ++i) {
                const double send = up ? vals[i] : vals[i + n];
                const double keep = up ? vals[i + n] : vals[i];
                vals[i] = keep + __shfl_xor_sync(kFull, send, o);
            }
        }
        const double v = vals[0] + __shfl_xor_sync(kFull, vals[0], 1);
        if ((lane & 1) == 0) sts_f64(part_a + 8u * static_cast<uint32_t>(warp * KB + (lane >> 1)), v);
        asm volatile("bar.sync 1, %0;" ::"r"(nwact * 32) : "memory");
        if (trace && tid == 0 && rank == 0 && jn < 64) trace[jn * 8 + 4] = clock64();
        // every row-owning warp forms the (identical) message and sends it to
        // its share of the destinations: warp w -> ranks w, w + nwact, ...
        if (warp < CS) {
            double val = 0.0;
            if (lane < KB) {
                for (int ww = 0; ww < nwact; ++ww) val += lds_f64(part_a + 8u * static_cast<uint32_t>(ww * KB + lane));
            } else if (jn >= r_beg && jn < r_beg + rc) {
                val = lds_f64(hsend_a + 8u * static_cast<uint32_t>(lane - KB));
            }
            const int par = jn & 1;
            const uint32_t off = msg_a + static_cast<uint32_t>(((par * CS + rank) * kMsg + lane) * 8);
            for (int dst = warp; dst < CS; dst += nwact)
                st_async_f64(mapa_u32(off, dst), val, mapa_u32(bar0 + 8 * par, dst));
            if (trace && tid == 0 && rank == 0 && jn < 64) trace[jn * 8 + 5] = clock64();
        }
    };

    double x[MR][KB];
    int phase = 0;
    // parities of the completed phases: bit 0 / 1 column barriers 0 / 1, bit 2 / 3 CQ hops 1 / 2
    unsigned phbits = 0;
    // CQ small matrices (16 x 16, row-major) by 32-bit shared addresses off one base
    constexpr uint32_t kRmat = 0;                     // R1(k, j) at [16 k + j]
    constexpr uint32_t kRfin = 8u * kCqMat;           // final R = (I + U1) R1
    constexpr uint32_t kLumat = 16u * kCqMat;         // I - Q(head), then its packed LU
    constexpr uint32_t kQ1in = 24u * kCqMat;          // head block of X1 (hop 2)
    constexpr uint32_t kQ1st = 32u * kCqMat;          // staging of my head rows of X1
    constexpr uint32_t kStg = 40u * kCqMat;           // staging of my packed Gram partial, hop 1 / hop 2
    constexpr uint32_t kRdinv = kStg + 16u * kNG;     // 1 / R1(k, k)
    constexpr uint32_t kUdinv = kRdinv + 8u * KB;     // 1 / U(k, k)
    constexpr uint32_t kFlag = kUdinv + 8u * KB;      // int [0] pass 1, [1] LU
    auto lds_i32 = [](uint32_t a) {
        int v;
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
        return v;
    };
    auto sts_i32 = [](uint32_t a, int v) { asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); };
    // this thread's packed Gram entry (i <= k), tid < kNG: pe = 16 i + k
    int pe = 0;
    if (tid < kNG) {
        int k = 0;
        while ((k + 1) * (k + 2) / 2 <= tid) ++k;
        pe = (tid - k * (k + 1) / 2) * KB + k;
    }
    auto packed_index = [&](int& pi, int& pk) {
        pi = pe >> 4;
        pk = pe & 15;
    };
    // Packed Gram partial of chunk columns [j0, j0 + 16) over the local rows [lo, rc), summed
    // over the warps in a fixed order and sent to every CTA's inbox (slot = my rank).
    auto gram_send = [&](int j0, int lo, double* inbox, int barid) {
        const int nk4 = (rc - lo + 3) >> 2;
        const int k0 = (warp * nk4) / kWarps, k1 = ((warp + 1) * nk4) / kWarps;
        double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};  // G(:, 0:8), G(:, 8:16)
        const uint32_t p0 = chunk_a + 8u * static_cast<uint32_t>((j0 + g) * LD + lo + t4);
        const uint32_t p1 = p0 + 8u * static_cast<uint32_t>(8 * LD);
        for (int k4 = k0; k4 < k1; ++k4) {
            const bool ok = lo + 4 * k4 + t4 < rc;  // a row past rc reads valid shared memory, selected away
            const uint32_t o = 32u * static_cast<uint32_t>(k4);
            const double r0 = lds_f64(p0 + o), r1 = lds_f64(p1 + o);
            const double v0 = ok ? r0 : 0.0, v1 = ok ? r1 : 0.0;  // X(row, g), X(row, g + 8)
            dmma(c0, v0, v1, v0);
            dmma(c1, v0, v1, v1);
        }
        const bool gt = trace && tid == 0 && rank == 0 && (j0 >> 4) < 8 && barid == 4;
        if (gt) trace[72 * 8 + (j0 >> 4) * 16 + 12] = clock64();
        // 16 warp partials in 8 slots: warps 0-7 store, warps 8-15 add
        const uint32_t slot = part_a + 8u * static_cast<uint32_t>((warp & 7) * kCqMat);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            if ((warp >> 3) == half) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int idx = (g + (r >= 2 ? 8 : 0)) * KB + 2 * t4 + (r & 1);
                    const uint32_t sa = slot + 8u * static_cast<uint32_t>(idx);
                    if (half == 0) {
                        sts_f64(sa, c0[r]);
                        sts_f64(sa + 64u, c1[r]);
                    } else {
                        sts_f64(sa, lds_f64(sa) + c0[r]);
                        sts_f64(sa + 64u, lds_f64(sa + 64u) + c1[r]);
                    }
                }
            }
            __syncthreads();
        }
        const uint32_t stg = cqb_a + kStg + (barid == 5 ? 8u * kNG : 0u);
        if (gt) trace[72 * 8 + (j0 >> 4) * 16 + 13] = clock64();
        if (tid < kNG) {
            double v = 0.0;
#pragma unroll
            for (int ws = 0; ws < 8; ++ws) v += lds_f64(part_a + 8u * static_cast<uint32_t>(ws * kCqMat + pe));
            sts_f64(stg + 8u * tid, v);
        }
        if (gt) trace[72 * 8 + (j0 >> 4) * 16 + 14] = clock64();
        __syncthreads();
        if (gt) trace[72 * 8 + (j0 >> 4) * 16 + 15] = clock64();
        // 68 pairs x CS destinations spread over all threads (16-byte remote stores: the CTA's
        // remote-store rate bounds this exchange; a bulk DSMEM copy per destination was
        // measured slower -- ~1.2 K cycles to issue behind a proxy fence)
        const uint32_t inbox_a = addr(inbox) + 8u * static_cast<uint32_t>(rank * kNG);
        for (int idx = tid; idx < (kNG / 2) * CS; idx += kT) {
            const int dst = idx / (kNG / 2), pr = idx - dst * (kNG / 2);
            double a, b;
            lds_v2f64(stg + 16u * pr, a, b);
            st_async_v2f64(mapa_u32(inbox_a + 16u * pr, dst), a, b, mapa_u32(bar0 + 8 * barid, dst));
        }
    };
    for (int j0 = 0; j0 < p; j0 += KB) {
        const int kb = min(KB, p - j0), kt = min(KB, w - j0);
        // ---- load the micro-panel tile into registers.  The tile is a window
        // that shifts left by one column per step: x[m][k] is always column
        // j + k of the current step j, so the step body is the same code for
        // every column (a runtime loop; a fully unrolled 16-column body
        // overflows the instruction cache).
#pragma unroll
        for (int m = 0; m < MR; ++m) {
            const int li = tid + kT * m;
#pragma unroll
            for (int k = 0; k < KB; ++k)
                x[m][k] = (li < rc && k < kt) ? lds_f64(chunk_a + 8u * static_cast<uint32_t>((j0 + k) * LD + li)) : 0.0;
        }
        // ---- CQ fast path for a full micro-panel (see the header); hh = the column loop runs
        bool hh = true;
        if (cq_mode && kb == KB && kt == KB && s - j0 >= 2 * KB) {
            const int lo = min(rc, max(0, j0 - r_beg));  // local rows with gi >= j0
            const uint32_t cq_a = cqb_a, scr_a = part_a;
            int lane_o;  // likewise the lane index (S2R SR_TID.X in the loops otherwise)
            asm volatile("mov.s32 %0, %1;" : "=r"(lane_o) : "r"(lane));
            int pe_i = 0, pe_k = 0;
            if (tid < kNG) packed_index(pe_i, pe_k);
            const bool force1 = cq_mode == 3 && ((j0 >> 4) & 1), force2 = cq_mode == 2 && ((j0 >> 4) & 1);
            const bool cqt = trace && tid == 0 && rank == 0 && (j0 >> 4) < 8;
#define CQT(k) \
    if (cqt) trace[72 * 8 + (j0 >> 4) * 16 + (k)] = clock64()
            CQT(0);
            // -- pass 1: G = X'X, R1 = chol(G)
            gram_send(j0, lo, S.rsb, 4);
            CQT(1);
            mbar_wait_a(bar0 + 8u * 4, (phbits >> 2) & 1u);
            phbits ^= 4u;
            CQT(2);
            if (tid == 0) mbar_arm_a(bar0 + 8u * 4, hop1_bytes);
            if (tid < kNG) {
                double v = 0.0;
                for (int src = 0; src < CS; ++src) v += lds_f64(rsb_a + 8u * static_cast<uint32_t>(src * kNG + tid));
                sts_f64(tmat_a + 8u * static_cast<uint32_t>(pe_i * KB + pe_k), v);
                sts_f64(tmat_a + 8u * static_cast<uint32_t>(pe_k * KB + pe_i), v);
            }
            __syncthreads();
            CQT(3);
            if (warp == 0) {
                const int kk = lane & (KB - 1);
                double v[KB];
#pragma unroll
                for (int i = 0; i < KB; ++i) v[i] = lds_f64(tmat_a + 8u * static_cast<uint32_t>(i * KB + kk));
                double mn, mx;
                const bool brk = warp_chol16(v, cq_a + kRmat, cq_a + kRdinv, scr_a, mn, mx, lane_o);
                if (lane == 0) sts_i32(cq_a + kFlag, (brk || !(mn > 1e-3 * mx) || force1) ? 1 : 0);
            }
            __syncthreads();
            CQT(4);
            if (lds_i32(cq_a + kFlag) == 0) {
                // -- X1 = X R1^-1 by rows (registers), mirrored into the chunk for the second Gram
#pragma unroll
                for (int m = 0; m < MR; ++m) {
                    const int li = tid + kT * m;
                    if (li >= lo && li < rc) {
#pragma unroll
                        for (int k = 0; k < KB; ++k) {
                            const double yk = x[m][k] * lds_f64(cq_a + kRdinv + 8u * k);
                            x[m][k] = yk;
#pragma unroll
                            for (int j = k + 1; j < KB; ++j)
                                x[m][j] = __fma_rn(-yk, lds_f64(cq_a + kRmat + 8u * (k * KB + j)), x[m][j]);
                        }
                        const int hr = r_beg + li - j0;  // head-block row, if < 16
#pragma unroll
                        for (int k = 0; k < KB; ++k) {
                            sts_f64(chunk_a + 8u * static_cast<uint32_t>((j0 + k) * LD + li), x[m][k]);
                            if (hr < KB) sts_f64(cq_a + kQ1st + 8u * (hr * KB + k), x[m][k]);
                        }
                    }
                }
                __syncthreads();
                CQT(5);
                // -- pass 2: E = X1'X1 - I, with the head block of X1 from its owner(s)
                gram_send(j0, lo, S.gin2, 5);
                {  // my head rows [h0, h1) of X1 to every CTA
                    const int h0 = max(0, r_beg - j0), h1 = min(KB, r_beg + rc - j0);
                    const int npr = max(0, h1 - h0) * (KB / 2);
                    for (int idx = tid; idx < npr * CS; idx += kT) {
                        const int dst = idx / npr, pr = h0 * (KB / 2) + idx - dst * npr;
                        double a, b;
                        lds_v2f64(cq_a + kQ1st + 16u * pr, a, b);
                        st_async_v2f64(mapa_u32(cq_a + kQ1in + 16u * pr, dst), a, b, mapa_u32(bar0 + 8 * 5, dst));
                    }
                }
                CQT(6);
                mbar_wait_a(bar0 + 8u * 5, (phbits >> 3) & 1u);
                CQT(7);
                phbits ^= 8u;
                if (tid == 0) mbar_arm_a(bar0 + 8u * 5, hop2_bytes);
                bool bad = false;
                if (tid < kNG) {
                    double v = 0.0;
                    for (int src = 0; src < CS; ++src) v += lds_f64(gin2_a + 8u * static_cast<uint32_t>(src * kNG + tid));
                    const double e = v - (pe_i == pe_k ? 1.0 : 0.0);
                    sts_f64(tmat_a + 8u * static_cast<uint32_t>(pe_i * KB + pe_k), e);
                    sts_f64(tmat_a + 8u * static_cast<uint32_t>(pe_k * KB + pe_i), e);
                    bad = !(fabs(e) <= 1e-9);
                }
                bool redo = __syncthreads_or(bad || force2) != 0;
                CQT(8);
                if (!redo) {
                    // -- Q(head) = X1(head) (I - U1), B = I - Q(head); R = (I + U1) R1
                    if (tid < kCqMat) {
                        const int r = tid >> 4, k = tid & 15;
                        double acc = lds_f64(cq_a + kQ1in + 8u * (r * KB + k)) * (1.0 - 0.5 * lds_f64(tmat_a + 8u * (k * KB + k)));
                        for (int i = 0; i < k; ++i)
                            acc = __fma_rn(-lds_f64(cq_a + kQ1in + 8u * (r * KB + i)), lds_f64(tmat_a + 8u * (i * KB + k)), acc);
                        sts_f64(cq_a + kLumat + 8u * (r * KB + k), (r == k ? 1.0 : 0.0) - acc);
                    } else {
                        const int i = (tid - kCqMat) >> 4, k = tid & 15;
                        double acc = 0.0;
                        if (i <= k) {
                            acc = lds_f64(cq_a + kRmat + 8u * (i * KB + k)) * (1.0 + 0.5 * lds_f64(tmat_a + 8u * (i * KB + i)));
                            for (int m2 = i + 1; m2 <= k; ++m2)
                                acc = __fma_rn(lds_f64(tmat_a + 8u * (i * KB + m2)), lds_f64(cq_a + kRmat + 8u * (m2 * KB + k)), acc);
                        }
                        sts_f64(cq_a + kRfin + 8u * (i * KB + k), acc);
                    }
                    __syncthreads();
                    CQT(9);
                    if (warp == 0) {
                        const int kk = lane & (KB - 1);
                        double v[KB];
#pragma unroll
                        for (int i = 0; i < KB; ++i) v[i] = lds_f64(cq_a + kLumat + 8u * (i * KB + kk));
                        __syncwarp();
                        // tau = diag(U) lands in S.taus (the block phase's T recurrence reads it)
                        const bool brk = warp_lu16(v, cq_a + kLumat, cq_a + kUdinv, taus_a, scr_a, lane_o);
                        const bool any = __any_sync(kFull, brk);
                        if (lane == 0) sts_i32(cq_a + kFlag + 4u, any ? 1 : 0);
                    }
                    __syncthreads();
                    CQT(10);
                    redo = lds_i32(cq_a + kFlag + 4u) != 0;
                }
                if (!redo) {
                    if (rank == 0 && tid < KB) tau[j0 + tid] = lds_f64(taus_a + 8u * tid);
                    // T of the block reflector from the reconstruction itself: U = T V1' with V1 = L,
                    // so row i of T solves t_i L' = u_i (one warp, beside the row finalisation);
                    // the block phase then needs neither V'V nor the form_wy_t recurrence.
                    if (warp == kWarps - 1 && lane < KB) {
                        double trow[KB];
#pragma unroll
                        for (int k = 0; k < KB; ++k) {
                            double acc = k >= lane ? lds_f64(cq_a + kLumat + 8u * (lane * KB + k)) : 0.0;
#pragma unroll
                            for (int m2 = 0; m2 < k; ++m2)
                                acc = __fma_rn(-trow[m2], lds_f64(cq_a + kLumat + 8u * (k * KB + m2)), acc);
                            trow[k] = acc;
                        }
#pragma unroll
                        for (int k = 0; k < KB; ++k) sts_f64(cq_a + kQ1in + 8u * (lane * KB + k), trow[k]);
                    }
                    // -- V = [L; -Q(below) U^-1], R into the head rows; retire the micro-panel
#pragma unroll
                    for (int m = 0; m < MR; ++m) {
                        const int li = tid + kT * m;
                        if (li >= lo && li < rc) {
                            const int hr = r_beg + li - j0;
                            if (hr >= KB) {
                                // y = x (I - U1), descending so x(i < k) is still X1
#pragma unroll
                                for (int k = KB - 1; k >= 0; --k) {
                                    double acc = x[m][k] * (1.0 - 0.5 * lds_f64(tmat_a + 8u * (k * KB + k)));
#pragma unroll
                                    for (int i = 0; i < k; ++i)
                                        acc = __fma_rn(-x[m][i], lds_f64(tmat_a + 8u * (i * KB + k)), acc);
                                    x[m][k] = acc;
                                }
                                // z U = -y
#pragma unroll
                                for (int k = 0; k < KB; ++k) {
                                    const double zk = -x[m][k] * lds_f64(cq_a + kUdinv + 8u * k);
                                    x[m][k] = zk;
#pragma unroll
                                    for (int j = k + 1; j < KB; ++j)
                                        x[m][j] = __fma_rn(zk, lds_f64(cq_a + kLumat + 8u * (k * KB + j)), x[m][j]);
                                }
                            } else {
#pragma unroll
                                for (int k = 0; k < KB; ++k)
                                    x[m][k] = lds_f64(cq_a + (k >= hr ? kRfin : kLumat) + 8u * (hr * KB + k));
                            }
#pragma unroll
                            for (int k = 0; k < KB; ++k)
                                sts_f64(chunk_a + 8u * static_cast<uint32_t>((j0 + k) * LD + li), x[m][k]);
                        }
                    }
                    hh = false;
                    CQT(11);
                } else {
                    // -- unsafe after pass 1: X = X1 R1 (descending, in place), then the column loop
#pragma unroll
                    for (int m = 0; m < MR; ++m) {
                        const int li = tid + kT * m;
                        if (li >= lo && li < rc) {
#pragma unroll
                            for (int j = KB - 1; j >= 0; --j) {
                                double acc = 0.0;
#pragma unroll
                                for (int k = 0; k <= j; ++k)
                                    acc = __fma_rn(x[m][k], lds_f64(cq_a + kRmat + 8u * (k * KB + j)), acc);
                                x[m][j] = acc;
                            }
                        }
                    }
                }
            }
        }
        // ---- column steps, row-owning warps only (no CTA-wide barrier).
        // Every such warp waits for the column's message itself, sums the CS
        // partials in rank order and evaluates house() redundantly (identical
        // in every warp of the cluster), lane k forming w_k.
        if (hh && warp < nwact) {
            if (tid == 0) {
                mbar_arm_a(bar0 + 8u * 0, col_bytes);
                if (kb > 1) mbar_arm_a(bar0 + 8u * 1, col_bytes);
            }
            {  // partials of column j0: x_j0' x_{j0+k} over rows > j0, head row j0
                double vals[KB];
#pragma unroll
                for (int k = 0; k < KB; ++k) vals[k] = 0.0;
#pragma unroll
                for (int m = 0; m < MR; ++m) {
                    const int li = tid + kT * m, gi = r_beg + li;
                    if (li < rc && gi > j0) {
#pragma unroll
                        for (int k = 0; k < KB; ++k) vals[k] += x[m][0] * x[m][k];
                    } else if (li < rc && gi == j0) {
#pragma unroll
                        for (int k = 0; k < KB; ++k) sts_f64(hsend_a + 8u * k, x[m][k]);
                    }
                }
                col_send(vals, j0);
            }
#pragma unroll 1
            for (int c = 0; c < kb; ++c) {
                const int j = j0 + c, par = j & 1;
                const bool tr = trace && tid == 0 && rank == 0 && j < 64;
                if (tr) trace[j * 8 + 0] = clock64();
                mbar_wait_a(bar0 + 8u * par, ((phbits >> par) + static_cast<unsigned>(c >> 1)) & 1u);
                if (tr) trace[j * 8 + 1] = clock64();
                double tsum;
                {
                    const uint32_t mp = msg_a + 8u * static_cast<uint32_t>(par * CS * kMsg + lane);
                    double t0 = 0.0, t1 = 0.0;
                    int r = 0;
                    for (; r + 1 < CS; r += 2) {
                        t0 += lds_f64(mp + 8u * static_cast<uint32_t>(r * kMsg));
                        t1 += lds_f64(mp + 8u * static_cast<uint32_t>((r + 1) * kMsg));
                    }
                    if (r < CS) t0 += lds_f64(mp + 8u * static_cast<uint32_t>(r * kMsg));
                    tsum = t0 + t1;
                }
                // house() (householder.cpp:20-34); 1/head and 1/beta by reciprocals
                const double sigma = __shfl_sync(kFull, tsum, 0);
                const double alpha = __shfl_sync(kFull, tsum, KB);
                const double hk = __shfl_sync(kFull, tsum, (lane + KB) & 31);  // lane k < 16: a(j, j+k)
                double beta, tj, rh = 1.0;
                bool scale = false;
                if (ablate & 2) {
                    beta = alpha;
                    tj = 1.0;
                    scale = true;
                } else if (sigma == 0.0) {
                    if (alpha >= 0.0) {
                        beta = alpha;
                        tj = 0.0;
                    } else {
                        beta = -alpha;
                        tj = 2.0;
                    }
                } else {
                    const double rsig = __drcp_rn(sigma);
                    beta = sqrt(alpha * alpha + sigma);
                    const double ab = alpha + beta;
                    const double rbeta = __drcp_rn(beta);
                    double head;
                    if (alpha >= 0.0) {
                        head = -sigma * __drcp_rn(ab);
                        rh = -ab * rsig;
                    } else {
                        head = alpha - beta;
                        rh = __drcp_rn(head);
                    }
                    tj = -head * rbeta;
                    scale = true;
                }
                // lane k: w_k = tau (a(j,k) + sum_{i>j} v_i a(i,k)) = tau (h_k + d_k / head)
                const double wkl = tj * (hk + (scale ? tsum * rh : tsum));
                if (tr) trace[j * 8 + 2] = clock64();
                // per-row multiplier of w_k: v_i below row j, 1 on row j, 0 above.
                // Branch-free: padded window columns are zero and get w_k = 0, so
                // every column of the window is updated unconditionally.
                double mult[MR], dm[MR];
#pragma unroll
                for (int m = 0; m < MR; ++m) {
                    const int li = tid + kT * m, gi = r_beg + li;
                    const bool below = li < rc && gi > j, diag = li < rc && gi == j;
                    const double v = scale ? x[m][0] * rh : x[m][0];
                    mult[m] = below ? v : (diag ? 1.0 : 0.0);
                    x[m][0] = below ? v : (diag ? beta : x[m][0]);
                }
                // apply the reflector to the window (householder.cpp:58-66) and
                // accumulate the next column's partials x_{j+1}' a_k over rows > j+1
                const bool nxt = c + 1 < kb;
                const int jn = j + 1;
#pragma unroll
                for (int k = 1; k < KB; ++k) {
                    const double wk = __shfl_sync(kFull, wkl, k);
#pragma unroll
                    for (int m = 0; m < MR; ++m) x[m][k] -= wk * mult[m];
                }
#pragma unroll
                for (int m = 0; m < MR; ++m) {
                    const int li = tid + kT * m, gi = r_beg + li;
                    dm[m] = (li < rc && gi > jn) ? x[m][1] : 0.0;
                }
                double vals[KB];
#pragma unroll
                for (int k = 0; k + 1 < KB; ++k) {
                    vals[k] = 0.0;
#pragma unroll
                    for (int m = 0; m < MR; ++m) vals[k] += dm[m] * x[m][k + 1];
                }
                vals[KB - 1] = 0.0;
                // retire column j to the chunk and shift the window
#pragma unroll
                for (int m = 0; m < MR; ++m) {
                    const int li = tid + kT * m;
                    if (li < rc) sts_f64(chunk_a + 8u * static_cast<uint32_t>(j * LD + li), x[m][0]);
#pragma unroll
                    for (int k = 0; k + 1 < KB; ++k) x[m][k] = x[m][k + 1];
                    x[m][KB - 1] = 0.0;
                }
                if (tid == 0) {  // off the critical chain: re-arm slot par, record tau
                    if (c + 2 < kb) mbar_arm_a(bar0 + 8u * par, col_bytes);
                    if (rank == 0) tau[j] = tj;
                    sts_f64(taus_a + 8u * static_cast<uint32_t>(c), tj);
                }
                if (tr) trace[j * 8 + 3] = clock64();
                if (nxt) {
#pragma unroll
                    for (int m = 0; m < MR; ++m) {
                        const int li = tid + kT * m, gi = r_beg + li;
                        if (li < rc && gi == jn) {
#pragma unroll
                            for (int k = 0; k < KB; ++k) sts_f64(hsend_a + 8u * k, x[m][k]);
                        }
                    }
                    col_send(vals, jn);
                }
            }
        }
        if (hh) phbits ^= static_cast<unsigned>(((kb + 1) >> 1) & 1) | (static_cast<unsigned>((kb >> 1) & 1) << 1);
        // ---- tile columns beyond the factorised ones (wide panels, p < w)
#pragma unroll
        for (int m = 0; m < MR; ++m) {
            const int li = tid + kT * m;
            if (hh && li < rc) {
#pragma unroll
                for (int k = 0; k < KB; ++k)
                    if (k < kt - kb) sts_f64(chunk_a + 8u * static_cast<uint32_t>((j0 + kb + k) * LD + li), x[m][k]);
            }
        }
        __syncthreads();
        if (j0 + kt >= w || (ablate & 1)) continue;

        const int tph = phase;
        const bool have_t = !hh;  // the micro-panel took the CQ path: T sits in the CQ scratch
        if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 0] = clock64();
        // ---- block phase: A_t <- A_t - V T' (V' A_t), A_t = columns [j0 + kt, w)
        const int nrest = w - j0 - kt, ncol = KB + nrest;
        const int lo = min(rc, max(0, j0 - r_beg));  // local rows with gi >= j0
        const int nk4 = (rc - lo + 3) >> 2;
        {
            // P = V'[V | A_t] over my rows: M = 16 (c), N = ncol (tiles of 8), K = rows; after a CQ
            // micro-panel T is already known (have_t): the two tiles of V'V are skipped
            const int tl0 = have_t ? 2 : 0, nt = ((ncol + 7) >> 3) - tl0;
            const int ksplit = max(1, kWarps / (nt + tl0));  // [ksplit][16][ncol] fits `part` (part_elems)
            for (int u = warp; u < nt * ksplit; u += kWarps) {
                const int tile = tl0 + u % nt, ks = u / nt;
                const int kb0 = (ks * nk4) / ksplit, kb1 = ((ks + 1) * nk4) / ksplit;
                const int q = tile * 8 + g;  // my B column
                double acc[4] = {0.0, 0.0, 0.0, 0.0}, acc2[4] = {0.0, 0.0, 0.0, 0.0};
                auto slow = [&](int k4) {  // rows in the unit-triangle zone or past rc
                    const int li = lo + 4 * k4 + t4, gi = r_beg + li;
                    const double a0 = vent(chunk_a, LD, li, rc, gi, j0, g, kb);
                    const double a1 = vent(chunk_a, LD, li, rc, gi, j0, g + 8, kb);
                    double b;
                    if (q < KB) b = vent(chunk_a, LD, li, rc, gi, j0, q, kb);
                    else if (q < ncol && li < rc) b = lds_f64(chunk_a + 8u * static_cast<uint32_t>((j0 + kt + q - KB) * LD + li));
                    else b = 0.0;
                    dmma(acc, a0, a1, b);
                };
                // k4 < kspec: rows gi < j0 + KB (unit triangle); k4 >= kfull: rows past rc.
                // In between V is the stored column and every row exists: plain
                // loads, two independent DMMA chains.
                const int kspec = min(kb1, max(kb0, (j0 + KB - r_beg - lo + 3) >> 2));
                const int kfull = max(kspec, min(kb1, (rc - lo) >> 2));
                const bool za0 = g >= kb, za1 = g + 8 >= kb, zb = q >= ncol || (q < KB && q >= kb);
                // masked operands read a valid clamped column (column j0) and are zeroed by select
                const uint32_t cbase = chunk_a + 8u * static_cast<uint32_t>(lo + t4);
                const uint32_t pa0 = cbase + 8u * static_cast<uint32_t>((za0 ? j0 : j0 + g) * LD);
                const uint32_t pa1 = cbase + 8u * static_cast<uint32_t>((za1 ? j0 : j0 + g + 8) * LD);
                const uint32_t pb =
                    cbase + 8u * static_cast<uint32_t>((zb ? j0 : (q < KB ? j0 + q : j0 + kt + q - KB)) * LD);
                int k4 = kb0;
                for (; k4 < kspec; ++k4) slow(k4);
                for (; k4 + 1 < kfull; k4 += 2) {
                    const uint32_t o = 32u * static_cast<uint32_t>(k4);
                    const double a0r = lds_f64(pa0 + o), a1r = lds_f64(pa1 + o), br = lds_f64(pb + o);
                    const double c0r = lds_f64(pa0 + o + 32), c1r = lds_f64(pa1 + o + 32), dr = lds_f64(pb + o + 32);
                    dmma(acc, za0 ? 0.0 : a0r, za1 ? 0.0 : a1r, zb ? 0.0 : br);
                    dmma(acc2, za0 ? 0.0 : c0r, za1 ? 0.0 : c1r, zb ? 0.0 : dr);
                }
                for (; k4 < kb1; ++k4) slow(k4);
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[r] += acc2[r];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int row = g + (r >= 2 ? 8 : 0), col = tile * 8 + 2 * t4 + (r & 1);
                    if (col < ncol) sts_f64(part_a + 8u * static_cast<uint32_t>((ks * KB + row) * ncol + col), acc[r]);
                }
            }
            __syncthreads();
    if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 1] = clock64();
            // reduce over the K splits (fixed order) and scatter column slices to their owners
            const int ns = (ncol + CS - 1) / CS;
            for (int e = tid; e < KB * ncol; e += kT) {
                const int row = e / ncol, col = e - row * ncol;
                double v = 0.0;
                if (col >= 8 * tl0)
                    for (int ks = 0; ks < ksplit; ++ks) v += lds_f64(part_a + 8u * static_cast<uint32_t>((ks * KB + row) * ncol + col));
                const int o = col / ns;
                const uint32_t off =
                    rsb_a + 8u * static_cast<uint32_t>((rank * KB + row) * ns + (col - o * ns));
                st_async_f64(mapa_u32(off, o), v, mapa_u32(bar0 + 16, o));
            }
            // owner: sum the CS partial slices in rank order and broadcast
            mbar_wait_a(bar0 + 8u * 2, static_cast<uint32_t>(phase & 1));
    if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 2] = clock64();
            const int nxt = next_phase_j0(j0);
            if (tid == 0 && nxt >= 0) mbar_arm_a(bar0 + 8u * 2, rs_bytes(nxt));
            const int mine = max(0, min(ncol, (rank + 1) * ns) - rank * ns);
            for (int e = tid; e < KB * mine; e += kT) {
                const int row = e / mine, qq = e - row * mine;
                double v = 0.0;
                for (int src = 0; src < CS; ++src) v += lds_f64(rsb_a + 8u * static_cast<uint32_t>((src * KB + row) * ns + qq));
                const uint32_t off = zg_a + 8u * static_cast<uint32_t>(row * ncol + rank * ns + qq);
                for (int dst = 0; dst < CS; ++dst) st_async_f64(mapa_u32(off, dst), v, mapa_u32(bar0 + 24, dst));
            }
            mbar_wait_a(bar0 + 8u * 3, static_cast<uint32_t>(phase & 1));
    if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 3] = clock64();
            if (tid == 0 && nxt >= 0) mbar_arm_a(bar0 + 8u * 3, ag_bytes(nxt));
            ++phase;
        }
        // T (form_wy_t recurrence, householder.cpp:69-97): T(c,c) = tau_c,
        // T(0:c, c) = -tau_c T(0:c, 0:c) G(0:c, c), G = V'V = zg[:, 0:16]
        if (warp == 0 && !have_t) {
            double trow[KB];
#pragma unroll
            for (int c = 0; c < KB; ++c) {
                const double tc = lds_f64(taus_a + 8u * static_cast<uint32_t>(c < kb ? c : 0));
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < c; ++q) acc += trow[q] * lds_f64(zg_a + 8u * static_cast<uint32_t>(q * ncol + c));
                trow[c] = c >= kb ? 0.0 : (lane < c ? -tc * acc : (lane == c ? tc : 0.0));
            }
            if (lane < KB)
#pragma unroll
                for (int c = 0; c < KB; ++c) sts_f64(tmat_a + 8u * static_cast<uint32_t>(lane * KB + c), trow[c]);
        }
        __syncthreads();
        if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 4] = clock64();
        // Y = -T' Z (Z = zg[:, 16:]) into part[16][nrest], one entry per thread and pass
        {
            const uint32_t tsrc = have_t ? cqb_a + kQ1in : tmat_a;
            const uint32_t zsrc = zg_a;
            for (int e = tid; e < KB * nrest; e += kT) {
                const int c = e / nrest, k = e - c * nrest;
                double acc = 0.0;
                for (int q = 0; q <= c; ++q)
                    acc = __fma_rn(lds_f64(tsrc + 8u * static_cast<uint32_t>(q * KB + c)),
                                   lds_f64(zsrc + 8u * static_cast<uint32_t>(q * ncol + KB + k)), acc);
                sts_f64(part_a + 8u * static_cast<uint32_t>(e), -acc);
            }
        }
        __syncthreads();
        if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 5] = clock64();
        // A_t += V Y over my rows >= j0: M = rows (tiles of 16), N = nrest (tiles of 8), K = 16
        {
            const int mt = (rc - lo + 15) >> 4, ntl = (nrest + 7) >> 3;
            const int ngr = max(1, min(ntl, kWarps / max(1, mt)));
            const int nk = (kb + 3) >> 2;
            for (int u = warp; u < mt * ngr; u += kWarps) {
                const int mi = u % mt, ng = u / mt;
                const int r0 = lo + 16 * mi;
                double av[4][2];
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int li = r0 + g + 8 * h;
                        av[ks][h] = ks < nk ? vent(chunk_a, LD, li, rc, r_beg + li, j0, 4 * ks + t4, kb) : 0.0;
                    }
                // two column tiles per iteration: both loaded before either is
                // stored (a load after a store to the chunk cannot be hoisted),
                // two independent DMMA chains
                const uint32_t cb = chunk_a;
                for (int tn = ng; tn < ntl; tn += 2 * ngr) {
                    double acc[2][4];
                    uint32_t ad[2][4];
                    bool ok[2][4];
                    const int tn2 = tn + ngr;
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const int colb = (h2 ? tn2 : tn) * 8;
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int li = r0 + g + (r >= 2 ? 8 : 0), col = colb + 2 * t4 + (r & 1);
                            ok[h2][r] = li < rc && col < nrest && (h2 == 0 || tn2 < ntl);
                            ad[h2][r] = ok[h2][r] ? cb + 8u * static_cast<uint32_t>((j0 + kt + col) * LD + li) : cb;
                            const double v = lds_f64(ad[h2][r]);
                            acc[h2][r] = ok[h2][r] ? v : 0.0;
                        }
                    }
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        if (ks < nk) {
#pragma unroll
                            for (int h2 = 0; h2 < 2; ++h2) {
                                const int yc = (h2 ? tn2 : tn) * 8 + g;
                                const bool yok = yc < nrest;
                                const double bv =
                                    lds_f64(part_a + 8u * static_cast<uint32_t>((4 * ks + t4) * nrest + (yok ? yc : 0)));
                                dmma(acc[h2], av[ks][0], av[ks][1], yok ? bv : 0.0);
                            }
                        }
                    }
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (ok[h2][r]) sts_f64(ad[h2][r], acc[h2][r]);
                }
            }
        }
        __syncthreads();
        if (trace && tid == 0 && rank == 0 && tph < 8) trace[64 * 8 + tph * 8 + 6] = clock64();
    }

    for (int idx = tid; idx < w * rc; idx += kT) {
        const int c = idx / rc, i = idx - c * rc;
        A[(r_beg + i) + static_cast<int64_t>(c) * lda] = S.chunk[static_cast<size_t>(c) * LD + i];
    }
    cluster.sync();  // no CTA exits while a peer may still write into it
}

int g_reg_cap = 0;  // dynamic shared memory cap for the kernel

void reg_init() {
    once_per_device(reinterpret_cast<const void*>(&g_reg_cap), [] {
        g_reg_cap = dyn_smem_cap(reinterpret_cast<const void*>(hqr_reg_kernel<1>));
        for (const void* f : {reinterpret_cast<const void*>(hqr_reg_kernel<1>),
                              reinterpret_cast<const void*>(hqr_reg_kernel<2>)}) {
            RUTV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            RUTV_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, g_reg_cap));
        }
    });
}


}  // namespace

// Largest column count the register kernel holds for s rows on cs CTAs (0 if
// the chunk is too tall for 2 rows per thread).
int qr_reg_capacity(int64_t s, int cs) {
    reg_init();
    const int64_t R = (s + cs - 1) / cs;
    if (R > 2 * kT) return 0;
    const int LD = static_cast<int>(R | 1);
    int w = static_cast<int>((g_reg_cap - 512) / (8 * (LD + 4 * KB)));
    while (w > 0 && reg_smem_doubles(w, LD, cs) * 8 > static_cast<size_t>(g_reg_cap) - 512) --w;
    return std::max(w, 0);
}

// Rows per CTA the cluster size is chosen for (env RUTV_QR_ROWS, default 256).
int qr_reg_rows() {
    static int rows = [] {
        const char* e = std::getenv("RUTV_QR_ROWS");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : 256;
    }();
    return rows;
}

void qr_reg_launch(cudaStream_t stream, const DView& a, double* tau, int cs) {
    reg_init();
    const int s = static_cast<int>(a.rows), w = static_cast<int>(a.cols);
    const int p = std::min(s, w);
    const int R = (s + cs - 1) / cs;
    const int LD = R | 1;
    const size_t smem = reg_smem_doubles(w, LD, cs) * 8;
    if (smem > static_cast<size_t>(g_reg_cap) || R > 2 * kT)
        throw Error(RUTV_ERR_INTERNAL, "hqr: sub-panel exceeds register-kernel capacity");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    static const bool tracing = std::getenv("RUTV_QR_TRACE") != nullptr;  // debug: per-column clock64 trace
    static const int ablate = [] {
        const char* e = std::getenv("RUTV_QR_ABLATE");
        const int v = e ? std::atoi(e) : 0;
        if (v) RUTV_CUDA(cudaMemcpyToSymbol(g_qr_ablate, &v, sizeof(int)));
        return v;
    }();
    (void)ablate;
    // RUTV_QR_CQ: 0 = column loop only, 1 (default) = CQ micro-panels; debug: 2 / 3 force the
    // pass-2 / pass-1 fallback on every odd micro-panel
    static const int cq_mode = [] {
        const char* e = std::getenv("RUTV_QR_CQ");
        return e ? std::atoi(e) : 1;
    }();
    long long* trace = nullptr;
    if (tracing) {
        RUTV_CUDA(cudaMalloc(&trace, 88 * 8 * sizeof(long long)));
        RUTV_CUDA(cudaMemset(trace, 0, 88 * 8 * sizeof(long long)));
    }
    if (R <= kT)
        RUTV_CUDA(cudaLaunchKernelEx(&cfg, hqr_reg_kernel<1>, a.data, a.ld, s, w, p, R, LD, tau, trace, cq_mode));
    else
        RUTV_CUDA(cudaLaunchKernelEx(&cfg, hqr_reg_kernel<2>, a.data, a.ld, s, w, p, R, LD, tau, trace, cq_mode));
    note_launch();
    if (tracing) {
        long long h[88 * 8];
        RUTV_CUDA(cudaStreamSynchronize(stream));
        RUTV_CUDA(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
        cudaFree(trace);
        std::fprintf(stderr, "qr_reg trace s=%d w=%d cs=%d (cycles: wait, house, update, reduce, send, next)\n", s, w, cs);
        for (int j = 0; j + 1 < std::min(p, 64); ++j) {
            const long long* r = h + j * 8;
            std::fprintf(stderr, "  col %2d: %6lld %6lld %6lld %6lld %6lld %6lld\n", j, r[1] - r[0], r[2] - r[1],
                         r[3] - r[2], h[(j + 1) * 8 + 4] - r[3], h[(j + 1) * 8 + 5] - h[(j + 1) * 8 + 4],
                         h[(j + 1) * 8 + 0] - h[(j + 1) * 8 + 5]);
        }
        std::fprintf(stderr,
                     "  CQ micro-panels (cycles: gram1, hop1, sum, chol, solve, gram2, hop2, E, products, LU, rows)\n");
        for (int mp = 0; mp < 8; ++mp) {
            const long long* r = h + 72 * 8 + mp * 16;
            if (!r[0]) continue;
            std::fprintf(stderr, "  mp %d:", mp);
            for (int k = 1; k < 12; ++k) std::fprintf(stderr, " %6lld", r[k] ? r[k] - r[k - 1] : -1LL);
            std::fprintf(stderr, " | gram1: dmma %lld slots %lld reduce+fence %lld sync %lld issue %lld\n", r[12] - r[0],
                         r[13] - r[12], r[14] - r[13], r[15] - r[14], r[1] - r[15]);
        }
        std::fprintf(stderr, "  block phases (cycles: partials, reduce-scatter, all-gather, T, Y, update)\n");
        for (int ph = 0; ph < 8; ++ph) {
            const long long* r = h + 64 * 8 + ph * 8;
            if (!r[0]) break;
            std::fprintf(stderr, "  phase %d: %6lld %6lld %6lld %6lld %6lld %6lld\n", ph, r[1] - r[0], r[2] - r[1],
                         r[3] - r[2], r[4] - r[3], r[5] - r[4], r[6] - r[5]);
        }
    }
}

}  // namespace rutv
