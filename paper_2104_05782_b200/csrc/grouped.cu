// grouped.cu -- the deferred beta stage's small products as ONE launch each.
//
// beta_stage (proj/src/randutv_blocked.cpp:66-82, :150-154) multiplies finished
// blocks by the b x b SVD factors of every step:
//   right: X_i <- X_i M_i   (T(0:r0, r0:r0+w) and V(:, r0:r0+w) by Vs, U(:, r0:r0+w) by Us;
//                            right_multiply, :17-23)
//   left:  S_i <- M_i' S_i  (the strip T(r0:r0+b, r0+b:) by Us; left_multiply_t, :25-30)
// One launch per kind covers every step: a CTA owns a 64-row (right) or
// 64-column (left) tile of one X_i, stages it and M_i in shared memory, forms
// the product with warp-level DMMA (mma.sync m16n8k4 f64) and writes it back
// IN PLACE (the tile was fully read first).  Distinct steps touch disjoint
// blocks, so the whole group is one kernel instead of 2 x steps GEMM + copy
// launches.
#include <algorithm>
#include <vector>

#include "rutv_common.cuh"

namespace rutv {

namespace {

constexpr int kGT = 512;    // threads per CTA
constexpr int kTile = 64;   // rows (right) / columns (left) per CTA
constexpr int kWMax = 128;  // largest w handled in shared memory

struct TileRef {
    int desc;
    int off;  // first row (right) / column (left) of the tile
};

__device__ __forceinline__ void dmma(double* c, double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// LEFT = false: X is rows x w, out = X M.  LEFT = true: X is w x cols, out = M' X.
template <bool LEFT>
__global__ void __launch_bounds__(kGT, 1) small_mul_kernel(const SmallMulDesc* __restrict__ descs,
                                                           const TileRef* __restrict__ tiles) {
    extern __shared__ __align__(16) double sm[];
    const TileRef tr = tiles[blockIdx.x];
    const SmallMulDesc d = descs[tr.desc];
    const int w = d.w, wp = (w + 15) & ~15;  // w padded to the 16-row fragment
    // leading dimensions chosen so a fragment load (lanes g = 0..7, t4 = 0..3)
    // touches every 8-byte bank exactly twice: LD = 4 (mod 16) when the lane
    // offset is g * LD + t4, LD = 8 (mod 16) when it is t4 * LD + g
    const int LDM = wp + 4, LDX = LEFT ? wp + 4 : kTile + 8;
    double* Ms = sm;                      // M(k, j) at Ms[j * LDM + k]
    double* Xs = Ms + static_cast<size_t>(wp) * LDM;  // right: X(r, k) at Xs[k * LDX + r]; left: X(k, c) at Xs[c * LDX + k]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int64_t extent = LEFT ? d.cols : d.rows;
    const int cnt = static_cast<int>(std::min<int64_t>(kTile, extent - tr.off));

    // stage M and the X tile with asynchronous copies (every load in flight)
    auto cp8 = [](double* dst, const double* src) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src));
    };
    for (int e = tid; e < wp * wp; e += kGT) {
        const int k = e % wp, j = e / wp;
        if (k < w && j < w) cp8(Ms + j * LDM + k, d.M + k + static_cast<int64_t>(j) * d.ldm);
        else Ms[j * LDM + k] = 0.0;
    }
    if (!LEFT) {
        for (int e = tid; e < wp * kTile; e += kGT) {
            const int r = e % kTile, k = e / kTile;
            if (r < cnt && k < w) cp8(Xs + k * LDX + r, d.X + (tr.off + r) + static_cast<int64_t>(k) * d.ldx);
            else Xs[k * LDX + r] = 0.0;
        }
    } else {
        for (int e = tid; e < wp * kTile; e += kGT) {
            const int k = e % wp, c = e / wp;
            if (c < cnt && k < w) cp8(Xs + c * LDX + k, d.X + k + static_cast<int64_t>(tr.off + c) * d.ldx);
            else Xs[c * LDX + k] = 0.0;
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // output tile OM x ON in 16 x 8 fragments
    const int OM = LEFT ? wp : kTile, ON = LEFT ? kTile : wp;
    const int nm = OM / 16, nn = ON / 8;
    // each warp: two 16 x 8 fragments with the same rows (independent DMMA chains)
    const int nn2 = (nn + 1) / 2;
    for (int u = warp; u < nm * nn2; u += kGT / 32) {
        const int mt = u % nm, nt = (u / nm) * 2;
        const int m0 = mt * 16;
        const bool two = nt + 1 < nn;
        double acc[2][4] = {};
        for (int k0 = 0; k0 < wp; k0 += 4) {
            const int k = k0 + t4;
            double a0, a1, b0, b1;
            if (!LEFT) {  // A = X (rows m, cols k), B = M (k, n)
                a0 = Xs[k * LDX + m0 + g];
                a1 = Xs[k * LDX + m0 + g + 8];
                b0 = Ms[(nt * 8 + g) * LDM + k];
                b1 = two ? Ms[(nt * 8 + 8 + g) * LDM + k] : 0.0;
            } else {  // A = M' (m, k) = M(k, m), B = X (k, n)
                a0 = Ms[(m0 + g) * LDM + k];
                a1 = Ms[(m0 + g + 8) * LDM + k];
                b0 = Xs[(nt * 8 + g) * LDX + k];
                b1 = two ? Xs[(nt * 8 + 8 + g) * LDX + k] : 0.0;
            }
            dmma(acc[0], a0, a1, b0);
            dmma(acc[1], a0, a1, b1);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
            const int n0 = (nt + h) * 8;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = m0 + g + (r >= 2 ? 8 : 0), col = n0 + 2 * t4 + (r & 1);
                if (!LEFT) {
                    if (row < cnt && col < w) d.X[(tr.off + row) + static_cast<int64_t>(col) * d.ldx] = acc[h][r];
                } else {
                    if (row < w && col < cnt) d.X[row + static_cast<int64_t>(tr.off + col) * d.ldx] = acc[h][r];
                }
            }
        }
    }
}

// block_i := rect-diag(sigma_i) (randutv_blocked.cpp:32-37); blockIdx.y selects the
// block, the x CTAs of a row stride over it (config 5's first block is 50000 x 512:
// one CTA per block made the whole launch wait ~6 ms on it).
__global__ void rect_diag_grouped_kernel(const RectDiagDesc* __restrict__ descs) {
    const RectDiagDesc d = descs[blockIdx.y];
    const int64_t total = d.rows * d.cols;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % d.rows, c = e / d.rows;
        d.A[r + c * d.ld] = (r == c && r < d.p) ? d.sigma[r] : 0.0;
    }
}

}  // namespace

void rect_diag_grouped(cudaStream_t st, const std::vector<RectDiagDesc>& descs, void* dev_scratch,
                       size_t scratch_bytes) {
    if (descs.empty()) return;
    const size_t db = descs.size() * sizeof(RectDiagDesc);
    if (db > scratch_bytes) throw Error(RUTV_ERR_INTERNAL, "rect_diag_grouped: scratch too small");
    RUTV_CUDA(cudaMemcpyAsync(dev_scratch, descs.data(), db, cudaMemcpyHostToDevice, st));
    int64_t most = 1;
    for (const auto& d : descs) most = std::max(most, d.rows * d.cols);
    // enough CTAs per block for the largest; a grid of about 8 waves overall
    const int64_t per = std::min<int64_t>((most + 1023) / 1024,
                                          std::max<int64_t>(1, 8 * kNumSMs / static_cast<int64_t>(descs.size())));
    rect_diag_grouped_kernel<<<dim3(static_cast<unsigned>(per), static_cast<unsigned>(descs.size())), 1024, 0, st>>>(
        static_cast<const RectDiagDesc*>(dev_scratch));
    note_launch();
    RUTV_CHECK_LAUNCH();
}

int small_mul_max_w() { return kWMax; }

// descs: host array (copied to `dev_scratch`), all with w <= kWMax.
void small_mul_grouped(cudaStream_t st, bool left, const std::vector<SmallMulDesc>& descs, void* dev_scratch,
                       size_t scratch_bytes) {
    if (descs.empty()) return;
    std::vector<TileRef> tiles;
    int wmax = 0;
    for (size_t i = 0; i < descs.size(); ++i) {
        const SmallMulDesc& d = descs[i];
        if (d.w > kWMax) throw Error(RUTV_ERR_INTERNAL, "small_mul: block wider than 128");
        wmax = std::max(wmax, d.w);
        const int64_t extent = left ? d.cols : d.rows;
        for (int64_t o = 0; o < extent; o += kTile) tiles.push_back({static_cast<int>(i), static_cast<int>(o)});
    }
    if (tiles.empty() || wmax == 0) return;
    const size_t db = descs.size() * sizeof(SmallMulDesc), tb = tiles.size() * sizeof(TileRef);
    if (db + tb + 16 > scratch_bytes) throw Error(RUTV_ERR_INTERNAL, "small_mul: scratch too small");
    char* base = static_cast<char*>(dev_scratch);
    RUTV_CUDA(cudaMemcpyAsync(base, descs.data(), db, cudaMemcpyHostToDevice, st));
    TileRef* dt = reinterpret_cast<TileRef*>(base + ((db + 15) & ~size_t(15)));
    RUTV_CUDA(cudaMemcpyAsync(dt, tiles.data(), tb, cudaMemcpyHostToDevice, st));
    const int wp = (wmax + 15) & ~15;
    const size_t smem = (static_cast<size_t>(wp) * (wp + 4) +
                         static_cast<size_t>(left ? kTile : wp) * (left ? wp + 4 : kTile + 8)) *
                        sizeof(double);
    once_per_device(reinterpret_cast<const void*>(small_mul_kernel<true>), [] {
        const int capl = dyn_smem_cap(reinterpret_cast<const void*>(small_mul_kernel<true>));
        const int capr = dyn_smem_cap(reinterpret_cast<const void*>(small_mul_kernel<false>));
        RUTV_CUDA(cudaFuncSetAttribute(small_mul_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, capl));
        RUTV_CUDA(cudaFuncSetAttribute(small_mul_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, capr));
    });
    const auto* dd = reinterpret_cast<const SmallMulDesc*>(base);
    if (left)
        small_mul_kernel<true><<<static_cast<unsigned>(tiles.size()), kGT, smem, st>>>(dd, dt);
    else
        small_mul_kernel<false><<<static_cast<unsigned>(tiles.size()), kGT, smem, st>>>(dd, dt);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

size_t small_mul_scratch_bytes(size_t ndesc, int64_t total_extent) {
    return ndesc * sizeof(SmallMulDesc) + 16 + static_cast<size_t>(total_extent / kTile + ndesc + 1) * 8 + 64;
}

}  // namespace rutv
