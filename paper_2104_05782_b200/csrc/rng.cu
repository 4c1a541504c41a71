// rng.cu -- on-device counter-based Gaussian stream (compiled with --fmad=false).
//
// Restates RngState (proj/include/randutv/rng.hpp:18-46, proj/src/rng.cpp:9-53):
// word(c) = mix64(seed + (c+1)*0x9E3779B97F4A7C15) is integer-exact on any
// device; uniform/normal_at use the same expression order as the reference.
// log/sqrt/cos/sin come from CUDA's libdevice (sqrt is IEEE exact; log, cos,
// sin are within 1-2 ulp of glibc), so deviates can differ from the host
// stream in the last bit -- the parity mode of rutv_b200_factorize takes G
// from the host instead.
#include "rutv_common.cuh"

namespace rutv {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

__host__ __device__ __forceinline__ uint64_t rng_word(uint64_t seed, uint64_t c) {
    return mix64(seed + (c + 1) * 0x9E3779B97F4A7C15ULL);
}

__host__ __device__ __forceinline__ double normal_at(uint64_t seed, uint64_t d) {
    const uint64_t p = d >> 1;
    const double u1 = static_cast<double>((rng_word(seed, 2 * p) >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(rng_word(seed, 2 * p + 1) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    return (d & 1) == 0 ? r * cos(th) : r * sin(th);
}

__global__ void normal_fill_kernel(uint64_t seed, uint64_t pos, int64_t rows, int64_t cols,
                                   double* g, int64_t ld) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i % rows, c = i / rows;
        g[r + c * ld] = normal_at(seed, pos + static_cast<uint64_t>(i));
    }
}

void normal_fill(cudaStream_t stream, uint64_t seed, uint64_t pos, const DView& g) {
    const int64_t total = g.rows * g.cols;
    if (total == 0) return;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs));
    normal_fill_kernel<<<blocks, 256, 0, stream>>>(seed, pos, g.rows, g.cols, g.data, g.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

// Block-cyclic rows of a step's G (s x cols, column-major in the stream):
// out(lr, j) = G((first + (lr / b) * stride) * b + lr % b, j), i.e. deviate
// pos + that row + j * s -- a rank's own rows of the replicated sketch matrix,
// drawn without communication (the stream is counter-based, rng.hpp:9-17).
__global__ void normal_fill_cyclic_kernel(uint64_t seed, uint64_t pos, int64_t s, int64_t b, int64_t first,
                                          int64_t stride, int64_t rows, int64_t cols, double* g, int64_t ld) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i % rows, c = i / rows;
        const int64_t gr = (first + (r / b) * stride) * b + r % b;
        g[r + c * ld] = normal_at(seed, pos + static_cast<uint64_t>(gr + c * s));
    }
}

void normal_fill_cyclic(cudaStream_t stream, uint64_t seed, uint64_t pos, int64_t s, int64_t b, int64_t first,
                        int64_t stride, const DView& g) {
    const int64_t total = g.rows * g.cols;
    if (total == 0) return;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs));
    normal_fill_cyclic_kernel<<<blocks, 256, 0, stream>>>(seed, pos, s, b, first, stride, g.rows, g.cols, g.data,
                                                          g.ld);
    note_launch();
    RUTV_CHECK_LAUNCH();
}

}  // namespace rutv

// Host evaluation of the same expression (glibc log / sqrt / cos / sin, no
// contraction): bit-identical to the reference's RngState::normal_at
// (rng.cpp:29-36); backs the drop-in header's RngState.
extern "C" double rutv_b200_normal_at(uint64_t seed, uint64_t d) { return rutv::normal_at(seed, d); }
