// runtime.cu -- per-device library state: one-time kernel attribute setup and
// the library-owned stream-ordered memory pool.
//
// The reference allocates every temporary with std::vector (matrix.hpp:63-118)
// and keeps no global state; the B200 library must likewise
// leave the host process's device state alone.  It therefore owns ONE
// cudaMemPool_t per device (never the device's default pool, which torch and
// other host allocators share) and trims it back to a bounded cache at the end
// of every public call, so a 60 GB config-5 workspace is returned to the
// driver instead of being held after the call.
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <utility>

#include "rutv_common.cuh"

namespace rutv {

namespace {

std::recursive_mutex g_once_mu;
std::set<std::pair<int, const void*>> g_once_done;

std::mutex g_pool_mu;
std::map<int, cudaMemPool_t> g_pools;

size_t keep_bytes() {
    static const size_t keep = [] {
        const char* e = std::getenv("RUTV_POOL_KEEP_MB");
        const long long mb = e ? std::atoll(e) : 4096;  // default: keep up to 4 GB cached
        return static_cast<size_t>(mb < 0 ? 0 : mb) << 20;
    }();
    return keep;
}

cudaMemPool_t pool_for(int dev) {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it != g_pools.end()) return it->second;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    RUTV_CUDA(cudaMemPoolCreate(&pool, &props));
    // hold freed blocks inside a call (no re-mapping between steps); trimmed at call end
    uint64_t thr = UINT64_MAX;
    RUTV_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_pools[dev] = pool;
    return pool;
}

}  // namespace

void once_per_device(const void* key, const std::function<void()>& init) {
    int dev = 0;
    RUTV_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::recursive_mutex> g(g_once_mu);
    if (g_once_done.count({dev, key})) return;
    init();
    g_once_done.insert({dev, key});
}

void* dev_alloc(size_t bytes, cudaStream_t st) {
    int dev = 0;
    RUTV_CUDA(cudaGetDevice(&dev));
    void* p = nullptr;
    const cudaError_t e = cudaMallocFromPoolAsync(&p, bytes ? bytes : 8, pool_for(dev), st);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw Error(RUTV_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    if (e != cudaSuccess) throw Error(RUTV_ERR_CUDA, std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
    return p;
}

namespace {
thread_local bool t_keep = false;
}

void pool_keep_this_call(bool keep) { t_keep = keep; }

void pool_release(int dev) {
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> g(g_pool_mu);
        auto it = g_pools.find(dev);
        if (it == g_pools.end()) return;
        pool = it->second;
    }
    cudaMemPoolTrimTo(pool, 0);
}

void pool_trim() {
    if (t_keep) {  // the caller asked to keep this call's workspace (rutv_opts.keep_workspace)
        t_keep = false;
        return;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> g(g_pool_mu);
        auto it = g_pools.find(dev);
        if (it == g_pools.end()) return;
        pool = it->second;
    }
    cudaMemPoolTrimTo(pool, keep_bytes());
}

}  // namespace rutv
