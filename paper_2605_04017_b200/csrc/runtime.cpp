// runtime.cpp -- library-owned device resources behind the kernels' per-call scratch.
//
// Every compute call is stream-ordered and capture-safe: its scratch (the trace's
// guard-band list, eval_map's tile counter) comes from cudaMallocFromPoolAsync on the
// caller's stream.  The pool is the LIBRARY's own (one per device, created on first use
// with a release threshold of "keep everything"), so repeated calls never reach
// cudaMalloc and no attribute of the process's default pool is changed.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "plt_internal.h"

namespace plt {

namespace {
std::mutex g_pool_mu;
std::vector<cudaMemPool_t> g_pools;   // indexed by device ordinal (nullptr = not yet created)
}  // namespace

static cudaError_t lib_pool(int dev, cudaMemPool_t* out) {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if ((int)g_pools.size() <= dev) g_pools.resize(dev + 1, nullptr);
    if (!g_pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        cudaError_t e = cudaMemPoolCreate(&p, &props);
        if (e != cudaSuccess) return e;
        uint64_t keep = ~0ull;
        e = cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        if (e != cudaSuccess) { cudaMemPoolDestroy(p); return e; }
        g_pools[dev] = p;
    }
    *out = g_pools[dev];
    return cudaSuccess;
}

int scratch_alloc(void** p, size_t bytes, void* stream) {
    *p = nullptr;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    cudaMemPool_t pool;
    e = lib_pool(dev, &pool);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaMallocFromPoolAsync(p, bytes, pool, (cudaStream_t)stream);
}

int scratch_free(void* p, void* stream) {
    return p ? (int)cudaFreeAsync(p, (cudaStream_t)stream) : 0;
}

}  // namespace plt
