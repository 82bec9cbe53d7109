// splat.cu -- sensor splatting of a hits buffer into an int64 fixed-point film, and film
// resolve (sm_100a).  The per-hit arithmetic (Eq. 8; Listing 1) and
// the warp-aggregated atomics live in splat_dev.cuh, shared with the fused query
// kernels; bright compact ghosts would otherwise serialise on a few L2 atomic units.
#include <cuda_runtime.h>

#include "plt_internal.h"
#include "splat_dev.cuh"

namespace plt {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) splat_kernel(SplatCtx ctx, plt_hits hits, int64_t n) {
#ifndef PLT_SPLAT_UNROLL
#define PLT_SPLAT_UNROLL 2
#endif
    constexpr int kUnroll = PLT_SPLAT_UNROLL;   // rays per thread per iteration (all loads issued up front)
    __shared__ long long wsm[kThreads];
    const int lane = threadIdx.x & 31;
    const int warp0 = threadIdx.x & ~31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kUnroll;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * kUnroll + warp0 * kUnroll; base < n; base += stride) {
        uint32_t word[kUnroll];
        float px[kUnroll], py[kUnroll], dz[kUnroll], I[kUnroll];
        int ch[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {      // independent loads: one memory latency per iteration
            const int64_t i = base + 32 * u + lane;
            const bool in = i < n;
            word[u] = in ? __ldg(hits.mask_bits + (i >> 5)) : 0u;
            px[u] = in ? __ldg(hits.px + i) : 0.f;
            py[u] = in ? __ldg(hits.py + i) : 0.f;
            dz[u] = in ? __ldg(hits.dz + i) : 0.f;
            I[u] = in ? __ldg(hits.throughput + i) : 0.f;
            ch[u] = (in && ctx.channel) ? (int)__ldg(ctx.channel + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            splat_warp(ctx, wsm + warp0, (word[u] >> lane) & 1u, px[u], py[u], dz[u], I[u], ch[u]);
    }
}

__global__ void resolve_kernel(const int64_t* __restrict__ film, float* __restrict__ out, int64_t n, double scale) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (float)((double)film[i] * (scale * 2.3283064365386963e-10));
}

}  // namespace

int launch_splat(const plt_film_desc& fd, int64_t* film, const plt_hits& hits, const uint8_t* channel,
                 float scale, int64_t n, unsigned long long* dropped, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n + PLT_SPLAT_UNROLL * kThreads - 1) / (PLT_SPLAT_UNROLL * kThreads);
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    splat_kernel<<<(int)blocks, kThreads, 0, (cudaStream_t)stream>>>(make_splat_ctx(fd, film, channel, scale, dropped),
                                                                     hits, n);
    return (int)cudaGetLastError();
}

int launch_resolve(const plt_film_desc& fd, const int64_t* film, float* out, double scale, void* stream) {
    const int64_t n = (int64_t)fd.channels * fd.height_px * fd.width_px;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    resolve_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(film, out, n, scale);
    return (int)cudaGetLastError();
}

}  // namespace plt
