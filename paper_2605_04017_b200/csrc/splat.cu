// splat.cu -- sensor splatting into an int64 fixed-point film and film resolve (sm_100a).
//
// Eq. 8 accumulates I_out^P * h(x_out^P) * G over the valid
// paths; Listing 1 adds I_out * dot(w_out, n_cmos) into the pixel of
// p_out.  With a one-pixel box filter h and G = |w_z|, each valid hit
// adds llrint(I * |w_z| * scale * 2^32) to film[c][iy][ix].  All arithmetic that
// decides the pixel and the fixed-point weight is IEEE double with explicit
// round-to-nearest intrinsics (no FMA contraction), so the integer sum is exact,
// order independent and bit-identical across runs and GPU counts.
//
// Warp-aggregated atomics: lanes whose hits share a pixel find each other with
// __match_any_sync; the lowest lane sums the group's weights from shared memory and
// issues ONE 64-bit atom.add per distinct pixel per warp (bright compact ghosts
// otherwise serialise on a few L2 atomic units).
#include <cuda_runtime.h>

#include "plt_internal.h"

namespace plt {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) splat_kernel(plt_film_desc fd, int64_t* __restrict__ film,
                                                         plt_hits hits, const uint8_t* __restrict__ channel,
                                                         float scale, int64_t n,
                                                         unsigned long long* dropped) {
    constexpr int kUnroll = 2;   // rays per thread per iteration (all loads issued up front)
    __shared__ long long wsm[kThreads];
    const int lane = threadIdx.x & 31;
    const int warp0 = threadIdx.x & ~31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kUnroll;
    const double W = fd.sensor_w_mm, H = fd.sensor_h_mm;
    constexpr float kGuard = 2e-3f;
    const float cxf = (float)fd.center_x_mm, cyf = (float)fd.center_y_mm;
    const float hwf = (float)(0.5 * W), hhf = (float)(0.5 * H);
    const float sxf = (float)(fd.width_px / W), syf = (float)(fd.height_px / H);
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
            ch[u] = (in && channel) ? (int)__ldg(channel + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            long long key = -1, w = 0;
            bool drop = false;
            if ((word[u] >> lane) & 1u) {
                // Pixel coordinate: fp32 estimate first.  Its error is < 1e-3 px for any
                // film below 10^5 px, so when it lies more than kGuard from an integer its
                // floor equals the floor of the exact double expression of O11; only rays
                // near a pixel edge evaluate the double expression (bit-exact film).
                float fxs = (px[u] - cxf + hwf) * sxf, fys = (hhf - (py[u] - cyf)) * syf;
                double fxf = floorf(fxs), fyf = floorf(fys);
                if (fabsf(fxs - rintf(fxs)) < kGuard || fabsf(fys - rintf(fys)) < kGuard) {
                    const double fx = __dmul_rn(__ddiv_rn(__dadd_rn(__dsub_rn((double)px[u], fd.center_x_mm), W * 0.5), W),
                                                (double)fd.width_px);
                    const double fy = __dmul_rn(__ddiv_rn(__dsub_rn(H * 0.5, __dsub_rn((double)py[u], fd.center_y_mm)), H),
                                                (double)fd.height_px);
                    fxf = floor(fx); fyf = floor(fy);
                }
                if (fxf >= 0.0 && fxf < (double)fd.width_px && fyf >= 0.0 && fyf < (double)fd.height_px &&
                    ch[u] < fd.channels) {
                    key = ((long long)ch[u] * fd.height_px + (long long)fyf) * fd.width_px + (long long)fxf;
                    w = __double2ll_rn(__dmul_rn(__dmul_rn(__dmul_rn((double)I[u], fabs((double)dz[u])), (double)scale),
                                                 4294967296.0));
                } else {
                    drop = true;
                }
            }
            wsm[threadIdx.x] = w;
            __syncwarp();
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            if (key >= 0 && lane == __ffs(peers) - 1) {
                long long sum = 0;
                for (unsigned p = peers; p; p &= p - 1) sum += wsm[warp0 + __ffs(p) - 1];
                atomicAdd(reinterpret_cast<unsigned long long*>(film + key), (unsigned long long)sum);
            }
            const unsigned dm = __ballot_sync(0xffffffffu, drop);
            if (dropped && lane == 0 && dm) atomicAdd(dropped, (unsigned long long)__popc(dm));
            __syncwarp();
        }
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
    int64_t blocks = (n + 2 * kThreads - 1) / (2 * kThreads);
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    splat_kernel<<<(int)blocks, kThreads, 0, (cudaStream_t)stream>>>(fd, film, hits, channel, scale, n, dropped);
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
