// camera.cu -- the backward camera integrand with a procedural scene (SURVEY.md §8(f)
// NEXT-3; Eq. 9; the depth-of-field integrator of P:422-427) and
// free-space ray propagation (sensor-shift focusing with one precomputed map).
//
// shade_plane: a valid exit ray of a BACKWARD query (origin on z = z_hits, direction to
// -z) continues in air to the scene plane z = z_scene; its radiance is a checkerboard,
// L = 1 on even squares and `contrast` on odd ones; film[i / spp] += llrint(I L s 2^32).
// The arithmetic that decides the square and the weight is IEEE double with explicit
// round-to-nearest intrinsics (the oracle's order), so the integer film is exact, order
// independent and bit-identical to oracle.shade_plane.  Consecutive rays of a pixel are
// summed per warp before one 64-bit atomic (__match_any_sync on the pixel).
#include <cuda_runtime.h>

#include "plt_internal.h"

namespace plt {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) shade_plane_kernel(ScenePlane sc, double z_hits, plt_hits hits, int spp,
                                                               int64_t pixels, float scale, int64_t* film, int64_t n,
                                                               const float* in_dz) {
    __shared__ long long wsm[kThreads];
    const int lane = threadIdx.x & 31, warp0 = threadIdx.x & ~31;
    for (int64_t base = (int64_t)blockIdx.x * kThreads + warp0; base < n; base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + lane;
        long long key = -1, w = 0;
        if (i < n && ((__ldg(hits.mask_bits + (i >> 5)) >> (i & 31)) & 1u)) {
            const double dz = (double)__ldg(hits.dz + i);
            const double t = __ddiv_rn(__dsub_rn(sc.z, z_hits), dz);
            const int64_t pix = i / spp;
            if (t > 0.0 && pix < pixels) {
                const double x = __dadd_rn((double)__ldg(hits.px + i), __dmul_rn(t, (double)__ldg(hits.dx + i)));
                const double y = __dadd_rn((double)__ldg(hits.py + i), __dmul_rn(t, (double)__ldg(hits.dy + i)));
                const long long q = (long long)floor(__ddiv_rn(x, sc.period)) + (long long)floor(__ddiv_rn(y, sc.period));
                const double L = (q & 1) ? sc.contrast : 1.0;
                double IL = __dmul_rn((double)__ldg(hits.throughput + i), L);
                if (in_dz) {   // pupil-sampling weight cos^4(theta) of the sensor ray (plt_shade_plane_weighted)
                    const double c = (double)__ldg(in_dz + i), c2 = __dmul_rn(c, c);
                    IL = __dmul_rn(IL, __dmul_rn(c2, c2));
                }
                w = __double2ll_rn(__dmul_rn(__dmul_rn(IL, (double)scale), 4294967296.0));
                key = pix;
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
        __syncwarp();
    }
}

// Several cards (plt_shade_cards): the nearest card whose rectangle contains the hit.
__global__ void __launch_bounds__(kThreads) shade_cards_kernel(const __grid_constant__ SceneCards sc, double z_hits,
                                                               plt_hits hits, int spp, int64_t pixels, float scale,
                                                               int64_t* film, int64_t n, const float* in_dz) {
    __shared__ long long wsm[kThreads];
    const int lane = threadIdx.x & 31, warp0 = threadIdx.x & ~31;
    for (int64_t base = (int64_t)blockIdx.x * kThreads + warp0; base < n; base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + lane;
        long long key = -1, w = 0;
        if (i < n && ((__ldg(hits.mask_bits + (i >> 5)) >> (i & 31)) & 1u)) {
            const int64_t pix = i / spp;
            if (pix < pixels) {
                const double dz = (double)__ldg(hits.dz + i), px = (double)__ldg(hits.px + i),
                             py = (double)__ldg(hits.py + i), dx = (double)__ldg(hits.dx + i),
                             dy = (double)__ldg(hits.dy + i);
                double L = sc.background, best = 0.0;
                bool found = false;
                for (int k = 0; k < sc.n; ++k) {
                    const double t = __ddiv_rn(__dsub_rn(sc.z[k], z_hits), dz);
                    if (!(t > 0.0) || (found && !(t < best))) continue;
                    const double x = __dadd_rn(px, __dmul_rn(t, dx)), y = __dadd_rn(py, __dmul_rn(t, dy));
                    if (x < sc.x0[k] || x > sc.x1[k] || y < sc.y0[k] || y > sc.y1[k]) continue;
                    const long long q = (long long)floor(__ddiv_rn(x, sc.period[k])) +
                                        (long long)floor(__ddiv_rn(y, sc.period[k]));
                    L = (q & 1) ? sc.contrast[k] : 1.0;
                    best = t;
                    found = true;
                }
                double IL = __dmul_rn((double)__ldg(hits.throughput + i), L);
                if (in_dz) {
                    const double c = (double)__ldg(in_dz + i), c2 = __dmul_rn(c, c);
                    IL = __dmul_rn(IL, __dmul_rn(c2, c2));
                }
                w = __double2ll_rn(__dmul_rn(__dmul_rn(IL, (double)scale), 4294967296.0));
                key = pix;
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
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kThreads) propagate_kernel(plt_rays in, plt_rays out, float z_target, float sdir,
                                                              int64_t n) {
    const float z0 = (float)in.plane_z_mm;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
        const float dx = in.dx[i], dy = in.dy[i];
        float dz;
        if (in.dz) {
            dz = in.dz[i];
        } else {   // omega in S^2_+  given by (dx, dy), with the sign of the query direction
            const float m = sqrtf(fmaxf(0.f, fmaf(-dx, dx, fmaf(-dy, dy, 1.f))));
            dz = sdir * m;
        }
        const float t = __fdiv_rn(__fsub_rn(z_target, z0), dz);
        const float lam = in.lambda_nm[i], ox = __fmaf_rn(t, dx, in.ox[i]), oy = __fmaf_rn(t, dy, in.oy[i]);
        // plt_rays carries const pointers; `out` is the caller's writable destination (may alias `in`)
        const_cast<float*>(out.ox)[i] = ox;
        const_cast<float*>(out.oy)[i] = oy;
        const_cast<float*>(out.dx)[i] = dx;
        const_cast<float*>(out.dy)[i] = dy;
        if (out.dz) const_cast<float*>(out.dz)[i] = dz;
        const_cast<float*>(out.lambda_nm)[i] = lam;
    }
}

int blocks_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t b = (n + kThreads - 1) / kThreads;
    if (b > (int64_t)sms * 16) b = (int64_t)sms * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

int launch_shade_plane(const ScenePlane& sc, double z_hits, const plt_hits& hits, int spp, int64_t pixels,
                       float scale, int64_t* film, int64_t n, void* stream, const float* in_dz) {
    shade_plane_kernel<<<blocks_for(n), kThreads, 0, (cudaStream_t)stream>>>(sc, z_hits, hits, spp, pixels, scale,
                                                                             film, n, in_dz);
    return (int)cudaGetLastError();
}

int launch_shade_cards(const SceneCards& sc, double z_hits, const plt_hits& hits, int spp, int64_t pixels,
                       float scale, int64_t* film, int64_t n, void* stream, const float* in_dz) {
    shade_cards_kernel<<<blocks_for(n), kThreads, 0, (cudaStream_t)stream>>>(sc, z_hits, hits, spp, pixels, scale,
                                                                             film, n, in_dz);
    return (int)cudaGetLastError();
}

int launch_propagate(const plt_rays& in, const plt_rays& out, float z_target, float sdir, int64_t n, void* stream) {
    propagate_kernel<<<blocks_for(n), kThreads, 0, (cudaStream_t)stream>>>(in, out, z_target, sdir, n);
    return (int)cudaGetLastError();
}

}  // namespace plt
