// splat_dev.cuh -- the per-hit sensor splat as a warp-synchronous device function, shared
// by the stand-alone splat kernel and the fused query kernels (trace / eval_map epilogues).
//
// Eq. 8 accumulates I_out^P * h(x_out^P) * G over the valid paths;
// Listing 1 adds I_out * dot(w_out, n_cmos) into the pixel of p_out.  With a
// one-pixel box filter h and G = |w_z|, each valid hit adds
// llrint(I * |w_z| * scale * 2^32) to film[c][iy][ix].  All arithmetic that decides the
// pixel and the fixed-point weight is IEEE double with explicit round-to-nearest
// intrinsics (no FMA contraction) or provably equal to it, so the integer sum is exact,
// order independent and bit-identical whichever kernel performs it.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "plt_internal.h"

namespace plt {

// Pixel key (or -1 with drop = true) and fixed-point weight of one valid hit.  Films are
// limited to < 2^31 entries (checked at the ABI), so the key is a 32-bit int and the warp
// groups lanes with the 32-bit __match_any_sync.
__device__ __forceinline__ int splat_key(const SplatCtx& c, float px, float py, float dz, float I, int ch,
                                         long long& w, bool& drop) {
    // Pixel coordinate: fp32 estimate first.  Its error is below c.guard (derived from the
    // film size in make_splat_ctx), so when it lies more than c.guard from an integer its
    // floor equals the floor of the exact double expression of O11; only hits near a pixel
    // edge evaluate the double expression (bit-exact film for any film size).
    const float fxs = (px - c.cxf + c.hwf) * c.sxf, fys = (c.hhf - (py - c.cyf)) * c.syf;
    int ix, iy;
    bool in;
    if (fabsf(fxs - rintf(fxs)) < c.guard || fabsf(fys - rintf(fys)) < c.guard) {
        const double fx = __dmul_rn(__ddiv_rn(__dadd_rn(__dsub_rn((double)px, c.cx), c.W * 0.5), c.W), (double)c.width);
        const double fy = __dmul_rn(__ddiv_rn(__dsub_rn(c.H * 0.5, __dsub_rn((double)py, c.cy)), c.H), (double)c.height);
        const double fxf = floor(fx), fyf = floor(fy);
        in = fxf >= 0.0 && fxf < (double)c.width && fyf >= 0.0 && fyf < (double)c.height;
        ix = in ? (int)fxf : 0;
        iy = in ? (int)fyf : 0;
    } else {
        // no pixel edge (integer) within the error bound: signs and floors of the fp32 estimate
        // are those of O11's double expression; NaN fails the >= 0 tests, far hits saturate
        ix = __float2int_rd(fxs);
        iy = __float2int_rd(fys);
        in = fxs >= 0.f && fys >= 0.f && ix < c.width && iy < c.height;
    }
    if (in && ch < c.channels) {
        // (I |w_z| scale) 2^32 with ONE rounding after I |w_z| (exact in double) as in O11: the
        // factor 2^32 is exact, so multiplying by scale 2^32 rounds identically
        w = __double2ll_rn(__dmul_rn(__dmul_rn((double)I, fabs((double)dz)), c.wscale));
        return (ch * c.height + iy) * c.width + ix;
    }
    drop = true;
    return -1;
}

// Lanes whose hits share a pixel found with __match_any_sync; the lowest lane sums the
// group's weights through `wsm` (this warp's 32 shared-memory slots) and issues ONE 64-bit
// atom.add per distinct pixel per warp.  All 32 lanes call it.
__device__ __forceinline__ void splat_aggregate(const SplatCtx& c, long long* wsm, int key, long long w) {
    const int lane = threadIdx.x & 31;
    wsm[lane] = w;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && lane == __ffs(peers) - 1) {
        long long sum = 0;
        for (unsigned p = peers; p; p &= p - 1) sum += wsm[__ffs(p) - 1];
        atomicAdd(reinterpret_cast<unsigned long long*>(c.film + key), (unsigned long long)sum);
    }
    __syncwarp();
}

// Warp-synchronous splat: ALL 32 lanes call it (hit = false for lanes without a valid
// hit).  Aggregate only where it pays: if no two neighbouring lanes share a pixel (a
// spread-out image: the warp's hits almost surely land on 32 distinct pixels) every lane
// adds its own weight; otherwise (a bright spot) lanes with the same pixel are grouped and
// summed first.  Integer adds: the film is the same either way.
__device__ __forceinline__ void splat_warp(const SplatCtx& c, long long* wsm, bool hit, float px, float py,
                                           float dz, float I, int ch) {
    const int lane = threadIdx.x & 31;
    int key = -1;
    long long w = 0;
    bool drop = false;
    if (hit) key = splat_key(c, px, py, dz, I, ch, w, drop);
    const int nb = __shfl_down_sync(0xffffffffu, key, 1);
    if (!__any_sync(0xffffffffu, lane < 31 && key >= 0 && key == nb)) {
        if (key >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(c.film + key), (unsigned long long)w);
    } else {
        splat_aggregate(c, wsm, key, w);
    }
    const unsigned dm = __ballot_sync(0xffffffffu, drop);
    if (c.dropped && lane == 0 && dm) atomicAdd(c.dropped, (unsigned long long)__popc(dm));
    __syncwarp();
}

// Two hits per lane (the packed trace's ray pair) in one warp-synchronous pass: the
// neighbour test, the vote and the drop count are shared by both hits (half the warp-level
// instructions of two splat_warp calls); the atomics are the same, so is the film.
__device__ __forceinline__ void splat_warp2(const SplatCtx& c, long long* wsm, bool hit0, float px0, float py0,
                                            float dz0, float I0, int ch0, bool hit1, float px1, float py1,
                                            float dz1, float I1, int ch1) {
    const int lane = threadIdx.x & 31;
    int k0 = -1, k1 = -1;
    long long w0 = 0, w1 = 0;
    bool d0 = false, d1 = false;
    if (hit0) k0 = splat_key(c, px0, py0, dz0, I0, ch0, w0, d0);
    if (hit1) k1 = splat_key(c, px1, py1, dz1, I1, ch1, w1, d1);
    const int nb0 = __shfl_down_sync(0xffffffffu, k0, 1), nb1 = __shfl_down_sync(0xffffffffu, k1, 1);
    const bool clash = lane < 31 && ((k0 >= 0 && k0 == nb0) || (k1 >= 0 && k1 == nb1));
    if (!__any_sync(0xffffffffu, clash)) {
        if (k0 >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(c.film + k0), (unsigned long long)w0);
        if (k1 >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(c.film + k1), (unsigned long long)w1);
    } else {
        splat_aggregate(c, wsm, k0, w0);
        splat_aggregate(c, wsm, k1, w1);
    }
    if (c.dropped) {
        const int nd = __popc(__ballot_sync(0xffffffffu, d0)) + __popc(__ballot_sync(0xffffffffu, d1));
        if (lane == 0 && nd) atomicAdd(c.dropped, (unsigned long long)nd);
    }
    __syncwarp();
}

}  // namespace plt
