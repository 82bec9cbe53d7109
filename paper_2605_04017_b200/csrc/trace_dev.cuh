// trace_dev.cuh -- device code of the float32 trace shared by the ahead-of-time kernels
// (trace.cu) and the run-time specialised ones (trace_jit.cpp compiles this file with
// NVRTC after appending a path program baked in as compile-time constants).
//
// Packed float32 trace: every thread carries TWO rays in float2 registers, so the ray
// arithmetic issues as FFMA2 / FMUL2 / FADD2 (one instruction for both rays) while the
// per-lane work -- comparisons, guard-band tests, MUFU rcp/rsqrt -- addresses the halves
// of the register pairs directly, and the path program loads, loop control and warp
// votes are shared by the two rays.  Same operators, order and guard bands as the scalar
// ray_steps<float> of trace.cu (Eq. 5-7, O4-O8); only the instruction packing differs.
#pragma once

#ifndef PLT_JIT
#include <cuda_runtime.h>
#include <cstdint>

#include "plt_internal.h"
#include "splat_dev.cuh"
#endif

namespace plt {

constexpr float kEpsT = 1e-6f;          // self-hit epsilon, mm
// Guard bands of the float32 pass: far above
// the float32 error of an all-T trace (~3e-5 mm, SURVEY [B1]).
constexpr float kBandEdge = 5e-4f;      // mm, on |rho - a|, sensor edges
constexpr float kBandKappa = 1e-4f;     // on |kappa| = cos^2(theta_t)
constexpr float kBandDisc = 1e-5f;      // |disc| < band * (|o'|^2 + R^2) (vertex-local o')
constexpr float kBandDir = 1e-4f;       // on |w_z|

struct RayOut { float px, py, dx, dy, dz, I; };

struct Scratch {
    int* count;   // number of listed rays
    int* list;    // indices of guard-band rays (capacity n)
};

__device__ __forceinline__ void write_out(const plt_hits& out, int64_t i, const RayOut& o) {
    out.px[i] = o.px; out.py[i] = o.py;
    out.dx[i] = o.dx; out.dy[i] = o.dy; out.dz[i] = o.dz;
    out.throughput[i] = o.I;
}

// Warp-aggregated append of guard-band rays to the float64 re-trace list (all lanes call).
__device__ __forceinline__ void list_append(const Scratch& scr, bool listed, int64_t i, int lane) {
    const unsigned m = __ballot_sync(0xffffffffu, listed);
    if (m) {
        const int leader = __ffs(m) - 1;
        int pos = 0;
        if (lane == leader) pos = atomicAdd(scr.count, __popc(m));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (listed) scr.list[pos + __popc(m & ((1u << lane) - 1u))] = (int)i;
    }
}

constexpr int kBlock = 256;

// Input direction z-component (include/plt.h): the caller's dz, or -- dz == NULL -- the
// hemisphere vector omega in S^2_+ of P:180 completed from (dx, dy), with the sign of the
// query direction (backward inputs travel towards -z before the mirroring).
__device__ __forceinline__ float load_dz(const plt_rays& in, int64_t i, float dx, float dy, int flip) {
    if (in.dz) return __ldg(in.dz + i);
    const float m = sqrtf(fmaxf(0.f, fmaf(-dx, dx, fmaf(-dy, dy, 1.f))));
    return flip ? -m : m;
}
__device__ __forceinline__ double load_dz64(const plt_rays& in, int64_t i, double dx, double dy, int flip) {
    if (in.dz) return (double)in.dz[i];
    const double m = sqrt(fmax(0.0, fma(-dx, dx, fma(-dy, dy, 1.0))));
    return flip ? -m : m;
}

struct f2 { float2 v; };
struct m2 { bool x, y; };
__device__ __forceinline__ f2 mk(float a) { return {make_float2(a, a)}; }
__device__ __forceinline__ f2 mk(float a, float b) { return {make_float2(a, b)}; }
__device__ __forceinline__ f2 operator+(f2 a, f2 b) { return {__fadd2_rn(a.v, b.v)}; }
__device__ __forceinline__ f2 operator-(f2 a, f2 b) { return {__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))}; }
__device__ __forceinline__ f2 operator-(f2 a) { return {make_float2(-a.v.x, -a.v.y)}; }
__device__ __forceinline__ f2 operator*(f2 a, f2 b) { return {__fmul2_rn(a.v, b.v)}; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return {__ffma2_rn(a.v, b.v, c.v)}; }
__device__ __forceinline__ f2 abs2(f2 a) { return {make_float2(fabsf(a.v.x), fabsf(a.v.y))}; }
__device__ __forceinline__ m2 operator&(m2 a, m2 b) { return {a.x && b.x, a.y && b.y}; }
__device__ __forceinline__ m2 operator|(m2 a, m2 b) { return {a.x || b.x, a.y || b.y}; }
__device__ __forceinline__ m2 lt(f2 a, f2 b) { return {a.v.x < b.v.x, a.v.y < b.v.y}; }
__device__ __forceinline__ m2 le(f2 a, f2 b) { return {a.v.x <= b.v.x, a.v.y <= b.v.y}; }
__device__ __forceinline__ f2 sel(m2 m, f2 a, f2 b) { return mk(m.x ? a.v.x : b.v.x, m.y ? a.v.y : b.v.y); }
__device__ __forceinline__ float rcp_approx1(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_approx1(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ f2 rcp_approx2(f2 b) { return mk(rcp_approx1(b.v.x), rcp_approx1(b.v.y)); }
__device__ __forceinline__ f2 rcp2(f2 b) {                      // Newton-refined, as Math<float>::rcp
    const f2 r = rcp_approx2(b);
    return fma2(r, fma2(-b, r, mk(1.f)), r);
}
__device__ __forceinline__ f2 sqrt2(f2 x) {                     // as Math<float>::sqrt
    x = mk(fmaxf(x.v.x, 1e-30f), fmaxf(x.v.y, 1e-30f));
    const f2 r = mk(rsqrt_approx1(x.v.x), rsqrt_approx1(x.v.y));
    const f2 s = x * r;
    return fma2(mk(0.5f) * r, fma2(-s, s, x), s);
}
__device__ __forceinline__ f2 rsqrt2(f2 x) {                    // as Math<float>::rsqrt
    const f2 r = mk(rsqrt_approx1(x.v.x), rsqrt_approx1(x.v.y));
    return r * fma2(mk(-0.5f) * x * r, r, mk(1.5f));
}
__device__ __forceinline__ bool any2(m2 m) { return m.x || m.y; }

__device__ __forceinline__ f2 glass_index2(const Step<float>& st, f2 u, f2 l2) {
#ifdef PLT_JIT   // Abbe glasses are Cauchy with C = 0: drop the (opaque) multiply by zero
    if (st.gform == kCauchyForm && st.g[2] == 0.f) return fma2(u, mk(st.g[1]), mk(st.g[0]));
#endif
    if (st.gform == kCauchyForm) return fma2(u, fma2(u, mk(st.g[2]), mk(st.g[1])), mk(st.g[0]));
    f2 s = mk(1.f);
    s = s + (mk(st.g[0]) * l2) * rcp2(l2 - mk(st.g[3]));
    s = s + (mk(st.g[1]) * l2) * rcp2(l2 - mk(st.g[4]));
    s = s + (mk(st.g[2]) * l2) * rcp2(l2 - mk(st.g[5]));
    return sqrt2(s);
}

struct Ray2 {
    f2 ox, oy, oz, wx, wy, wz, I, ncur, u, l2;
    m2 alive, near;
};

// complete: the input carries no dz (include/plt.h, A32) -- w_z = sqrt(1 - w_x^2 - w_y^2) in
// the traversal frame (towards +z after the backward mirroring), already unit length.
__device__ __forceinline__ void ray_init2(const Program<float>& P, Ray2& r, m2 alive, f2 ox, f2 oy, float plane_z,
                                          f2 wx, f2 wy, f2 wz, f2 lam_nm, bool complete) {
    if (P.flip) { wz = -wz; plane_z = P.z_mirror - plane_z; }
    r.ox = ox; r.oy = oy; r.oz = mk(plane_z);
    if (complete) {
        // w_z = sqrt(max(1 - w_x^2 - w_y^2, 1e-30)) from the MUFU rsqrt seed (~2 ulp; the fp32
        // pass takes no Newton steps)
        const f2 m = fma2(-wx, wx, fma2(-wy, wy, mk(1.f)));
        const f2 mc = mk(fmaxf(m.v.x, 1e-30f), fmaxf(m.v.y, 1e-30f));
        r.wx = wx; r.wy = wy; r.wz = mc * mk(rsqrt_approx1(mc.v.x), rsqrt_approx1(mc.v.y));
    } else {
        const f2 inv = rsqrt2(fma2(wx, wx, fma2(wy, wy, wz * wz)));
        r.wx = wx * inv; r.wy = wy * inv; r.wz = wz * inv;
    }
    const f2 lum = lam_nm * mk(1e-3f);
    r.l2 = lum * lum;
    r.u = rcp_approx2(r.l2);   // 1/lambda^2 (MUFU seed): feeds the eta polynomial / glass formulas
    r.I = mk(1.f); r.ncur = mk(1.f);
    r.alive = alive; r.near = {false, false};
}

// One step S_{L_k, sigma_k} of Eq. 5 on a ray pair (O4-O7).  `st` may be a compile-time
// constant (the JIT-specialised kernels pass literal steps: branches on kind / is_R /
// glass form and every lens constant fold away) or a __grid_constant__ program entry.
// Single-layer AR film (NEXT-4): Airy reflectance per polarisation, as the oracle.
__device__ __forceinline__ f2 coated_rf2(const Step<float>& st, f2 ncur, f2 n2, f2 cosi, f2 cost, f2 A, f2 B, f2 u,
                                         m2 tir) {
    const f2 nc = mk(st.coat_n), e1 = ncur * mk(1.f / st.coat_n);
    const f2 c2 = fma2(-(e1 * e1), fma2(-cosi, cosi, mk(1.f)), mk(1.f));
    const f2 cosc = sqrt2(c2);   // sqrt2 clamps at 1e-30 (covers c2 < 0)
    const f2 ph = (mk(st.coat_kpi) * cosc) * sqrt2(u);
    const f2 cb = mk(cospif(ph.v.x), cospif(ph.v.y));
    const f2 ncc = nc * cosc;
    const f2 as = (A - ncc) * rcp2(A + ncc), bs = (ncc - B) * rcp2(ncc + B);
    const f2 ap = fma2(nc, cosi, -(ncur * cosc)) * rcp2(fma2(nc, cosi, ncur * cosc));
    const f2 bp = fma2(n2, cosc, -(nc * cost)) * rcp2(fma2(n2, cosc, nc * cost));
    const f2 ks = (mk(2.f) * as) * (bs * cb), kp = (mk(2.f) * ap) * (bp * cb);
    const f2 Rs = (fma2(as, as, bs * bs) + ks) * rcp2(fma2(as * as, bs * bs, mk(1.f)) + ks);
    const f2 Rp = (fma2(ap, ap, bp * bp) + kp) * rcp2(fma2(ap * ap, bp * bp, mk(1.f)) + kp);
    return sel(tir, mk(1.f), mk(0.5f) * (Rs + Rp));
}

// Relative index of a step as a polynomial in the ray's wavelength variable (JIT only):
// eta(u) = n_before(u) / n_behind(u) with u = 1/lambda^2 [um^-2] is smooth over the visible
// range, so the host fits it (Chebyshev interpolation, checked to ~1 fp32 ulp over
// 380-780 nm, trace_jit.cpp) as sum_k c_k v^k in v = (u - kEtaU0) * kEtaUS in [-1, 1];
// the step then needs neither the glass formula, nor the reciprocal of n, nor the
// running index ncur -- and the Fresnel factors take their eta form (r_s = (eta c_i -
// c_t)/(eta c_i + c_t), r_p = (c_i - eta c_t)/(c_i + eta c_t), same values).
struct NoEta { static constexpr bool on = false; static constexpr int deg = 0; float c[1]; };
template <int D>
struct EtaPoly { static constexpr bool on = true; static constexpr int deg = D; float c[D + 1]; };
constexpr float kEtaU0 = 4.3f, kEtaUS = 1.f / 2.7f;   // u in [1.6, 7.0] (lambda 378-791 nm)

// kN1 (JIT only): the ray is in air before this step, so ncur == 1 exactly and the
// products with it are dropped (the packed intrinsics are opaque to constant folding).
template <bool kAsph, class PP, bool kN1 = false, class EP = NoEta>   // PP: Program<float>, or the JIT's header
// rho2o: x^2 + y^2 of the ray's origin (the previous step's hit, computed by its aperture
// test), kept by the caller across steps.
__device__ __forceinline__ void step2(const Step<float>& st, const PP& P, f2& ox, f2& oy, f2& oz,
                                      f2& wx, f2& wy, f2& wz, f2& I, f2& ncur, const f2 u, const f2 l2,
                                      m2& alive, m2& near, f2& rho2o, const EP& ep = EP{}, const f2 v = f2{}) {
    // O4 direction sanity
    near = near | (alive & lt(abs2(wz), mk(kBandDir)));
#ifdef PLT_JIT   // constant program: the sign test and the air shortcut below fold at compile time
    alive = alive & (st.sdir > 0.f ? lt(mk(0.f), wz) : lt(wz, mk(0.f)));   // w_z * sdir > 0, sdir = +-1
#else
    alive = alive & lt(mk(0.f), wz * mk(st.sdir));
#endif
    // O5 intersection
    const f2 lz = oz - mk(st.z);
    f2 t, ga = mk(0.f);
#ifdef PLT_NO_ASPH
    if (false) {
#else
    if (kAsph && st.kind == kAsphere) {
#endif
        // even asphere (NEXT-4): 6 Newton steps on F(t) = z - sag(rho) from the tangent plane
        // (both lanes, no early exit); a lane whose last step is not below the tolerance, or
        // that hits near-grazing, is flagged for the float64 re-trace
        const f2 c = mk(st.invR), k1c2 = mk((1.f + st.asph[0]) * st.invR * st.invR);
        const f2 A4 = mk(st.asph[1]), A6 = mk(st.asph[2]), A8 = mk(st.asph[3]), A10 = mk(st.asph[4]);
        const f2 B4 = mk(4.f * st.asph[1]), B6 = mk(6.f * st.asph[2]), B8 = mk(8.f * st.asph[3]),
                 B10 = mk(10.f * st.asph[4]);
        t = -lz * rcp2(wz);
        f2 dt = mk(0.f), Fp = mk(1.f);
        m2 dom{true, true};
#pragma unroll 1
        for (int it = 0; it < 6; ++it) {
            const f2 x = fma2(t, wx, ox), y = fma2(t, wy, oy), z = fma2(t, wz, lz);
            const f2 r2 = fma2(x, x, y * y);
            const f2 q = fma2(-k1c2, r2, mk(1.f));
            dom = dom & le(mk(0.f), q);
            const f2 sq = sqrt2(q);
            const f2 poly = fma2(r2, fma2(r2, fma2(r2, A10, A8), A6), A4);
            const f2 sag = fma2(c * r2, rcp2(sq + mk(1.f)), (r2 * r2) * poly);
            const f2 dpoly = fma2(r2, fma2(r2, fma2(r2, B10, B8), B6), B4);
            const f2 g = fma2(c, rcp2(sq), r2 * dpoly);
            Fp = fma2(-g, fma2(x, wx, y * wy), wz);
            dt = (z - sag) * rcp2(Fp);
            t = t - dt;
        }
        alive = alive & dom;
        const f2 tolt = mk(2e-6f) * (mk(1.f) + abs2(t));
        near = near | (alive & (lt(tolt, abs2(dt)) | lt(abs2(Fp), mk(1e-3f))));
        const f2 x = fma2(t, wx, ox), y = fma2(t, wy, oy), r2 = fma2(x, x, y * y);
        const f2 q = fma2(-k1c2, r2, mk(1.f));
        alive = alive & le(mk(0.f), q);
        ga = fma2(c, rcp2(sqrt2(q)),
                  r2 * fma2(r2, fma2(r2, fma2(r2, B10, B8), B6), B4));
    } else if (st.kind != kSphere) {
        t = -lz * rcp2(wz);
    } else {
        const f2 b = fma2(ox, wx, fma2(oy, wy, (lz - mk(st.R)) * wz));
        const f2 c = fma2(lz, lz - mk(st.twoR), rho2o);   // |o'|^2 - R^2 (vertex-local origin)
        const f2 disc = fma2(b, b, -c);
        // guard band on |disc| scaled by |o'|^2 + R^2 = c + R (2 lz + R): the float32 rounding
        // of b^2 - c is ~eps (|o'| + |R|)^2 for hits and near-tangent misses alike (a band
        // relative to b^2 alone under-covers rays whose closest approach is near their
        // origin; the band used to cover every miss instead, re-tracing ~37 % of C3's rays)
        near = near | (alive & lt(abs2(disc), fma2(lz, mk(kBandDisc * 2.f * st.R),
                                                   fma2(c, mk(kBandDisc), mk(kBandDisc * st.R * st.R)))));
#ifdef PLT_TRACE_EXPLICIT_KILLS
        alive = alive & le(mk(0.f), disc);
#endif
        // a miss (disc < 0) needs no test of its own: the root of disc is NaN there, so t is NaN
        // and the lane dies at t > eps below (comparisons with NaN are false)
        // sqrt(disc) = disc rsqrt(disc) from the MUFU seed (~2 ulp), no Newton step: C2 / C3
        // errors vs the oracle unchanged at the 2.6e-5 / 1.5e-5 mm level (tolerance 1e-4; they
        // come from the accumulated roundings, not this root).  disc < 0 or = 0: NaN -> the
        // lane dies at t > eps (disc = 0 lies inside the disc guard band: fp64 re-trace)
        const f2 rt = disc * mk(rsqrt_approx1(disc.v.x), rsqrt_approx1(disc.v.y));
        // q = -(b + copysign(rt, b)) (b = -0 takes -rt: same root pair {q, c/q} = {-+rt, +-rt}).
        // q = 0 (b = disc = 0) needs no test: t is then 0, +-inf or NaN, and the lane dies at
        // t > eps or at the aperture
        const f2 q = -(b + mk(copysignf(rt.v.x, b.v.x), copysignf(rt.v.y, b.v.y)));
        // the MUFU reciprocal without a Newton step (~1 ulp): measured position errors vs the
        // oracle 4.8e-6 -> 7.2e-6 mm (tolerance 1e-4) for 2 fewer FFMA2 per ray pair and step
        const f2 t1 = c * rcp_approx2(q);
        const bool neg_R = st.R < 0.f;
#ifdef PLT_JIT   // a live lane has sign(w_z) = sdir (O4 above), a compile-time constant here
        const bool cx = (st.sdir > 0.f) != neg_R, cy = cx;                      // pbrt cap rule (A3)
#else
        const bool cx = (wz.v.x > 0.f) != neg_R, cy = (wz.v.y > 0.f) != neg_R;   // pbrt cap rule (A3)
#endif
        t = mk(cx ? fminf(q.v.x, t1.v.x) : fmaxf(q.v.x, t1.v.x), cy ? fminf(q.v.y, t1.v.y) : fmaxf(q.v.y, t1.v.y));
    }
    alive = alive & lt(mk(kEpsT), t);
    ox = fma2(t, wx, ox); oy = fma2(t, wy, oy); oz = fma2(t, wz, oz);
    // O6 clear aperture / stop / housing
    const f2 rho2 = fma2(ox, ox, oy * oy);
    rho2o = rho2;
    near = near | (alive & lt(abs2(rho2 - mk(st.a2)), mk(st.band_a)));
    alive = alive & le(rho2, mk(st.a2));
    if (P.has_housing) {
        near = near | (alive & lt(abs2(rho2 - mk(P.housing2)), mk(P.band_h)));
        alive = alive & le(rho2, mk(P.housing2));
    }
    if (st.kind == kStop) return;
    // O7 interaction (sign of the normal folded into g, as in ray_steps)
    f2 nx, ny, nz;
    if (st.kind == kSphere) { nx = ox * mk(st.invR); ny = oy * mk(st.invR); nz = fma2(oz - mk(st.z), mk(st.invR), mk(-1.f)); }
    else if (kAsph && st.kind == kAsphere) {   // gradient of z - sag: (-g x, -g y, 1), normalised
        const f2 inv = rsqrt2(fma2(ga * ga, fma2(ox, ox, oy * oy), mk(1.f)));
        nx = -(ga * ox) * inv; ny = -(ga * oy) * inv; nz = inv;
    } else { nx = mk(0.f); ny = mk(0.f); nz = mk(1.f); }
    const f2 wn = fma2(nx, wx, fma2(ny, wy, nz * wz));
    const f2 cosi = abs2(wn);
    // air on the far side (constant n = 1): n2 = 1 and eta = ncur exactly
#ifdef PLT_JIT
    const bool air = st.gform == kCauchyForm && st.g[0] == 1.f && st.g[1] == 0.f && st.g[2] == 0.f;
#else
    constexpr bool air = false;
#endif
    f2 n2 = mk(1.f), eta;
    if constexpr (EP::on) {
        eta = mk(ep.c[EP::deg]);
#pragma unroll
        for (int k = EP::deg - 1; k >= 0; --k) eta = fma2(eta, v, mk(ep.c[k]));
    } else {
        n2 = air ? mk(1.f) : glass_index2(st, u, l2);
        eta = air ? ncur : (kN1 ? rcp2(n2) : ncur * rcp2(n2));
    }
    const f2 kappa = fma2(-(eta * eta), fma2(-cosi, cosi, mk(1.f)), mk(1.f));
    near = near | (alive & lt(abs2(kappa), mk(kBandKappa)));
    // cos(theta_t) = kappa rsqrt(kappa) from the MUFU seed, no Newton step (~2 ulp; it only
    // feeds the new direction and the Fresnel factors: direction errors 3.7e-7 -> 4.8e-7,
    // tolerance 1e-5).  kappa < 0: NaN (TIR: a T lane dies, an R lane takes R = 1);
    // kappa = 0: 0 * inf = NaN, inside the kappa guard band (re-traced in fp64).
    const f2 cost = kappa * mk(rsqrt_approx1(kappa.v.x), rsqrt_approx1(kappa.v.y));
    f2 A, B, C, D;   // r_s = (A - B)/(A + B), r_p = (C - D)/(C + D)
    if constexpr (EP::on) { A = eta * cosi; B = cost; C = cosi; D = eta * cost; }   // both divided by n_behind
    else { A = kN1 ? cosi : ncur * cosi; B = n2 * cost; C = n2 * cosi; D = kN1 ? cost : ncur * cost; }
    const f2 ApB = A + B, CpD = C + D;
    const f2 inv = rcp_approx2(ApB * CpD);
    const f2 rs = ((A - B) * CpD) * inv, rp = ((C - D) * ApB) * inv;
    const f2 Rf0 = mk(0.5f) * fma2(rs, rs, rp * rp);
    const m2 tir = lt(kappa, mk(0.f));
#ifdef PLT_NO_COAT
    const f2 Rf = st.is_R ? sel(tir, mk(1.f), Rf0) : Rf0;   // a T lane with TIR dies below: R unused
#else
    const f2 Rf = (kAsph && st.coat_n > 0.f) ? coated_rf2(st, ncur, n2, cosi, cost, A, B, u, tir)
                                             : (st.is_R ? sel(tir, mk(1.f), Rf0) : Rf0);
#endif
    if (!st.is_R) {
        // TIR on a T step absorbs (A6): cost = root of kappa < 0 is NaN, so the new
        // direction is NaN and the lane dies at the next step's direction test (or at the
        // output plane's w_z > 0) -- no test here
#ifdef PLT_TRACE_EXPLICIT_KILLS
        alive = alive & m2{!tir.x, !tir.y};
#endif
        const f2 g0 = fma2(eta, cosi, -cost);
        // g = w.n > 0 ? -g0 : g0 as a sign-bit flip (one LOP3 per lane); differs only at
        // w.n = +0 exactly (a ray exactly tangent to the surface: a measure-zero set)
        const f2 g = mk(__int_as_float(__float_as_int(g0.v.x) ^ (~__float_as_int(wn.v.x) & 0x80000000)),
                        __int_as_float(__float_as_int(g0.v.y) ^ (~__float_as_int(wn.v.y) & 0x80000000)));
        wx = fma2(eta, wx, g * nx); wy = fma2(eta, wy, g * ny); wz = fma2(eta, wz, g * nz);
        I = fma2(-I, Rf, I);
        if constexpr (!EP::on) ncur = n2;
    } else {
        const f2 two_wn = wn + wn;
        wx = fma2(-two_wn, nx, wx); wy = fma2(-two_wn, ny, wy); wz = fma2(-two_wn, nz, wz);
        I = I * Rf;
    }
}

// Steps [s0, s1) of the program (the generic, runtime-indexed path).  The warp leaves the
// loop once every lane is dead (warp-uniform; no divergent exits).
template <bool kAsph>
__device__ __forceinline__ void ray_steps2(const Program<float>& P, Ray2& r, int s0, int s1) {
    f2 ox = r.ox, oy = r.oy, oz = r.oz, wx = r.wx, wy = r.wy, wz = r.wz, I = r.I, ncur = r.ncur;
    m2 alive = r.alive, near = r.near;
    f2 rho2o = fma2(ox, ox, oy * oy);
    for (int s = s0; s < s1; ++s) {
        if (!__any_sync(0xffffffffu, any2(alive))) break;
        step2<kAsph>(P.st[s], P, ox, oy, oz, wx, wy, wz, I, ncur, r.u, r.l2, alive, near, rho2o);
    }
    r.ox = ox; r.oy = oy; r.oz = oz; r.wx = wx; r.wy = wy; r.wz = wz; r.I = I; r.ncur = ncur;
    r.alive = alive; r.near = near;
}

// Step policy of the generic kernel: phases [0, split) and [split, n_steps) of P.
template <bool kAsph>
struct GenericSteps {
    __device__ __forceinline__ static bool compact(const Program<float>& P) {
        return P.split > 0 && P.split < P.n_steps;
    }
    __device__ __forceinline__ static void run(const Program<float>& P, Ray2& r, int phase) {
        const bool c = compact(P);
        if (phase == 0) ray_steps2<kAsph>(P, r, 0, c ? P.split : P.n_steps);
        else ray_steps2<kAsph>(P, r, P.split, P.n_steps);
    }
};

// O8 for one lane of the pair (cheap; scalar keeps it simple).
__device__ __forceinline__ bool ray_finish1(const Program<float>& P, bool alive, bool& near, float ox, float oy,
                                            float oz, float wx, float wy, float wz, float I, RayOut& out) {
    near |= alive && fabsf(wz) < kBandDir;
    alive = alive && wz > 0.f;
    const float t = (P.z_out - oz) * rcp_approx1(wz);   // MUFU seed (~1 ulp), as t1 above
    alive = alive && t > 0.f;
    const float px = fmaf(t, wx, ox), py = fmaf(t, wy, oy);
    if (P.has_rect) {
        const float ex = fabsf(px - P.rect_cx) - P.rect_hw, ey = fabsf(py - P.rect_cy) - P.rect_hh;
        near |= alive && (fabsf(ex) < kBandEdge || fabsf(ey) < kBandEdge);
        alive = alive && ex <= 0.f && ey <= 0.f;
    }
    if (alive) out = RayOut{px, py, wx, wy, P.flip ? -wz : wz, I};
    else out = RayOut{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    return alive;
}

// Main pass, packed: a block owns 512 consecutive rays (thread t: rays base + t and
// base + 256 + t, so loads stay 128-byte coalesced).  Compaction after step `split` puts
// the survivors into slots 0..S-1 and thread t continues with slots 2t and 2t + 1.
template <class Steps>
__device__ __forceinline__ void trace_x2_body(const Program<float>& P, const plt_rays& in, const plt_hits& out,
                                              int64_t n, const Scratch& scr, const SplatCtx& sc) {
    constexpr int kRays = 2 * kBlock;
    __shared__ float sm_v[8][kRays];       // ox oy oz wx wy wz I ncur of the survivors
    __shared__ float sm_lam[kRays];
    __shared__ int sm_idx[kRays];
    // mask words of the tile, double-buffered when compacting: tile k's words are stored
    // after the first compaction barrier of tile k+1 (every atomicOr of tile k precedes it),
    // so warps left without survivors go on to the next tile instead of waiting at an
    // end-of-tile barrier for the warps that carry the survivors
    __shared__ unsigned sm_mask[2][kRays / 32];
    __shared__ int sm_wcnt[kBlock / 32];
    __shared__ long long sm_w[kBlock];     // fused splat: per-warp aggregation slots
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool compact = Steps::compact(P);
    const unsigned lt_mask = (1u << lane) - 1u;
    if (tid < kRays / 32) { sm_mask[0][tid] = 0u; sm_mask[1][tid] = 0u; }
    int buf = 0;
    int64_t pending = -1;                  // base of the tile whose words sit in sm_mask[buf ^ 1]
    auto flush = [&](int64_t b, unsigned* words) {   // threads < kRays/32, after a barrier
        if (b >= 0 && tid < kRays / 32) {
            if (b + 32 * tid < n) out.mask_bits[(b >> 5) + tid] = words[tid];
            words[tid] = 0u;
        }
    };
    __syncthreads();
    for (int64_t base = (int64_t)blockIdx.x * kRays; base < n; base += (int64_t)gridDim.x * kRays) {
        int64_t ix = base + tid, iy = base + kBlock + tid;
        const m2 in_range{ix < n, iy < n};
        float v[2][6] = {{0.f, 0.f, 0.f, 0.f, 1.f, 550.f}, {0.f, 0.f, 0.f, 0.f, 1.f, 550.f}};
        if (in_range.x) {
            v[0][0] = __ldg(in.ox + ix); v[0][1] = __ldg(in.oy + ix); v[0][2] = __ldg(in.dx + ix);
            v[0][3] = __ldg(in.dy + ix); v[0][5] = __ldg(in.lambda_nm + ix);
            if (in.dz) v[0][4] = __ldg(in.dz + ix);
        }
        if (in_range.y) {
            v[1][0] = __ldg(in.ox + iy); v[1][1] = __ldg(in.oy + iy); v[1][2] = __ldg(in.dx + iy);
            v[1][3] = __ldg(in.dy + iy); v[1][5] = __ldg(in.lambda_nm + iy);
            if (in.dz) v[1][4] = __ldg(in.dz + iy);
        }
        f2 lam = mk(v[0][5], v[1][5]);
        Ray2 r;
        ray_init2(P, r, in_range, mk(v[0][0], v[1][0]), mk(v[0][1], v[1][1]), in.plane_z_mm, mk(v[0][2], v[1][2]),
                  mk(v[0][3], v[1][3]), mk(v[0][4], v[1][4]), lam, in.dz == nullptr);
        Steps::run(P, r, 0);
        m2 own = in_range;
        int slot_x = tid, slot_y = kBlock + tid;   // position within the block's 512 rays
        if (compact) {
            const RayOut zero{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (in_range.x && !r.alive.x) { write_out(out, ix, zero); if (out.flags) out.flags[ix] = (uint8_t)r.near.x; }
            if (in_range.y && !r.alive.y) { write_out(out, iy, zero); if (out.flags) out.flags[iy] = (uint8_t)r.near.y; }
            list_append(scr, in_range.x && !r.alive.x && r.near.x, ix, lane);
            list_append(scr, in_range.y && !r.alive.y && r.near.y, iy, lane);
            const unsigned lx = __ballot_sync(0xffffffffu, r.alive.x), ly = __ballot_sync(0xffffffffu, r.alive.y);
            if (lane == 0) sm_wcnt[warp] = __popc(lx) + __popc(ly);
            __syncthreads();
            flush(pending, sm_mask[buf ^ 1]);   // the previous tile's words are complete
            int before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < kBlock / 32; ++w) { const int c = sm_wcnt[w]; before += w < warp ? c : 0; total += c; }
            auto put = [&](int slot, float a0, float a1, float a2, float a3, float a4, float a5, float a6, float a7,
                           float lm, int code) {
                sm_v[0][slot] = a0; sm_v[1][slot] = a1; sm_v[2][slot] = a2; sm_v[3][slot] = a3;
                sm_v[4][slot] = a4; sm_v[5][slot] = a5; sm_v[6][slot] = a6; sm_v[7][slot] = a7;
                sm_lam[slot] = lm; sm_idx[slot] = code;
            };
            if (r.alive.x)
                put(before + __popc(lx & lt_mask), r.ox.v.x, r.oy.v.x, r.oz.v.x, r.wx.v.x, r.wy.v.x, r.wz.v.x, r.I.v.x,
                    r.ncur.v.x, lam.v.x, tid | (r.near.x ? 0x10000 : 0));
            if (r.alive.y)
                put(before + __popc(lx) + __popc(ly & lt_mask), r.ox.v.y, r.oy.v.y, r.oz.v.y, r.wx.v.y, r.wy.v.y,
                    r.wz.v.y, r.I.v.y, r.ncur.v.y, lam.v.y, (kBlock + tid) | (r.near.y ? 0x10000 : 0));
            __syncthreads();
            own = m2{2 * tid < total, 2 * tid + 1 < total};
            if (own.x) {
                auto ld2 = [&](int k) { const float2 p = *reinterpret_cast<const float2*>(&sm_v[k][2 * tid]); return f2{p}; };
                r.ox = ld2(0); r.oy = ld2(1); r.oz = ld2(2); r.wx = ld2(3); r.wy = ld2(4); r.wz = ld2(5);
                r.I = ld2(6); r.ncur = ld2(7);
                const float2 lm = *reinterpret_cast<const float2*>(&sm_lam[2 * tid]);
                const int2 code = *reinterpret_cast<const int2*>(&sm_idx[2 * tid]);
                lam = f2{lm};
                if (!own.y) { lam.v.y = 550.f; r.wz.v.y = 1.f; }   // idle lane: harmless finite state
                const f2 lum = lam * mk(1e-3f);
                r.l2 = lum * lum;
                r.u = rcp_approx2(r.l2);
                r.near = m2{(code.x & 0x10000) != 0, own.y && (code.y & 0x10000) != 0};
                slot_x = code.x & 0xFFFF;
                slot_y = own.y ? (code.y & 0xFFFF) : 0;
                ix = base + slot_x;
                iy = base + slot_y;
            }
            r.alive = own;
            Steps::run(P, r, 1);
        }
        RayOut ox_, oy_;
        bool nx = r.near.x, ny = r.near.y;
        const bool vx = ray_finish1(P, r.alive.x, nx, r.ox.v.x, r.oy.v.x, r.oz.v.x, r.wx.v.x, r.wy.v.x, r.wz.v.x, r.I.v.x, ox_);
        const bool vy = ray_finish1(P, r.alive.y, ny, r.ox.v.y, r.oy.v.y, r.oz.v.y, r.wx.v.y, r.wy.v.y, r.wz.v.y, r.I.v.y, oy_);
        if (own.x) {
            write_out(out, ix, ox_);
            if (out.flags) out.flags[ix] = (uint8_t)nx;
            if (vx) atomicOr(&sm_mask[buf][slot_x >> 5], 1u << (slot_x & 31));
        }
        if (own.y) {
            write_out(out, iy, oy_);
            if (out.flags) out.flags[iy] = (uint8_t)ny;
            if (vy) atomicOr(&sm_mask[buf][slot_y >> 5], 1u << (slot_y & 31));
        }
        list_append(scr, own.x && nx, ix, lane);
        list_append(scr, own.y && ny, iy, lane);
        if (sc.film) {   // fused splat; guard-band rays are splatted by the fp64 refine instead
            const int cx = (own.x && sc.channel) ? (int)sc.channel[ix] : 0;
            const int cy = (own.y && sc.channel) ? (int)sc.channel[iy] : 0;
            splat_warp2(sc, sm_w + 32 * warp, own.x && vx && !nx, ox_.px, ox_.py, ox_.dz, ox_.I, cx,
                        own.y && vy && !ny, oy_.px, oy_.py, oy_.dz, oy_.I, cy);
        }
        if (compact) {
            pending = base;
            buf ^= 1;
        } else {
            __syncthreads();
            flush(base, sm_mask[buf]);
            __syncthreads();   // sm_* reused by the next iteration
        }
    }
    if (compact) {
        __syncthreads();
        flush(pending, sm_mask[buf ^ 1]);
    }
}

#ifndef PLT_JIT
// The generic packed kernel (runtime path program).
template <bool kAsph>
__global__ void __launch_bounds__(kBlock) trace_kernel_x2(const __grid_constant__ Program<float> P, plt_rays in,
                                                          plt_hits out, int64_t n, Scratch scr,
                                                          const __grid_constant__ SplatCtx sc) {
    trace_x2_body<GenericSteps<kAsph>>(P, in, out, n, scr, sc);
}
#endif

}  // namespace plt
