// eval_map.cu -- fused factorised lens-map query on 5th-generation tensor cores (sm_100a).
//
// The paper's query: {y} = f(x) if g(x) = 1 else {}, with a
// classifier g (4 -> 32 -> 32 -> 1) gating a regressor f (4 -> 32^5 -> 6), tanh
// hidden layers and linear outputs, evaluated on inputs reduced by the
// rotation/reflection symmetry of §4.1 (Eq. 10).  The paper fuses the
// MLP into its render kernels and replaces tanh by an approximation.
//
// B200 design:
//  * one persistent CTA per SM, G = 8 independent "tile pipelines" (groups of 4 warps);
//    a group owns 128 rays = one M=128 tcgen05 tile, thread t of the group = row t =
//    TMEM lane t (warp q of the group reads TMEM lanes 32q..32q+31);
//  * every layer is tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32) with the
//    activation operand A in TMEM (written by tcgen05.st; 32 columns per group), the
//    weights B resident in shared memory (TMA bulk-copied once per CTA) and the
//    accumulator D in TMEM (32 columns per group) -- G x 64 of the 512 TMEM columns;
//  * activations are carried as a bf16 hi/lo pair (A = [h_hi | h_lo], B = W for both
//    halves), so the contraction keeps ~16 mantissa bits; plain bf16 activations
//    would exceed the 2e-3 output tolerance (SURVEY [B3]);
//  * biases are folded into the contraction (bf16 hi/mid/lo bias columns in B times a
//    constant ones A tile shared by all groups in shared memory); epilogue per layer:
//    tcgen05.ld -> tanh -> split -> tcgen05.st -> named barrier -> warp (g mod 4) of
//    group g issues the next layer's MMAs (the 16 most logit-influential units of the
//    classifier's first hidden layer -- ordered first at map load, map.cpp -- use an
//    accurate rational tanh instead of tanh.approx);
//    the regressor's 6-wide output layer is one more MMA round (N = 16), the classifier's
//    single output an fp32 dot product;
//  * tiles go in pairs: the ray inputs of the next pair (two 128-ray tiles) are staged by
//    cp.async.bulk (TMA) while the current pair runs; the pair claim and the staging are done
//    by warp ((g + 2) mod 4) -- single-warp duties spread over the four SM sub-partitions
//    (warp q of every group runs on sub-partition q);
//  * gating: rays with logit >= 0 are appended to a per-group queue in shared
//    memory; the regressor only runs on full 128-row tiles of queued rays (plus one
//    final partial flush), so its tensor and MUFU work scales with the valid fraction.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cstdio>

#include "plt_internal.h"
#include "splat_dev.cuh"

namespace plt {

namespace {

constexpr int kTile = 128;                   // rays per tile (UMMA M)
constexpr int kGroups = 8;                   // tile pipelines per SM (8 x 64 TMEM columns = 512)
constexpr int kQueue = 256;                  // per-group queue capacity (ring of ray indices)
constexpr int kACols = 32;                   // A operand in TMEM: 64 bf16 per row = 32 columns
                                             // (cols 0-15 hi, 16-31 lo); the bias K-step reads a
                                             // constant "ones" A tile from shared memory instead
constexpr int kOnesBytes = kTile * 16 * 2;    // 128 x 16 bf16, canonical K-major (LBO 128, SBO 256)
constexpr int kNumIn = 5;                    // staged SoA inputs: ox, oy, dx, dy, lambda (dz unused)
constexpr int kStageBytes = kNumIn * kTile * 4;
constexpr uint32_t kMaxImageBytes = 20480;

struct GroupSmem {
    alignas(16) float stage[2][kNumIn][2 * kTile];  // TMA-staged ray inputs of a tile pair
    // queue of valid rays, kept with their canonical inputs so the regressor neither
    // gathers the inputs again nor re-canonicalises them (SoA: conflict-free)
    float qx[4][kQueue];                     // normalised canonical inputs x
    float qc[kQueue], qs[kQueue];            // rotation (cos, sin) to undo
    int qi[kQueue];                          // ray index | reflection flag << 31
    int wcount[4];                           // per-warp valid counts (prefix)
    int next_tile[2];                        // dynamic scheduler: the group's next tile pair (by parity)
    long long wsum[kTile];                   // fused splat: per-warp aggregation slots
};

template <int G>
struct Smem {
    alignas(128) uint8_t w[kMaxImageBytes];   // packed weights (+ folded biases)
    alignas(128) uint8_t ones[kOnesBytes];    // A operand of every bias K-step: rows (1, 1, 1, 0, ...)
    GroupSmem g[G];
    alignas(8) uint64_t bar_w;                // weights loaded
    alignas(8) uint64_t bar_mma[G];           // MMA complete
    alignas(8) uint64_t bar_in[G][2];         // input stage full
    uint32_t tmem_base;
    int fl_head[G], fl_count[G];              // end of the tile loop: each pipeline's leftover queue
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n" : "=r"(ok) : "r"(smem_u32(b)), "r"(phase) : "memory");
    return ok != 0;
}
// (Measured alternatives: try_wait with a suspend-time hint, one polling warp per
// pipeline -- none faster.)
// Iteration-bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
// Each mbarrier.try_wait suspends the warp for up to a hardware time limit while the phase
// is incomplete, so 2^26 iterations (~1 s .. 1 min) far exceed any legitimate wait (< 1 ms); a poll iteration is ~4
// instructions (the former clock-bounded loop read the clock with 64-bit arithmetic in
// every iteration, ptxas hoisting clock64() above its k % 64 test: same speed, measured).
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    for (uint32_t k = 0; !mbar_try_wait(b, phase); ++k)
        if (k == (1u << 26)) __trap();
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(128) : "memory");
}

// Shared-memory matrix descriptor, K-major, SWIZZLE_NONE (canonical 8x16B core
// matrices): LBO = byte distance between adjacent core matrices along K, SBO =
// byte distance between adjacent 8-row groups; version field = 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// Instruction descriptor kind::f16: D f32, A/B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ float tanh_approx(float x) {   // MUFU.TANH, |error| <= 7.9e-6 (measured)
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// tanh(x) = 1 - 2 / (1 + 2^(2x log2 e)) with MUFU ex2 + rcp (~2^-22 relative each): |error|
// <~ 5e-7.  Used where a trained network amplifies activation error the most (the
// classifier's first hidden layer); saturates cleanly
// (e = inf -> 1, e = 0 -> -1).
__device__ __forceinline__ float tanh_accurate(float x) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * 2.8853900817779268f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + e));
    return fmaf(-2.f, r, 1.f);
}
// Accurate tanh for a PAIR of units on the FMA pipe with one MUFU reciprocal each:
// tanh(x) ~= x P(x^2) / Q(x^2) on |x| <= 8.5 (clamped beyond: tanh(8.5) = 1 - 8e-8), P and
// Q of degree 4 fitted by tools/fit_tanh_rational.py (float64 fit error 1.1e-8; float32
// evaluation |error| <= 3.3e-7, as accurate as ex2 + rcp).  Packed FFMA2 Horner steps serve
// both units; per pair 2 MUFU instead of 4 -- MUFU is eval_map's bound.
__device__ __forceinline__ void tanh_rational2(float& x0, float& x1) {
    constexpr float kXMax = 8.5f;
    const float2 x = make_float2(fminf(fmaxf(x0, -kXMax), kXMax), fminf(fmaxf(x1, -kXMax), kXMax));
    const float2 s = __fmul2_rn(x, x);
    auto c2 = [](float c) { return make_float2(c, c); };
    float2 P = c2(0x1.e48b04p-27f);
    P = __ffma2_rn(P, s, c2(0x1.6264eap-16f));
    P = __ffma2_rn(P, s, c2(0x1.ce26d2p-9f));
    P = __ffma2_rn(P, s, c2(0x1.128fa6p-3f));
    P = __ffma2_rn(P, s, c2(0x1.fffffep-1f));
    float2 Q = c2(0x1.b18288p-21f);
    Q = __ffma2_rn(Q, s, c2(0x1.5dcaf6p-12f));
    Q = __ffma2_rn(Q, s, c2(0x1.a9d89ap-6f));
    Q = __ffma2_rn(Q, s, c2(0x1.de9d1ap-2f));
    Q = __ffma2_rn(Q, s, c2(1.f));
    float r0, r1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(Q.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(Q.y));
    const float2 t = __fmul2_rn(__fmul2_rn(x, P), make_float2(r0, r1));
    x0 = t.x; x1 = t.y;
}
#ifndef PLT_MAP_CLS_ACCURATE_UNITS
#define PLT_MAP_CLS_ACCURATE_UNITS 16   // most logit-influential classifier h1 units with the accurate tanh
#endif
// pack (lo_elem, hi_elem) -> bf16x2 with lo_elem in the low half (lower address)
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
    return d;
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                   "r"(v[7]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// A operand in TMEM (kind::f16, M = 128): row m = lane m, element k of the row in 32-bit
// column k/2 (even k in the low half).  Hidden/output layers read K = 64 from TMEM:
// columns 0-15 hold bf16(h) (hi, round-to-nearest), 16-31 the bf16 residual h - hi (lo);
// their bias K-step takes its A operand -- rows (1, 1, 1, 0, ...) multiplying the folded
// bias hi/mid/lo columns of B -- from the shared "ones" tile in shared memory.
// hi + lo carries ~17 significant bits of h (the residual is exact in fp32 and rounded
// once); the 3-term bias is exact for an fp32 bias.
// The residuals x - hi come from the mixed-precision fma.rn.f32.bf16 (SASS FHFMA.BF16: one
// instruction per element reads the bf16 half of the packed pair directly -- no unpacking
// shift/mask), exact because |x - hi| <= 2^-9 |x| fits the fp32 mantissa of x.
__device__ __forceinline__ void resid_pair(uint32_t hi, float x0, float x1, float& r0, float& r1) {
    asm("{\n.reg .b16 h0, h1, m;\n"
        "mov.b32 {h0, h1}, %2;\n"
        "mov.b16 m, 0xBF80;\n"                       // bf16 -1.0
        "fma.rn.f32.bf16 %0, h0, m, %3;\n"
        "fma.rn.f32.bf16 %1, h1, m, %4;\n}\n"
        : "=f"(r0), "=f"(r1) : "r"(hi), "f"(x0), "f"(x1));
}
__device__ __forceinline__ uint32_t split_pair(float x0, float x1, uint32_t& lo) {
    const uint32_t hi = pack_bf16(x0, x1);
    float r0, r1;
    resid_pair(hi, x0, x1, r0, r1);   // exact
    lo = pack_bf16(r0, r1);
    return hi;
}

// Split 16 activations (D columns c0..c0+15) into hi/lo pairs and store them.
__device__ __forceinline__ void store_hidden16(uint32_t a_row, int c0, const float (&h)[16]) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) hi[p] = split_pair(h[2 * p], h[2 * p + 1], lo[p]);
    tmem_st8(a_row + c0 / 2, hi);
    tmem_st8(a_row + 16 + c0 / 2, lo);
}
// Input-layer A row (K = 16): x_hi[4], x_mid[4], x_lo[4] (an exact 3-term bf16 split of the
// fp32 inputs), then (1, 1, 1) for the folded bias hi/mid/lo, zero.  The input layer is
// where trained weights amplify a 2-term split the most.
__device__ __forceinline__ void store_input(uint32_t a_row, const float (&x)[4]) {
    uint32_t v[8];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const float x0 = x[2 * p], x1 = x[2 * p + 1];
        v[p] = pack_bf16(x0, x1);
        float r0, r1;
        resid_pair(v[p], x0, x1, r0, r1);
        v[2 + p] = split_pair(r0, r1, v[4 + p]);
    }
    v[6] = 0x3F803F80u;   // bf16 (1.0, 1.0)
    v[7] = 0x00003F80u;   // bf16 (1.0, 0)
    tmem_st8(a_row, v);
}

struct Params {
    plt_rays in;
    plt_hits out;
    float* raw;            // SoA 7*n (nullable)
    int64_t n;
    int64_t n_tiles;
    int tma_ok;            // input pointers 16-byte aligned
    MapLayout lay;
    MapParams mp;
    const uint8_t* wimg;   // device weight image
    SplatCtx sc;           // fused splat of the valid outputs (sc.film == nullptr: none)
    int* tile_ctr;         // dynamic tile scheduler: tiles handed out beyond the first G per CTA
};

// Canonicalisation of §4.1 (Eq. 10): rotate p onto +x, reflect so w'_y >= 0,
// x = (r, w'_x, w'_y, lambda) normalised to [-1, 1] (clamped).
struct Canon { float x[4]; float c, s; bool flip; };
__device__ __forceinline__ Canon canonicalise(const MapParams& mp, float px, float py, float wx, float wy, float lam) {
    Canon k;
    const float r2 = fmaf(px, px, py * py);
    float r = 0.f;
    if (r2 > 0.f) {   // MUFU rsqrt + one Newton step (~1 ulp; the oracle's tolerance is 2e-3)
        float ir;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ir) : "f"(r2));
        ir = ir * fmaf(-0.5f * r2 * ir, ir, 1.5f);
        r = r2 * ir; k.c = px * ir; k.s = py * ir;
    } else {
        const float tt = sqrtf(wx * wx + wy * wy);
        if (tt > 0.f) { k.c = wx / tt; k.s = wy / tt; } else { k.c = 1.f; k.s = 0.f; }
    }
    const float wpx = k.c * wx + k.s * wy;
    float wpy = -k.s * wx + k.c * wy;
    k.flip = wpy < 0.f;
    if (k.flip) wpy = -wpy;
    const float xin[4] = {r, wpx, wpy, lam};
#pragma unroll
    for (int d = 0; d < 4; ++d) k.x[d] = fminf(fmaxf((xin[d] - mp.in_lo[d]) * mp.in_scale[d] - 1.f, -1.f), 1.f);
    return k;
}

// Layer MMAs (A from TMEM, B = weights in shared memory), issued with their commit by a
// converged warp: elect.sync picks the issuing lane inside one asm block (the operands are
// warp-uniform, so ptxas emits no per-MMA ELECT / R2UR.BROADCAST loop).  Input layer: one
// K = 16 step (x hi/mid/lo + bias-ones).  Hidden / output layers: K = 64 of A from TMEM
// (32 hi, 32 lo) plus one K = 16 step whose A is the shared constant ones tile in shared
// memory, against B = [W | bias chunk] stored once as K = 48 (hi and lo reuse the same W).
__device__ __forceinline__ void issue_input_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                                 uint32_t bar) {
    asm volatile(
        "{\n.reg .pred p, f;\n"
        "setp.ne.b32 f, 0, 0;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, f;\n"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n}\n"
        ::"r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(bar) : "memory");
}
__device__ __forceinline__ void issue_hidden_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t b0, uint64_t b1,
                                                  uint64_t onesd, uint64_t bb, uint32_t idesc, uint32_t bar) {
    asm volatile(
        "{\n.reg .pred p, f, t;\n.reg .b32 a1, a2, a3;\n"
        "setp.ne.b32 f, 0, 0;\nsetp.eq.b32 t, 0, 0;\n"
        "add.u32 a1, %1, 8;\nadd.u32 a2, %1, 16;\nadd.u32 a3, %1, 24;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %6, f;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], %3, %6, t;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], %2, %6, t;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], %3, %6, t;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %6, t;\n"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n}\n"
        ::"r"(tmem_d), "r"(tmem_a), "l"(b0), "l"(b1), "l"(onesd), "l"(bb), "r"(idesc), "r"(bar) : "memory");
}

// Classifier: last hidden layer + fp32 output layer, h = tanh(D) from TMEM, logit = b +
// sum_j w[j] h[j], no MMA round for the single output.  The weights are kernel-parameter
// constants (constant-bank FFMA operands): no shared-memory loads through the MIO queue,
// which the tanh bursts keep full (8 LDS.128 per row before; C2 0.711 -> 0.709 ms, C3 0.492
// -> 0.491, profiles/r02_map_pair_ab.jsonl).  Even / odd j accumulate apart.
__device__ __forceinline__ void output_epilogue_cls(uint32_t tmem_row, const MapParams& mp, float& y) {
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        float v[16];
        tmem_ld16(tmem_row + 16 * half, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = tanh_approx(v[j]);
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            a0 = fmaf(mp.cls_w3[16 * half + j], v[j], a0);
            a1 = fmaf(mp.cls_w3[16 * half + j + 1], v[j + 1], a1);
        }
    }
    y = mp.cls_b3 + (a0 + a1);
}
template <int G>
__global__ void __launch_bounds__(128 * G, 1) eval_map_kernel(const __grid_constant__ Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<G>& S = *reinterpret_cast<Smem<G>*>(smem_raw);
    const int tid = threadIdx.x;
    const int g = tid >> 7;          // group
    const int t = tid & 127;         // row within the group's tile
    const int warp = tid >> 5;
    const int q = warp & 3;          // TMEM lane quarter
    const int lane = tid & 31;
    const int issue_q = g & 3;       // the pipeline's MMA-issuing warp (see mma_layer)
    GroupSmem& Gs = S.g[g];
    constexpr uint32_t kTmemCols = 512;   // 32 accumulator + 32 A columns per pipeline, G <= 8

    // ---- setup: barriers, TMEM, weights -------------------------------------------------
    if (tid == 0) {
        mbar_init(&S.bar_w, 1);
        for (int i = 0; i < G; ++i) {
            mbar_init(&S.bar_mma[i], 1);
            mbar_init(&S.bar_in[i][0], 1);
            mbar_init(&S.bar_in[i][1], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&S.tmem_base)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;                        // this warp's lane quarter
    const uint32_t tmem = S.tmem_base + (uint32_t)(32 * g);                    // accumulator (32 cols)
    const uint32_t tmem_row = tmem + lane_off;
    const uint32_t tmem_a = S.tmem_base + (uint32_t)(32 * G + kACols * g);     // A operand (32 cols)
    const uint32_t a_row = tmem_a + lane_off;
    // constant bias-ones A tile (shared by all pipelines): element (m, k) at
    // (m/8)*256 + (k/8)*128 + (m%8)*16 + (k%8)*2; k = 0, 1, 2 -> bf16 1.0 (bias hi/mid/lo)
    for (int i = tid; i < kOnesBytes / 4; i += blockDim.x) {
        const int byte = 4 * i, in_core = byte & 127, kchunk = (byte >> 7) & 1, kk = (in_core & 15) >> 1;
        uint32_t v = 0u;
        if (kchunk == 0 && kk == 0) v = 0x3F803F80u;        // k = 0, 1
        else if (kchunk == 0 && kk == 2) v = 0x00003F80u;   // k = 2
        reinterpret_cast<uint32_t*>(S.ones)[i] = v;
    }
    fence_proxy_async();   // generic-proxy writes -> visible to the tensor core (async proxy)
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&S.bar_w, P.lay.total_bytes);
        tma_bulk_g2s(S.w, P.wimg, P.lay.total_bytes, &S.bar_w);
    }

    // ray indices < 2^31 per call (checked at the ABI): 32-bit index arithmetic
    const int n = (int)P.n;
    const int n_tiles = (int)P.n_tiles;
    const int group_id = (int)blockIdx.x * G + g;
    const int group_stride = (int)gridDim.x * G;
    // tile pairs: pair p = tiles 2p, 2p + 1, staged together (5 bulk copies of 1 KB per pair
    // instead of 5 of 512 B per tile) when both tiles are full
    const int n_pairs = (n_tiles + 1) / 2;
    auto pair_full_tma = [&](int pr) { return P.tma_ok && 2 * pr + 1 < n / kTile; };
    auto issue_pair = [&](int pr, int st) {   // one thread of the group
        fence_proxy_async();
        mbar_expect_tx(&S.bar_in[g][st], 2 * kStageBytes);
        const int o = pr * 2 * kTile;
        tma_bulk_g2s(Gs.stage[st][0], P.in.ox + o, 2 * kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][1], P.in.oy + o, 2 * kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][2], P.in.dx + o, 2 * kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][3], P.in.dy + o, 2 * kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][4], P.in.lambda_nm + o, 2 * kTile * 4, &S.bar_in[g][st]);
    };

    const uint32_t w_base = smem_u32(S.w);
    const uint32_t ones_base = smem_u32(S.ones);
    uint32_t mma_phase = 0;
    uint32_t in_phase[2] = {0, 0};

    int pair = group_id, half = 0, pit = 0;
    // the per-tile duties (tile claim, input TMA) go to lane 0 of warp (g + 2) mod 4: neither
    // the MMA-issuing warp nor, for all pipelines, sub-partition 0
    const int duty_t = 32 * ((g + 2) & 3);
    if (t == duty_t && pair < n_pairs && pair_full_tma(pair)) issue_pair(pair, 0);
    mbar_wait(&S.bar_w, 0);

#ifdef PLT_MAP_PROFILE
    long long pr_bar = 0, pr_issue = 0, pr_wait = 0, pr_epi = 0, pr_ld = 0, pr_tanh = 0, pr_st = 0, pr_fence = 0;
    long long pr_layers = 0, pr_ifence = 0, pr_immas = 0, pr_icommit = 0;
    long long pr_lastbar = 0, pr_inbar = 0, pr_claim = 0, pr_top = 0;
    long long pr_tiles = 0, pr_in = 0, pr_outep = 0, pr_write = 0, pr_queue = 0, pr_reg = 0, pr_regs = 0, pr_gather = 0;
    const long long pr_t0 = clock64();
#define PLT_CLK(v) const long long v = clock64()
#else
#define PLT_CLK(v)
#endif
    // A stored + fenced by every thread -> barrier -> one thread issues -> wait.
    auto claim_pair = [&](int slot, int st) {   // one thread of the group
        const int nextp = group_stride + atomicAdd(P.tile_ctr, 1);
        Gs.next_tile[slot] = nextp;
        if (nextp < n_pairs && pair_full_tma(nextp)) issue_pair(nextp, st ^ 1);
    };
    auto mma_layer = [&](bool input, uint32_t b_off, int n_out) {
        PLT_CLK(c0);
        tc_fence_before();
        group_bar(g);
        PLT_CLK(c1);
        // one converged warp of the pipeline issues (elect.sync inside the issue asm): warp
        // (g mod 4), so the 8 pipelines' issue work is spread over the 4 SM sub-partitions
        // (warp q of every pipeline runs on sub-partition q; with warp 0 issuing for all of
        // them, sub-partition 0 ran the slowest epilogues and every pipeline waited for it)
        if (q == issue_q) {
            tc_fence_after();
            PLT_CLK(i0);
            const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0), ta = __shfl_sync(0xffffffffu, tmem_a, 0);
            const uint32_t bar = smem_u32(&S.bar_mma[g]);
            if (input) {
                issue_input_warp(tm, ta, sdesc(w_base + b_off, 128, 256), idesc_bf16(32), bar);
            } else {
                const uint32_t bb = w_base + b_off;
                issue_hidden_warp(tm, ta, sdesc(bb, 128, 768), sdesc(bb + 256, 128, 768), sdesc(ones_base, 128, 256),
                                  sdesc(bb + 512, 128, 768), idesc_bf16(n_out), bar);
            }
            PLT_CLK(i1);
#ifdef PLT_MAP_PROFILE
            const long long i2 = clock64();
            pr_ifence += i0 - c1; pr_immas += i1 - i0; pr_icommit += i2 - i1;
#endif
        }
        PLT_CLK(c2);
        mbar_wait(&S.bar_mma[g], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();
#ifdef PLT_MAP_PROFILE
        const long long c3 = clock64();
        pr_bar += c1 - c0; pr_issue += c2 - c1; pr_wait += c3 - c2; ++pr_layers; pr_lastbar = c1 - c0;
#endif
    };
    // hidden epilogue: TMEM (bias already folded) -> tanh -> hi/lo -> A operand, in two halves
    auto hidden_epilogue = [&](bool accurate) {
        PLT_CLK(e0);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            PLT_CLK(h0);
            float v[16];
            tmem_ld16(tmem_row + 16 * half, v);
            PLT_CLK(h1);
            // the classifier's h1 units are ordered by influence on the logit (map.cpp):
            // the first PLT_MAP_CLS_ACCURATE_UNITS take the accurate tanh
            if (accurate && 16 * half < PLT_MAP_CLS_ACCURATE_UNITS) {
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    if (16 * half + j + 1 < PLT_MAP_CLS_ACCURATE_UNITS) tanh_rational2(v[j], v[j + 1]);
                    else if (16 * half + j < PLT_MAP_CLS_ACCURATE_UNITS) { v[j] = tanh_accurate(v[j]); v[j + 1] = tanh_approx(v[j + 1]); }
                    else { v[j] = tanh_approx(v[j]); v[j + 1] = tanh_approx(v[j + 1]); }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = tanh_approx(v[j]);
            }
#ifdef PLT_MAP_PROFILE
            float sink = 0.f;
            for (int j = 0; j < 16; ++j) sink += v[j];
            if (sink == 12345.f) v[0] += 1.f;   // force tanh completion before the next stamp
#endif
            PLT_CLK(h2);
            store_hidden16(a_row, 16 * half, v);
            PLT_CLK(h3);
#ifdef PLT_MAP_PROFILE
            pr_ld += h1 - h0; pr_tanh += h2 - h1; pr_st += h3 - h2;
#endif
        }
        PLT_CLK(f0);
        tmem_st_wait();
#ifdef PLT_MAP_PROFILE
        const long long e1 = clock64();
        pr_fence += e1 - f0; pr_epi += e1 - e0;
#endif
    };

    int qhead = 0, qcount = 0;
    // regressor over queue entries [qhead, qhead + rows), rows <= 128; chunk >= 0: rows
    // [128 chunk, 128 chunk + rows) of the CTA's pooled leftovers (the pipelines' queues
    // concatenated in pipeline order, read in place)
    auto run_regressor = [&](int rows, int chunk) {
        if (chunk < 0) group_bar(g);   // publish queue entries written by other threads of the group
        PLT_CLK(g0);
        const bool live = t < rows;
        const GroupSmem* src = &Gs;
        int slot = (qhead + t) & (kQueue - 1);
        if (chunk >= 0 && live) {
            int e = kTile * chunk + t, p = 0;
#pragma unroll 1
            while (p < G - 1 && e >= S.fl_count[p]) e -= S.fl_count[p++];
            src = &S.g[p];
            slot = (S.fl_head[p] + e) & (kQueue - 1);
        }
        Canon k;
        int qi = 0;
        if (live) {
            const int code = src->qi[slot];
            qi = code & 0x7FFFFFFF;
            k.flip = code < 0;
#pragma unroll
            for (int d = 0; d < 4; ++d) k.x[d] = src->qx[d][slot];
            k.c = src->qc[slot]; k.s = src->qs[slot];
        } else {
#pragma unroll
            for (int d = 0; d < 4; ++d) k.x[d] = 0.f;
            k.c = 1.f; k.s = 0.f; k.flip = false;
        }
        store_input(a_row, k.x);
        tmem_st_wait();
#ifdef PLT_MAP_PROFILE
        pr_gather += clock64() - g0;
#endif
        mma_layer(true, P.lay.reg_w[0], 32);
        hidden_epilogue(false);
#pragma unroll 1
        for (int l = 1; l < 4; ++l) {
            mma_layer(false, P.lay.reg_w[l], 32);
            hidden_epilogue(false);
        }
        mma_layer(false, P.lay.reg_w[4], 32);
        float y[6];
        hidden_epilogue(false);
        // output layer (6 wide, bias folded) as one more N = 16 MMA round: measured 0.5 % faster
        // than fp32 FFMA2 dot products against weights broadcast from shared memory (96 FFMA2
        // + 48 LDS.128 per row); same hi/lo activation precision as the hidden layers
        mma_layer(false, P.lay.reg_out, 16);
        {
            float v8[8];
            tmem_ld8(tmem_row, v8);
#pragma unroll
            for (int d = 0; d < 6; ++d) y[d] = v8[d];
        }
        float o[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) o[d] = P.mp.out_mid[d] + P.mp.out_half[d] * y[d];
        if (k.flip) { o[1] = -o[1]; o[3] = -o[3]; }  // undo the reflection
        const float ox = k.c * o[0] - k.s * o[1], oy = k.s * o[0] + k.c * o[1];
        const float wx2 = k.c * o[2] - k.s * o[3], wy2 = k.s * o[2] + k.c * o[3], wz2 = o[4];
        const float inv = rsqrtf(wx2 * wx2 + wy2 * wy2 + wz2 * wz2);
        const float dz_out = wz2 * inv, I_out = fminf(fmaxf(o[5], 0.f), 1.f);
        if (live) {
            P.out.px[qi] = ox; P.out.py[qi] = oy;
            P.out.dx[qi] = wx2 * inv; P.out.dy[qi] = wy2 * inv; P.out.dz[qi] = dz_out;
            P.out.throughput[qi] = I_out;
            if (P.raw) {
#pragma unroll
                for (int d = 0; d < 6; ++d) P.raw[(int64_t)(1 + d) * n + qi] = y[d];
            }
        }
        if (P.sc.film) {   // fused splat of the valid outputs (the same floats as written above)
            const int ch = (live && P.sc.channel) ? (int)P.sc.channel[qi] : 0;
            splat_warp(P.sc, Gs.wsum + 32 * q, live, ox, oy, dz_out, I_out, ch);
        }
        if (chunk < 0) {
            qhead = (qhead + rows) & (kQueue - 1);
            qcount -= rows;
        }
    };

    // tile pairs: the first G per CTA statically (pair = group id), then dynamically -- one
    // atomicAdd per pair hands the next one to whichever pipeline is free, so pipelines whose
    // tiles held more valid rays (more regressor work) take fewer tiles and the SMs finish
    // together.  A pair's two tiles are staged by one set of five bulk copies (1 KB each): the
    // duty warp's claim + copy issue -- ~1000-1300 cycles per tile on its path to the input
    // layer's barrier, where the pipeline's other warps waited for it (in-kernel clock profile)
    // -- happens once per two tiles (C2 0.715 -> 0.710 ms, C3 0.496 -> 0.491;
    // profiles/r02_map_pair_ab.jsonl)
    for (int it = 0; pair < n_pairs; ++it) {
        const int tile = 2 * pair + half;
        const int st = pit & 1;
        const int base = tile * kTile;
        const int i = base + t;
        const bool in_range = i < n;
        PLT_CLK(ot);
        // at the first tile of a pair: claim the next pair (one global atomic per two tiles)
        // and prefetch both its tiles into the other stage; published through next_tile[pit & 1]
        if (half == 0 && t == duty_t) claim_pair(pit & 1, st);
        PLT_CLK(o0);
#ifdef PLT_MAP_PROFILE
        pr_claim += o0 - ot;
#endif
        float px = 0.f, py = 0.f, wx = 0.f, wy = 0.f, lam = 550.f;
        if (pair_full_tma(pair)) {
            if (half == 0) {
                mbar_wait(&S.bar_in[g][st], in_phase[st]);
                in_phase[st] ^= 1u;
            }
            const int e = half * kTile + t;
            px = Gs.stage[st][0][e]; py = Gs.stage[st][1][e];
            wx = Gs.stage[st][2][e]; wy = Gs.stage[st][3][e]; lam = Gs.stage[st][4][e];
        } else if (in_range) {
            px = P.in.ox[i]; py = P.in.oy[i]; wx = P.in.dx[i]; wy = P.in.dy[i]; lam = P.in.lambda_nm[i];
        }
        const Canon k = canonicalise(P.mp, px, py, wx, wy, lam);
        // ---- classifier g: 4 -> 32 -> 32 -> 1 ------------------------------
        store_input(a_row, k.x);
        tmem_st_wait();
        PLT_CLK(o1);
        mma_layer(true, P.lay.cls_w[0], 32);
#ifdef PLT_MAP_PROFILE
        pr_inbar += pr_lastbar; pr_top += o1 - ot;
#endif
        hidden_epilogue(true);
        mma_layer(false, P.lay.cls_w[1], 32);
        PLT_CLK(o2);
        float logit;
        output_epilogue_cls(tmem_row, P.mp, logit);
        PLT_CLK(o3);
        const bool valid = in_range && logit >= 0.f;     // g(x) = 1 <=> logit >= 0 (A13)
        // ---- mask word + zeros for blocked rays -----------------------------------------
        const unsigned word = __ballot_sync(0xffffffffu, valid);
        if (lane == 0 && base + 32 * q < n) P.out.mask_bits[(base >> 5) + q] = word;
        if (in_range) {
            if (P.raw) P.raw[i] = logit;
            if (!valid) {
                P.out.px[i] = 0.f; P.out.py[i] = 0.f; P.out.dx[i] = 0.f; P.out.dy[i] = 0.f;
                P.out.dz[i] = 0.f; P.out.throughput[i] = 0.f;
                if (P.raw) {
#pragma unroll
                    for (int d = 0; d < 6; ++d) P.raw[(int64_t)(1 + d) * n + i] = 0.f;
                }
            }
        }
        PLT_CLK(o4);
        // ---- gate: append valid rays to the group queue (f only on the valid set)
        if (lane == 0) Gs.wcount[q] = __popc(word);
        group_bar(g);
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) { const int cw = Gs.wcount[w]; before += w < q ? cw : 0; total += cw; }
        if (valid) {
            const int slot = (qhead + qcount + before + __popc(word & ((1u << lane) - 1u))) & (kQueue - 1);
#pragma unroll
            for (int d = 0; d < 4; ++d) Gs.qx[d][slot] = k.x[d];
            Gs.qc[slot] = k.c; Gs.qs[slot] = k.s;
            Gs.qi[slot] = (int)i | (k.flip ? (int)0x80000000u : 0);
        }
        qcount += total;
        PLT_CLK(o5);
        if (qcount >= kTile) run_regressor(kTile, -1);
#ifdef PLT_MAP_PROFILE
        const long long o6 = clock64();
        ++pr_tiles; pr_in += o1 - o0; pr_outep += o3 - o2; pr_write += o4 - o3; pr_queue += o5 - o4;
        if (o6 - o5 > 100) { pr_reg += o6 - o5; ++pr_regs; }
#endif
        // next: the pair's second tile, else the claimed pair (written at this pair's first
        // tile, before at least one group barrier)
        if (half == 0 && 2 * pair + 1 < n_tiles) {
            half = 1;
        } else {
            pair = Gs.next_tile[pit & 1];
            half = 0;
            ++pit;
        }
    }
    // Leftovers (< 128 rays per pipeline): pooled across the CTA and run as full tiles,
    // chunk c by pipeline c mod G -- one or two regressor runs per CTA instead of G partial
    // ones (per-row results do not depend on the tile a ray shares).
    if (t == 0) { S.fl_head[g] = qhead; S.fl_count[g] = qcount; }
    __syncthreads();
    int pooled = 0;
#pragma unroll
    for (int j = 0; j < G; ++j) pooled += S.fl_count[j];
    for (int c = g; kTile * c < pooled; c += G) run_regressor(min(kTile, pooled - kTile * c), c);
#ifdef PLT_MAP_PROFILE
    if (blockIdx.x == 0 && (t & 31) == 0 && g < 2) {
        printf("PROF inbar pipe %d warp %d (duty %d, issue %d): per tile claim+stage issue %lld, top->stored %lld, "
               "input-layer bar wait %lld\n", g, t >> 5, duty_t >> 5, issue_q, pr_claim / (pr_tiles ? pr_tiles : 1),
               pr_top / (pr_tiles ? pr_tiles : 1), pr_inbar / (pr_tiles ? pr_tiles : 1));
        const long long tot = clock64() - pr_t0;
        printf("PROF blk0 pipe %d t %d: total %lld layers %lld | per layer: bar %lld issue %lld wait %lld epi %lld "
               "(ld %lld tanh %lld st %lld fence %lld) | other/layer %lld | issue: fence %lld mmas %lld commit %lld\n",
               g, t, tot, pr_layers, pr_bar / pr_layers, pr_issue / pr_layers, pr_wait / pr_layers,
               pr_epi / pr_layers, pr_ld / pr_layers, pr_tanh / pr_layers, pr_st / pr_layers, pr_fence / pr_layers,
               (tot - pr_bar - pr_issue - pr_wait - pr_epi) / pr_layers, pr_ifence / pr_layers,
               pr_immas / pr_layers, pr_icommit / pr_layers);
        printf("PROF tiles pipe %d t %d: tiles %lld | per tile: stage+canon+store %lld, out-epilogue %lld, "
               "writes %lld, queue %lld | regressor runs %lld avg %lld (gather+canon %lld)\n", g, t, pr_tiles,
               pr_in / pr_tiles, pr_outep / pr_tiles, pr_write / pr_tiles, pr_queue / pr_tiles, pr_regs,
               pr_regs ? pr_reg / pr_regs : 0, pr_regs ? pr_gather / pr_regs : 0);
    }
#endif

    // ---- teardown --------------------------------------------------------------------------
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(S.tmem_base), "r"(kTmemCols));
    }
}

template <int G>
int launch_groups(const Params& P, int sms, cudaStream_t stream) {
    const size_t smem = sizeof(Smem<G>);
    static int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {   // benign race: the attribute call is idempotent
        cudaError_t e = cudaFuncSetAttribute(eval_map_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        configured = dev;
    }
    const int64_t groups_needed = (P.n_tiles + G - 1) / G;
    const int grid = (int)(groups_needed < sms ? (groups_needed < 1 ? 1 : groups_needed) : sms);
    eval_map_kernel<G><<<grid, 128 * G, smem, stream>>>(P);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_eval_map(const void* d_weights, const MapLayout& lay, const MapParams& mp, const plt_rays& in,
                    const plt_hits& out, float* raw, int64_t n, void* stream, const SplatCtx& sc) {
    if (lay.total_bytes > kMaxImageBytes) return (int)cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Params P{};
    P.in = in;
    P.out = out;
    P.raw = raw;
    P.n = n;
    P.n_tiles = (n + kTile - 1) / kTile;
    auto al = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
    P.tma_ok = al(in.ox) && al(in.oy) && al(in.dx) && al(in.dy) && al(in.lambda_nm);
    P.lay = lay;
    P.mp = mp;
    P.wimg = (const uint8_t*)d_weights;
    P.sc = sc;
    // tile counter from the library's stream-ordered pool (no host synchronisation;
    // capture-safe; freed on every exit path)
    ScratchGuard scratch(stream);
    cudaError_t e = (cudaError_t)scratch.alloc(256);
    if (e != cudaSuccess) return (int)e;
    e = cudaMemsetAsync(scratch.p, 0, 256, (cudaStream_t)stream);
    if (e != cudaSuccess) return (int)e;
    P.tile_ctr = (int*)scratch.p;
    const int rc = launch_groups<kGroups>(P, sms, (cudaStream_t)stream);
    const int fe = scratch.release();
    return rc != 0 ? rc : fe;
}

}  // namespace plt
