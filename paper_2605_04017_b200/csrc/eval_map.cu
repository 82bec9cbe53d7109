// eval_map.cu -- fused factorised lens-map query on 5th-generation tensor cores (sm_100a).
//
// The paper's query: {y} = f(x) if g(x) = 1 else {}, with a
// classifier g (4 -> 32 -> 32 -> 1) gating a regressor f (4 -> 32^5 -> 6), tanh
// hidden layers and linear outputs, evaluated on inputs reduced by the
// rotation/reflection symmetry of §4.1 (Eq. 10).  The paper fuses the
// MLP into its render kernels and replaces tanh by an approximation.
//
// B200 design:
//  * one persistent CTA per SM, G independent "tile pipelines" (groups of 4 warps);
//    a group owns 128 rays = one M=128 tcgen05 tile, thread t of the group = row t =
//    TMEM lane t (warp q of the group reads TMEM lanes 32q..32q+31);
//  * every layer is tcgen05.mma.cta_group::1.kind::f16 (bf16 x bf16 -> fp32) with the
//    activation tile A in shared memory and the weights B resident in shared memory
//    (TMA bulk-copied once per CTA), accumulator D in TMEM (32 columns per group);
//  * activations are carried as a bf16 hi/lo pair (A = [h_hi | h_lo], B = W for both
//    halves), so the contraction keeps ~16 mantissa bits; plain bf16 activations
//    would exceed the 2e-3 output tolerance (SURVEY [B3]);
//  * epilogue per layer: tcgen05.ld -> +bias -> tanh.approx -> split -> st.shared ->
//    fence.proxy.async -> named barrier -> one thread issues the next MMA;
//  * ray inputs for tile k+1 are staged by cp.async.bulk (TMA) while tile k runs;
//  * gating: rays with logit >= 0 are appended to a per-group queue in shared
//    memory; the regressor only runs on full 128-row tiles of queued rays (plus one
//    final partial flush), so its tensor and MUFU work scales with the valid fraction.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "plt_internal.h"

namespace plt {

namespace {

constexpr int kTile = 128;                   // rays per tile (UMMA M)
constexpr int kQueue = 256;                  // per-group queue capacity (ring of ray indices)
constexpr int kAChunks = 10;                 // A row: 4 hi + 4 lo + 2 bias-ones chunks of 8 bf16
constexpr int kARowGroupBytes = kAChunks * 128;       // SBO of the A operand
constexpr int kATileBytes = 16 * kARowGroupBytes;     // 128 rows x 80 bf16 = 20 KB
constexpr int kNumIn = 5;                    // staged SoA inputs: ox, oy, dx, dy, lambda (dz unused)
constexpr int kStageBytes = kNumIn * kTile * 4;
constexpr uint32_t kMaxImageBytes = 20480;

struct GroupSmem {
    alignas(128) uint8_t a[kATileBytes];     // activation tile (K-major, no swizzle)
    alignas(16) float stage[2][kNumIn][kTile];  // TMA-staged ray inputs
    int qi[kQueue];                          // queued valid ray indices
    int wcount[4];                           // per-warp valid counts (prefix)
};

template <int G>
struct Smem {
    alignas(128) uint8_t w[kMaxImageBytes];   // packed weights (+ folded biases)
    GroupSmem g[G];
    alignas(8) uint64_t bar_w;                // weights loaded
    alignas(8) uint64_t bar_mma[G];           // MMA complete
    alignas(8) uint64_t bar_in[G][2];         // input stage full
    uint32_t tmem_base;
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
// Bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    if (mbar_try_wait(b, phase)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(b, phase)) {
        if (clock64() - t0 > (1ll << 34)) __trap();   // ~9 s at 1.9 GHz
    }
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
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
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
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// pack (lo_elem, hi_elem) -> bf16x2 with lo_elem in the low half (lower address)
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
    return d;
}
__device__ __forceinline__ float bf16lo_f(uint32_t p) { return __uint_as_float(p << 16); }
__device__ __forceinline__ float bf16hi_f(uint32_t p) { return __uint_as_float(p & 0xFFFF0000u); }

// A-tile addressing: element (row m, k) lives at (m/8)*SBO + (k/8)*128 + (m%8)*16 + (k%8)*2.
__device__ __forceinline__ uint32_t a_row_off(int m) {
    return (uint32_t)((m >> 3) * kARowGroupBytes + (m & 7) * 16);
}

// Split 16 activations (columns c0..c0+15) into bf16 hi/lo and store them in chunks
// c0/8, c0/8+1 (hi, K 0..31) and 4+c0/8, 5+c0/8 (lo, K 32..63) of the row.
__device__ __forceinline__ void store_hidden16(uint8_t* row, int c0, const float (&h)[16]) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float x0 = h[8 * c + 2 * p], x1 = h[8 * c + 2 * p + 1];
            hi[p] = pack_bf16(x0, x1);
            lo[p] = pack_bf16(x0 - bf16lo_f(hi[p]), x1 - bf16hi_f(hi[p]));
        }
        *reinterpret_cast<uint4*>(row + (c0 / 8 + c) * 128) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(row + (4 + c0 / 8 + c) * 128) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}
// Input-layer A row: chunk 0 = x_hi[4], x_lo[4]; chunk 1 = (1, 1, 0, ...) (folded bias hi/lo).
__device__ __forceinline__ void store_input(uint8_t* row, const float (&x)[4]) {
    const uint32_t h01 = pack_bf16(x[0], x[1]), h23 = pack_bf16(x[2], x[3]);
    const uint32_t l01 = pack_bf16(x[0] - bf16lo_f(h01), x[1] - bf16hi_f(h01));
    const uint32_t l23 = pack_bf16(x[2] - bf16lo_f(h23), x[3] - bf16hi_f(h23));
    *reinterpret_cast<uint4*>(row) = make_uint4(h01, h23, l01, l23);
    *reinterpret_cast<uint4*>(row + 128) = make_uint4(0x3F803F80u, 0u, 0u, 0u);   // bf16 1.0, 1.0
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
};

// Canonicalisation of §4.1 (Eq. 10): rotate p onto +x, reflect so w'_y >= 0,
// x = (r, w'_x, w'_y, lambda) normalised to [-1, 1] (clamped).
struct Canon { float x[4]; float c, s; bool flip; };
__device__ __forceinline__ Canon canonicalise(const MapParams& mp, float px, float py, float wx, float wy, float lam) {
    Canon k;
    const float r = sqrtf(px * px + py * py);
    if (r > 0.f) { const float ir = 1.f / r; k.c = px * ir; k.s = py * ir; }
    else {
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

// Layer MMAs.  Input layer: one K=16 step (x hi/lo + bias-ones).  Hidden / output
// layers: K = 80 of A (32 hi, 32 lo, 16 bias-ones) against B = [W | W | bias chunk]
// stored once as K = 48 (the hi and lo halves of A reuse the same W columns).
__device__ __forceinline__ void issue_input(uint32_t tmem_d, uint32_t a_base, uint32_t b_base) {
    umma(tmem_d, sdesc(a_base, 128, kARowGroupBytes), sdesc(b_base, 128, 256), idesc_bf16(32), 0u);
}
__device__ __forceinline__ void issue_hidden(uint32_t tmem_d, uint32_t a_base, uint32_t b_base, int n_out) {
    const uint32_t id = idesc_bf16(n_out);
#pragma unroll
    for (int ks = 0; ks < 5; ++ks) {
        const int bk = ks < 4 ? (ks & 1) : 2;
        umma(tmem_d, sdesc(a_base + ks * 256, 128, kARowGroupBytes), sdesc(b_base + bk * 256, 128, 768), id,
             ks > 0 ? 1u : 0u);
    }
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
    GroupSmem& Gs = S.g[g];
    constexpr uint32_t kTmemCols = G <= 4 ? 128 : 256;

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
    // constant bias-ones chunks (8, 9) of every row of this group's A tile
    {
        uint8_t* row = Gs.a + a_row_off(t);
        *reinterpret_cast<uint4*>(row + 8 * 128) = make_uint4(0x3F803F80u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(row + 9 * 128) = make_uint4(0u, 0u, 0u, 0u);
        fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base + (uint32_t)(32 * g);      // this group's 32 accumulator columns
    const uint32_t tmem_row = tmem + ((uint32_t)(32 * q) << 16);   // + lane quarter
    if (tid == 0) {
        mbar_expect_tx(&S.bar_w, P.lay.total_bytes);
        tma_bulk_g2s(S.w, P.wimg, P.lay.total_bytes, &S.bar_w);
    }

    const int64_t n = P.n;
    const int64_t group_id = (int64_t)blockIdx.x * G + g;
    const int64_t group_stride = (int64_t)gridDim.x * G;
    auto tile_full_tma = [&](int64_t tile) { return P.tma_ok && (tile + 1) * kTile <= n; };
    auto issue_stage = [&](int64_t tile, int st) {   // one thread of the group
        fence_proxy_async();
        mbar_expect_tx(&S.bar_in[g][st], kStageBytes);
        const int64_t o = tile * kTile;
        tma_bulk_g2s(Gs.stage[st][0], P.in.ox + o, kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][1], P.in.oy + o, kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][2], P.in.dx + o, kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][3], P.in.dy + o, kTile * 4, &S.bar_in[g][st]);
        tma_bulk_g2s(Gs.stage[st][4], P.in.lambda_nm + o, kTile * 4, &S.bar_in[g][st]);
    };

    uint8_t* arow = Gs.a + a_row_off(t);
    const uint32_t a_base = smem_u32(Gs.a);
    const uint32_t w_base = smem_u32(S.w);
    uint32_t mma_phase = 0;
    uint32_t in_phase[2] = {0, 0};

    int64_t tile = group_id;
    if (t == 0 && tile < P.n_tiles && tile_full_tma(tile)) issue_stage(tile, 0);
    mbar_wait(&S.bar_w, 0);

    // A stored + fenced by every thread -> barrier -> one thread issues -> wait.
    auto mma_layer = [&](bool input, uint32_t b_off, int n_out) {
        tc_fence_before();
        group_bar(g);
        if (t == 0) {
            tc_fence_after();
            if (input) issue_input(tmem, a_base, w_base + b_off);
            else issue_hidden(tmem, a_base, w_base + b_off, n_out);
            umma_commit(&S.bar_mma[g]);
        }
        mbar_wait(&S.bar_mma[g], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();
    };
    // hidden epilogue: TMEM (bias already folded) -> tanh -> hi/lo -> A tile, in two halves
    auto hidden_epilogue = [&]() {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float v[16];
            tmem_ld16(tmem_row + 16 * half, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = tanh_approx(v[j]);
            store_hidden16(arow, 16 * half, v);
        }
        fence_proxy_async();
    };

    int qhead = 0, qcount = 0;
    // regressor over queue entries [qhead, qhead + rows), rows <= 128
    auto run_regressor = [&](int rows) {
        group_bar(g);   // publish queue entries written by other threads of the group
        const bool live = t < rows;
        const int qi = live ? Gs.qi[(qhead + t) & (kQueue - 1)] : 0;
        float px = 0.f, py = 0.f, wx = 0.f, wy = 0.f, lam = 550.f;
        if (live) {
            px = __ldg(P.in.ox + qi); py = __ldg(P.in.oy + qi); wx = __ldg(P.in.dx + qi);
            wy = __ldg(P.in.dy + qi); lam = __ldg(P.in.lambda_nm + qi);
        }
        const Canon k = canonicalise(P.mp, px, py, wx, wy, lam);
        store_input(arow, k.x);
        fence_proxy_async();
        mma_layer(true, P.lay.reg_w[0], 32);
        hidden_epilogue();
#pragma unroll 1
        for (int l = 1; l < 5; ++l) {
            mma_layer(false, P.lay.reg_w[l], 32);
            hidden_epilogue();
        }
        mma_layer(false, P.lay.reg_w[5], 16);
        float y[16];
        tmem_ld16(tmem_row, y);
        if (live) {
            float o[6];
#pragma unroll
            for (int d = 0; d < 6; ++d) o[d] = P.mp.out_mid[d] + P.mp.out_half[d] * y[d];
            if (k.flip) { o[1] = -o[1]; o[3] = -o[3]; }  // undo the reflection
            const float ox = k.c * o[0] - k.s * o[1], oy = k.s * o[0] + k.c * o[1];
            const float wx2 = k.c * o[2] - k.s * o[3], wy2 = k.s * o[2] + k.c * o[3], wz2 = o[4];
            const float inv = rsqrtf(wx2 * wx2 + wy2 * wy2 + wz2 * wz2);
            P.out.px[qi] = ox; P.out.py[qi] = oy;
            P.out.dx[qi] = wx2 * inv; P.out.dy[qi] = wy2 * inv; P.out.dz[qi] = wz2 * inv;
            P.out.throughput[qi] = fminf(fmaxf(o[5], 0.f), 1.f);
            if (P.raw) {
#pragma unroll
                for (int d = 0; d < 6; ++d) P.raw[(int64_t)(1 + d) * n + qi] = y[d];
            }
        }
        qhead = (qhead + rows) & (kQueue - 1);
        qcount -= rows;
    };

    for (int it = 0; tile < P.n_tiles; ++it, tile += group_stride) {
        const int st = it & 1;
        const int64_t base = tile * kTile;
        const int64_t i = base + t;
        const bool in_range = i < n;
        // next tile's inputs -> other stage (its previous contents were consumed a tile ago)
        const int64_t next = tile + group_stride;
        if (t == 0 && next < P.n_tiles && tile_full_tma(next)) issue_stage(next, st ^ 1);
        float px = 0.f, py = 0.f, wx = 0.f, wy = 0.f, lam = 550.f;
        if (tile_full_tma(tile)) {
            mbar_wait(&S.bar_in[g][st], in_phase[st]);
            in_phase[st] ^= 1u;
            px = Gs.stage[st][0][t]; py = Gs.stage[st][1][t];
            wx = Gs.stage[st][2][t]; wy = Gs.stage[st][3][t]; lam = Gs.stage[st][4][t];
        } else if (in_range) {
            px = P.in.ox[i]; py = P.in.oy[i]; wx = P.in.dx[i]; wy = P.in.dy[i]; lam = P.in.lambda_nm[i];
        }
        const Canon k = canonicalise(P.mp, px, py, wx, wy, lam);
        // ---- classifier g: 4 -> 32 -> 32 -> 1 ------------------------------
        store_input(arow, k.x);
        fence_proxy_async();
        mma_layer(true, P.lay.cls_w[0], 32);
        hidden_epilogue();
        mma_layer(false, P.lay.cls_w[1], 32);
        hidden_epilogue();
        mma_layer(false, P.lay.cls_w[2], 16);
        float lg[16];
        tmem_ld16(tmem_row, lg);
        const float logit = lg[0];
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
        // ---- gate: append valid rays to the group queue (f only on the valid set)
        if (lane == 0) Gs.wcount[q] = __popc(word);
        group_bar(g);
        int before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) { const int cw = Gs.wcount[w]; before += w < q ? cw : 0; total += cw; }
        if (valid) Gs.qi[(qhead + qcount + before + __popc(word & ((1u << lane) - 1u))) & (kQueue - 1)] = (int)i;
        qcount += total;
        if (qcount >= kTile) run_regressor(kTile);
    }
    if (qcount > 0) run_regressor(qcount);

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
                    const plt_hits& out, float* raw, int64_t n, void* stream) {
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
    static const int groups = [] {
        const char* e = getenv("PLT_MAP_GROUPS");   // tuning knob (4, 6 or 7 tile pipelines per SM)
        return e ? atoi(e) : 6;
    }();
    cudaStream_t s = (cudaStream_t)stream;
    if (groups == 4) return launch_groups<4>(P, sms, s);
    if (groups == 7) return launch_groups<7>(P, sms, s);
    return launch_groups<6>(P, sms, s);
}

}  // namespace plt
