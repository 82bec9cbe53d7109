// plt_internal.h -- internal types shared by the host layer (lens.cpp, map.cpp, abi.cpp)
// and the sm_100a kernels (trace.cu, eval_map.cu, splat.cu).  Not part of the ABI.
#pragma once

#include <cstdint>
#include <cstddef>

#include "../../include/plt.h"

namespace plt {

// ---------------------------------------------------------------------------
// Path program: the host compiles (lens, path id, direction) into a straight
// sequence of surface steps (SURVEY.md §8(c) O2-O3 evaluated once on the host:
// which surface the ray meets next, which interaction it takes there, which way
// it travels).  The device executes the sequence; the program travels as a
// __grid_constant__ kernel parameter (read through the constant bank).
// ---------------------------------------------------------------------------
constexpr int kMaxSteps = 72;   // four-bounce paths of a 13-surface lens: <= 61 interactions + stop crossings

enum StepKind : int { kSphere = 0, kPlane = 1, kStop = 2, kAsphere = 3 };
enum GlassForm : int { kCauchyForm = 0, kSellmeier = 1 };

// Guard band of the float32 trace on geometric edges (mm); see trace.cu.
constexpr double kTraceBandEdge = 5e-4;

template <typename T>
struct Step {
    T z;        // vertex z in the traversal frame
    T R;        // signed radius (0 for planes / stop)
    T twoR;     // 2R
    T invR;     // 1/R (0 for planes)
    T a2;       // clear semi-aperture squared
    T band_a;   // 2 a kTraceBandEdge: guard band on rho^2 - a^2
    T sdir;     // expected sign of w_z when the ray meets this surface (+1 / -1)
    T g[6];     // glass on the far side: Cauchy form n = g0 + g1 u + g2 u^2 (u = 1/lambda_um^2)
                // or Sellmeier B1..B3, C1..C3 (um^2)
    int kind;   // StepKind
    int is_R;   // interaction: 0 = T (refract), 1 = R (reflect)
    int gform;  // GlassForm
    int pad;
    T asph[5];  // kAsphere: conic k, A4, A6, A8, A10 (sag in the traversal frame; c = invR)
    T coat_n;   // AR coating index (0 = bare surface)
    T coat_kpi; // 4 n_c d (um): film phase 2 beta = pi coat_kpi cos_c / lambda_um
};

template <typename T>
struct Program {
    int n_steps;
    int split;        // block-level compaction of surviving rays before this step
    int flip;         // 1 for PLT_BACKWARD: input dz and plane are mirrored, output dz negated
    int has_rect;
    int has_housing;
    int has_asph;     // any aspheric or coated step (selects the kernel instantiation with that code)
    T z_out;          // output plane in the traversal frame
    T z_mirror;       // zS for the backward frame (z' = zS - z)
    T housing;        // housing radius
    T housing2;
    T band_h;         // 2 H kTraceBandEdge
    T rect_hw, rect_hh, rect_cx, rect_cy;
    Step<T> st[kMaxSteps];
};

// ---------------------------------------------------------------------------
// Map (factorised network) device image.  Weights are pre-packed on the host
// into the tcgen05 "K-major, no swizzle" canonical layout (8-row x 16-byte core
// matrices) so the kernel can TMA-copy the whole image into shared memory.
// ---------------------------------------------------------------------------
struct MapDims {
    static constexpr int kHidden = 32;
    static constexpr int kClsLayers = 3;   // 4->32, 32->32, 32->1
    static constexpr int kRegLayers = 6;   // 4->32, 32->32 x4, 32->6
};

// Byte offsets of each packed B operand (bf16) inside the weight image.  Biases of the
// MMA layers are folded into the contraction: each operand carries an extra K chunk with
// the bf16 hi/lo split of the fp32 bias, matched by constant-one columns in A.
//   input layer : N=32, K=16 (W | W | b_hi b_lo 0..)        -> 1024 B
//   hidden layer: N=32, K=48 (W[32] | b_hi b_lo 0.. | 0..)   -> 3072 B
// The classifier's output layer (32->1) is evaluated in fp32 from the last hidden
// activations (no MMA round): its weights (bf16 values widened) and bias live in an fp32
// block at `out_off`: W[32], b, pad to 4 (eval_map reads the copy in MapParams.cls_w3 /
// cls_b3 as kernel-parameter constants).  The regressor's (32->6) is an MMA operand.
struct MapLayout {
    uint32_t cls_w[2];     // classifier input + hidden operands
    uint32_t reg_w[5];     // regressor input + 4 hidden operands
    uint32_t reg_out;      // regressor output layer as an N = 16 operand (K = 48, like a hidden layer)
    uint32_t out_off;      // byte offset of the fp32 output-layer block (16-byte aligned)
    uint32_t total_bytes;  // multiple of 16
};
constexpr int kOutClsW = 0, kOutClsB = 32, kOutFloats = 36;

struct MapParams {
    float in_lo[4], in_scale[4];   // x_hat = clamp((x - lo) * scale - 1, -1, 1), scale = 2/(hi-lo)
    float out_mid[6], out_half[6];
    float cls_w3[32], cls_b3;      // classifier output layer (also in the weight image's fp32 block)
};

// ---------------------------------------------------------------------------
// Kernel launchers (implemented in .cu files); return cudaError_t as int.
// ---------------------------------------------------------------------------
// Fused sensor splat target (film description folded into kernel constants); film ==
// nullptr means "no splat".  Device arithmetic: splat_dev.cuh.
struct SplatCtx {
    int64_t* film;                 // nullptr: no splat
    const uint8_t* channel;        // nullable: per-ray channel, indexed by ray index
    unsigned long long* dropped;   // nullable device counter
    double W, H, cx, cy;
    int width, height, channels;
    float scale;
    double wscale;                        // (double)scale * 2^32, exact (a power-of-two factor)
    float cxf, cyf, hwf, hhf, sxf, syf;   // fp32 fast-path constants
    float guard;                          // fp32 pixel-coordinate error bound (px), see make_splat_ctx
};

inline SplatCtx make_splat_ctx(const plt_film_desc& fd, int64_t* film, const uint8_t* channel, float scale,
                               unsigned long long* dropped) {
    SplatCtx c;
    c.film = film; c.channel = channel; c.dropped = dropped;
    c.W = fd.sensor_w_mm; c.H = fd.sensor_h_mm; c.cx = fd.center_x_mm; c.cy = fd.center_y_mm;
    c.width = fd.width_px; c.height = fd.height_px; c.channels = fd.channels;
    c.scale = scale;
    c.wscale = (double)scale * 4294967296.0;
    c.cxf = (float)fd.center_x_mm; c.cyf = (float)fd.center_y_mm;
    c.hwf = (float)(0.5 * c.W); c.hhf = (float)(0.5 * c.H);
    c.sxf = (float)(fd.width_px / c.W); c.syf = (float)(fd.height_px / c.H);
    // Error of the fp32 pixel coordinate (px - cxf + hwf) * sxf against the exact double
    // expression of O11, for hits inside (or near) the film: each of cxf, hwf, sxf and the
    // three roundings contributes <= 2^-24 relative to a term of magnitude <= |c| s + 2
    // width (in px), i.e. <= ((|cx| + |cy|) max(sx, sy) + 5 max(width, height)) 2^-24 with
    // headroom x2 (4.6e-4 px for the bench's 768-px film; the former fixed floor of 2e-3 px
    // sent ~4x more hits -- 13 % of the trace's splatting warps -- down the double path).
    // Hits closer than this to a pixel edge take the double path, so the film stays
    // bit-identical for any film size.
    {
        const double s = fd.width_px / c.W > fd.height_px / c.H ? fd.width_px / c.W : fd.height_px / c.H;
        const double m = fd.width_px > fd.height_px ? fd.width_px : fd.height_px;
        const double ac = (c.cx < 0 ? -c.cx : c.cx) + (c.cy < 0 ? -c.cy : c.cy);
        const double g = 2.0 * (ac * s + 5.0 * m) * 5.9604644775390625e-8;
        c.guard = (float)g;
    }
    return c;
}

#ifndef PLT_JIT
// Stream-ordered scratch from the library's own per-device pool (runtime.cpp); both
// return cudaError_t as int.  ScratchGuard frees on every exit path of a launcher.
int scratch_alloc(void** p, size_t bytes, void* stream);
int scratch_free(void* p, void* stream);
struct ScratchGuard {
    void* p = nullptr;
    void* stream = nullptr;
    explicit ScratchGuard(void* s) : stream(s) {}
    ScratchGuard(const ScratchGuard&) = delete;
    ScratchGuard& operator=(const ScratchGuard&) = delete;
    int alloc(size_t bytes) { return scratch_alloc(&p, bytes, stream); }
    int release() { const int e = scratch_free(p, stream); p = nullptr; return e; }
    ~ScratchGuard() { if (p) scratch_free(p, stream); }
};
#endif

int launch_trace_fp32(const Program<float>& pf, const Program<double>& pd, const plt_rays& in,
                      const plt_hits& out, int64_t n, void* stream, const SplatCtx& sc);
int launch_trace_fp64(const Program<double>& pd, const plt_rays& in, const plt_hits& out,
                      int64_t n, void* stream, const SplatCtx& sc);
#ifndef PLT_JIT
}  // namespace plt
#include <vector>
namespace plt {
// plt_trace_paths in float64 (trace.cu): the paths share the all-T program `pre` up to step
// depth[p] (0: traced alone); outs[p] receives path p's hits.
int launch_trace_paths_fp64(const Program<double>& pre, const std::vector<const Program<double>*>& paths,
                            const std::vector<int>& depth, const plt_rays& in, const plt_hits* outs, int64_t n,
                            void* stream, const SplatCtx& sc);
#endif
// Run-time specialised packed trace kernel for P (trace_jit.cpp): cudaKernel_t or nullptr.
void* trace_jit_kernel(const Program<float>& P);
// plt_kernel_kind of the float32 kernel that runs P (trace.cu); *jit receives the JIT kernel.
int trace_fp32_kind(const Program<float>& P, void** jit);
#ifndef PLT_JIT
}  // namespace plt
#include <string>
namespace plt {
// The specialised kernel's cubin compiled without a GPU ("" on failure; log in *log_out).
std::string trace_jit_cubin(const Program<float>& P, std::string* log_out);
#endif
struct ScenePlane { double z, period, contrast; };
int launch_shade_plane(const ScenePlane& sc, double z_hits, const plt_hits& hits, int spp, int64_t pixels,
                       float scale, int64_t* film, int64_t n, void* stream, const float* in_dz = nullptr);
constexpr int kMaxCards = 8;
struct SceneCards {
    int n;
    double background;
    double z[kMaxCards], period[kMaxCards], contrast[kMaxCards];
    double x0[kMaxCards], x1[kMaxCards], y0[kMaxCards], y1[kMaxCards];
};
int launch_shade_cards(const SceneCards& sc, double z_hits, const plt_hits& hits, int spp, int64_t pixels,
                       float scale, int64_t* film, int64_t n, void* stream, const float* in_dz);
int launch_propagate(const plt_rays& in, const plt_rays& out, float z_target, float sdir, int64_t n, void* stream);
int launch_splat(const plt_film_desc& fd, int64_t* film, const plt_hits& hits, const uint8_t* channel,
                 float scale, int64_t n, unsigned long long* dropped, void* stream);
int launch_gen_rays(const plt_ray_law& law, uint64_t seed, int64_t start, const plt_rays& out, int64_t n,
                    void* stream);
int launch_resolve(const plt_film_desc& fd, const int64_t* film, float* out, double scale, void* stream);
int launch_eval_map(const void* d_weights, const MapLayout& lay, const MapParams& mp,
                    const plt_rays& in, const plt_hits& out, float* raw, int64_t n, void* stream,
                    const SplatCtx& sc);

}  // namespace plt
