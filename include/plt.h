/*
 * plt.h -- C ABI of libplt.so, the B200 (sm_100a) precomputed-lens-transport query library.
 *
 * The library answers the batched per-ray lens transport query of
 * "Precomputed Lens Transport Maps" (arxiv 2605.04017): for each incident ray
 * (position on an input plane, direction, wavelength) it returns an occlusion
 * mask, the exit ray (position on the output plane, direction) and the Fresnel
 * throughput, either by the exact sequential trace (plt_trace_rays) or by the
 * factorised classifier/regressor network (plt_eval_map).
 *
 * Citations: P:n = PAPER.md line n (the paper text); S:n = SPEC.md line n;
 * SURVEY.md §8(b)/(c) readings A1..A30 are restated in DESIGN.md.
 *
 * Conventions (all functions):
 *  - Return plt_status; 0 = PLT_OK.  Never throw, never exit, never print.
 *    On error, plt_last_error() returns a thread-local message valid until the
 *    next plt_* call on the same thread.
 *  - Units: millimetres and nanometres; +z runs from object side to image side;
 *    surfaces are listed front to back with the first vertex at z = 0.
 *  - Ray / hit / film buffers are DEVICE pointers owned by the caller (e.g.
 *    torch.Tensor.data_ptr()); every float array must be 4-byte aligned and
 *    hold n elements; mask_bits holds ceil(n/32) uint32 words.
 *  - Asynchronous: compute calls enqueue on `cuda_stream` (a cudaStream_t;
 *    NULL = legacy default stream) on the CALLER's current device and return.
 *    Argument errors are reported synchronously; CUDA launch errors are
 *    reported as PLT_E_CUDA; faults inside kernels surface on a later call.
 *  - Absence is not an error: a blocked ray gets mask bit 0
 *    and all-zero outputs.  NaN is never used as a sentinel.
 *  - Mask bit convention: bit (i mod 32) of word i/32 is 1 <=> ray i is valid.
 *    (This is Listing 1's `is_blocked` with the polarity reversed; A13.)
 *  - Handles (plt_lens, plt_map) are immutable after creation and may be used
 *    concurrently from several threads/streams/devices.
 *  - There is no CPU fallback: every compute entry point requires an sm_100a
 *    device and returns PLT_E_CUDA otherwise.
 */
#ifndef PLT_H_
#define PLT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PLT_API __attribute__((visibility("default")))
#else
#define PLT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PLT_OK = 0,
    PLT_E_INVALID_ARG = 1,  /* null / misaligned pointer, n < 0, bad enum, unknown path id     */
    PLT_E_PARSE = 2,        /* prescription or map blob cannot be parsed (message: line/field) */
    PLT_E_VALIDATION = 3,   /* parsed but violates an invariant (message names it)             */
    PLT_E_CAPACITY = 4,     /* output array too small (two-call pattern, see enumerate_ghosts) */
    PLT_E_UNSUPPORTED = 5,  /* valid request the library does not implement                    */
    PLT_E_CUDA = 6,         /* CUDA runtime error, or no sm_100a device                        */
    PLT_E_OOM = 7           /* host or device allocation failed                                */
} plt_status;

/* Thread-local message for the last failing call on this thread ("" if none). */
PLT_API const char* plt_last_error(void);

/* Library version string, e.g. "plt 0.1 sm_100a". */
PLT_API const char* plt_version(void);

typedef struct plt_lens plt_lens; /* opaque: parsed prescription + compiled path programs */
typedef struct plt_map plt_map;   /* opaque: one path's factorised network (bf16 weights)  */

typedef enum {
    PLT_FORWARD = 0,  /* object side -> sensor: input plane in front, output plane = sensor */
    PLT_BACKWARD = 1  /* sensor -> object side: rays start on the sensor (A9 separate maps) */
} plt_dir;

typedef enum {
    PLT_FP32 = 0,  /* float32 trace + float64 re-trace of rays within a guard band of any edge */
    PLT_FP64 = 1   /* whole trace in float64 (binding precision for ghost paths)    */
} plt_precision;

/* Lens options that are not part of the prescription. */
typedef struct {
    double input_plane_z_mm;   /* forward input plane z (informational; rays carry their own plane_z)     */
    double sensor_z_mm;        /* forward output plane; NaN -> paraxial focus at lambda_ref_nm (ABCD)      */
    double sensor_w_mm;        /* sensor rectangle ("CMOS sized rectangle"); 0 -> unbounded plane    */
    double sensor_h_mm;
    double backward_exit_z_mm; /* output plane for PLT_BACKWARD, in front of the first vertex (e.g. -5)    */
    double housing_radius_mm;  /* barrel cylinder radius ("housing"); 0 -> clear apertures only     */
    double lambda_ref_nm;      /* reference wavelength for the paraxial focus and ghost pruning (587.5618) */
} plt_lens_opts;

/*
 * Parse and validate a lens prescription ("lens configurations are provided
 * as JSON"; format in DESIGN.md): either the line-oriented table
 *     name <id>
 *     <radius_mm> <thickness_mm> <glass> <aperture_diameter_mm>
 * (glass = air | stop | n:<n> | abbe:<nd>,<Vd> | cauchy:<A>,<B>,<C> |
 *  sellmeier:<B1>,<B2>,<B3>,<C1>,<C2>,<C3>, or a bare Kolb n_d [V_d]) or a JSON
 * object {"name":..,"surfaces":[{"radius_mm","thickness_mm","glass","semi_aperture_mm"}]}.
 * text need not be NUL-terminated.  opts may be NULL (defaults above, sensor at focus).
 * Errors: PLT_E_PARSE (line/field in message), PLT_E_VALIDATION (invariant named:
 * more than one stop, non-positive aperture, negative thickness, |R| < aperture,
 * index < 1 in [380,780] nm, no optical surface), PLT_E_OOM.
 * Ownership: *out is owned by the caller and released with plt_lens_free.
 */
PLT_API plt_status plt_lens_load(const char* text, size_t len, const plt_lens_opts* opts, plt_lens** out);
PLT_API void plt_lens_free(plt_lens* lens);

/*
 * Paraxial summary at lambda_nm (ABCD matrices).
 * abcd = {A, B, C, D} from the first to the last vertex (ray vector (h, u), u = slope);
 * efl = -1/C, bfl = -A/C (from the last vertex).  Any output pointer may be NULL.
 * Errors: PLT_E_INVALID_ARG (lambda outside [380, 780] nm).
 */
PLT_API plt_status plt_lens_info(const plt_lens* lens, double lambda_nm, int* n_optical, int* stop_index,
                         double abcd[4], double* efl_mm, double* bfl_mm, double* sensor_z_mm);

/*
 * Paraxial entrance / exit pupils at lambda_nm (lens frame, mm): the aperture stop imaged
 * through the surfaces in front of it / behind it (backward camera
 * rays aimed at the exit pupil instead of the rear clear aperture waste fewer samples).
 * Errors: PLT_E_INVALID_ARG (null), PLT_E_VALIDATION (no stop).
 */
PLT_API plt_status plt_lens_pupils(const plt_lens* lens, double lambda_nm, double* entrance_z_mm,
                                   double* entrance_r_mm, double* exit_z_mm, double* exit_r_mm);

/*
 * Path ids ("Each sequence can be converted to a binary number"):
 * id = 2^K + sum_k 2^(k-1) [interaction k is R], the stop is not an interaction.
 * The all-transmission path of an m-surface lens is 2^m; the two-bounce ghost that
 * reflects at optical surface i and then j (1 <= j < i <= m) is
 * 2^(m+2(i-j)) + 2^(i-1) + 2^(2i-j-1)  (e.g. 65616 = ghost (5,3) of a 12-surface lens).
 *
 * plt_enumerate_ghosts lists the all-T path followed by every two-bounce ghost
 * ("contributions from higher-order paths ... are negligible"), ascending
 * by id.  max_bounces: 0 (all-T only), 2, or 4: adds the four-bounce paths that
 * reflect at i, then j < i, then k > j, then l < k (ids with
 * K > 63 interactions are skipped).  min_throughput > 0 drops paths whose
 * normal-incidence throughput (product of R at the reflections and T elsewhere) at
 * lambda_ref is below it.  ij_pairs (nullable) receives the first reflection pair
 * (i, j) per id ((0,0) for all-T).
 * Two-call pattern: with ids == NULL or capacity < count, *count is set and
 * PLT_E_CAPACITY is returned.
 */
PLT_API plt_status plt_enumerate_ghosts(const plt_lens* lens, int max_bounces, double min_throughput,
                                uint64_t* ids, int32_t* ij_pairs, int capacity, int* count);

/* Device SoA input rays: origin (ox, oy, plane_z) in the lens frame, direction
 * (dx, dy, dz) (unit; dz > 0 for PLT_FORWARD, dz < 0 for PLT_BACKWARD), wavelength
 * in nm (caller precondition: 380..780; not checked per ray -- the run-time
 * specialised fp32 trace evaluates each surface's relative index as a polynomial fitted
 * on 378..791 nm and sends rays outside that range to its exact float64 re-trace).
 * dz may be NULL: the direction is then the hemisphere vector omega in S^2_+ of P:180
 * given by its (x, y) components, |dz| = sqrt(max(0, 1 - dx^2 - dy^2)) with the sign of
 * the query direction (+ forward, - backward), completed per ray in the kernel's own
 * precision (fp32 passes in fp32, float64 passes and the guard-band re-trace in fp64).
 * A caller holding unit directions then moves 20 instead of 24 bytes per ray. */
typedef struct {
    const float* ox;
    const float* oy;
    const float* dx;
    const float* dy;
    const float* dz;
    const float* lambda_nm;
    double plane_z_mm;
} plt_rays;

/* Device SoA outputs (all written for every ray; zeros where invalid). */
typedef struct {
    uint32_t* mask_bits;  /* ceil(n/32) words, bit set <=> valid                          */
    float* px;            /* exit position on the output plane                            */
    float* py;
    float* dx;            /* exit direction (unit)                                        */
    float* dy;
    float* dz;
    float* throughput;    /* Fresnel throughput I_out                      */
    uint8_t* flags;       /* nullable; trace: bit0 = re-traced in fp64 (guard band)       */
} plt_hits;

/*
 * Exact sequential trace T^P = S_K o ... o S_1 of path `path_id` (Eq. 5-7):
 * per surface, closest hit on the spherical/planar cap (positional operator p_sigma),
 * clear-aperture/stop/housing test, Snell refraction or mirror reflection
 * (directional operator d_{L,sigma}), unpolarised Fresnel R/T with Sellmeier/Abbe/
 * Cauchy dispersion (f_{L,sigma}); valid iff sigma_{K+1} is the output plane
 * and, for PLT_FORWARD with a sensor rectangle, the hit lies inside it.
 * Errors: PLT_E_INVALID_ARG (null pointers, n < 0, n >= 2^31, path id inconsistent
 * with the lens, a path program of more than 72 surface steps), PLT_E_CUDA.  n == 0 is
 * a no-op.  Which kernel runs a PLT_FP32 trace (run-time specialised, generic packed,
 * scalar) is reported by plt_trace_kernel; their outputs agree with the oracle within the
 * same tolerances but not bit for bit.
 */
PLT_API plt_status plt_trace_rays(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                          const plt_rays* in, const plt_hits* out, int64_t n, void* cuda_stream);

/*
 * Load one path's factorised map: a binary valid-mask classifier
 * g: 4 -> 32 -> 32 -> 1 and a regressor f: 4 -> 32^5 -> 6, tanh hidden layers,
 * linear outputs.  Blob layout (little-endian): magic
 * "PLTMAP01", u32 version (1 or 2), u32 direction, u64 path_id, u32 n_cls_layers=3,
 * u32 n_reg_layers=6, [version 2: f64 plane_z_mm, the input plane the map was trained
 * on], f32 in_lo[4], in_hi[4], out_mid[6], out_half[6], then per layer u32 out, u32 in,
 * bf16 W[out][in], f32 b[out].  `lens` may be NULL (no cross-check); otherwise the
 * blob's path id must be consistent with the lens.  plt_eval_map rejects rays whose
 * plane_z_mm differs from a version-2 map's plane (PLT_E_INVALID_ARG).
 * Errors: PLT_E_PARSE (truncated / bad magic), PLT_E_VALIDATION (dimensions), PLT_E_OOM.
 */
PLT_API plt_status plt_map_load(const plt_lens* lens, const void* blob, size_t len, plt_map** out);
PLT_API void plt_map_free(plt_map* map);

/*
 * Factorised query {y} = f(x) if g(x) = 1 else {} for n rays:
 * canonicalise by the rotation/reflection symmetry of §4.1 (Eq. 10) to
 * x = (r, w'_x, w'_y >= 0, lambda), normalise to [-1,1], run the classifier; rays
 * with logit >= 0 are valid and only those run the regressor (gating);
 * outputs are de-normalised, un-reflected, rotated back, direction renormalised,
 * throughput clamped to [0,1].  One fused sm_100a kernel: tcgen05.mma tiles with
 * TMEM accumulators, weights resident in shared memory, inputs staged by TMA bulk copies.
 * raw_out (nullable, device, 7*n floats, SoA: raw_out[k*n + i] with k = 0 the
 * classifier logit and k = 1..6 the regressor outputs y before de-normalisation,
 * y = 0 for invalid rays) exposes the network outputs for parity.
 * Errors: PLT_E_INVALID_ARG (also: in->plane_z_mm is not the plane a version-2 map was
 * trained on), PLT_E_CUDA.
 */
PLT_API plt_status plt_eval_map(const plt_map* map, const plt_rays* in, const plt_hits* out,
                        float* raw_out, int64_t n, void* cuda_stream);

/* Film description for sensor splatting (Eq. 8).  All sizes > 0 and
 * channels * height_px * width_px < 2^31 (PLT_E_INVALID_ARG otherwise). */
typedef struct {
    int width_px, height_px, channels;
    double sensor_w_mm, sensor_h_mm, center_x_mm, center_y_mm;
} plt_film_desc;

/*
 * Splat valid hits into an int64 fixed-point film (Eq. 8; Listing 1):
 * ix = floor((px - cx + W/2)/W * width), iy = floor((H/2 - (py - cy))/H * height)
 * (row 0 at +y); film[c][iy][ix] += llrint(I * |dz| * weight_scale * 2^32), computed in
 * IEEE double so the sum is exact and order independent.  Hits outside the film are
 * dropped and counted in *dropped (device counter, nullable, incremented atomically).
 * channel (nullable, device, n bytes) selects c (NULL -> 0); channels outside the
 * film are dropped.  Warp-aggregated atomics (one atom.add per distinct pixel per warp).
 * film: device, caller-owned, channels*height*width int64, NOT cleared by this call.
 * Errors: PLT_E_INVALID_ARG, PLT_E_CUDA.
 */
PLT_API plt_status plt_splat_sensor(const plt_film_desc* film_desc, int64_t* film, const plt_hits* hits,
                            const uint8_t* channel, float weight_scale, int64_t n,
                            unsigned long long* dropped, void* cuda_stream);

/*
 * Fused query + splat.  plt_trace_rays_splat / plt_eval_map_splat compute exactly what
 * plt_trace_rays / plt_eval_map compute (same hits written to `out`) AND splat every valid
 * hit into splat->film inside the same kernels (the epilogue of the trace / of the
 * regressor), with the arithmetic of plt_splat_sensor: the film is bit-identical to
 * calling the query and then plt_splat_sensor on its hits, without re-reading the hits
 * or a separate launch.  splat->channel (nullable, device, n bytes) is indexed like the
 * rays.  For PLT_FP32 traces, rays inside a guard band are splatted after their float64
 * re-trace.  Errors: as the query, plus PLT_E_INVALID_ARG for a bad film description.
 */
typedef struct {
    const plt_film_desc* film_desc;
    int64_t* film;                  /* device, caller-owned, NOT cleared */
    const uint8_t* channel;         /* nullable, device, n bytes */
    float weight_scale;
    unsigned long long* dropped;    /* nullable device counter */
} plt_splat_target;

PLT_API plt_status plt_trace_rays_splat(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                                        const plt_rays* in, const plt_hits* out, const plt_splat_target* splat,
                                        int64_t n, void* cuda_stream);
PLT_API plt_status plt_eval_map_splat(const plt_map* map, const plt_rays* in, const plt_hits* out, float* raw_out,
                                      const plt_splat_target* splat, int64_t n, void* cuda_stream);

/*
 * Trace one ray batch along several paths of the same lens and direction -- the flare
 * image's per-path forward loop (Listing 1: every ghost path traced from the
 * same input rays).  Results are exactly those of one plt_trace_rays call per path
 * (plt_trace_rays_splat when splat != NULL: every path splats into the one film), in
 * order, on cuda_stream: path p's hits go to outs[p].
 * PLT_FP64 shares the work the paths have in common: a path's steps before its first
 * reflection are the all-T path's first steps (the same surfaces, interactions and
 * media), so the batch is traced ONCE along the all-T program, the float64 state of the
 * rays still alive before each path's first reflection is kept in device scratch, and each
 * path resumes from its depth.  The state is the one the single-path kernel carries, so
 * hits, masks and film are bit-identical to the per-path calls (a path whose prefix
 * program differs, or the all-T path itself, is traced alone).  Scratch: 68 B per ray per
 * distinct first-reflection depth (batches beyond 2 GiB of it run in chunks).  PLT_FP32
 * traces each path with plt_trace_rays.
 * path_ids: host, n_paths ids; outs: host array of n_paths plt_hits (device pointers).
 * Errors: as plt_trace_rays for any path (ids validated before any device work), plus
 * PLT_E_INVALID_ARG for n_paths < 0 or null path_ids / outs; n == 0 or n_paths == 0 is a
 * no-op.
 */
PLT_API plt_status plt_trace_paths(const plt_lens* lens, const uint64_t* path_ids, int n_paths, plt_dir dir,
                                   plt_precision prec, const plt_rays* in, const plt_hits* outs,
                                   const plt_splat_target* splat, int64_t n, void* cuda_stream);

/*
 * Inspection: the sm_100a cubin of the float32 trace kernel specialised for this path
 * program (the kernel plt_trace_rays launches for large batches; compiled with NVRTC, no
 * GPU needed).  Two-call pattern: *size receives the cubin size; the bytes are written
 * when buf != NULL and capacity >= size.  Errors: PLT_E_UNSUPPORTED (NVRTC unavailable),
 * PLT_E_VALIDATION (compilation failed; plt_last_error holds the log), PLT_E_CAPACITY.
 */
PLT_API plt_status plt_trace_jit_cubin(const plt_lens* lens, uint64_t path_id, plt_dir dir, void* buf,
                                       size_t capacity, size_t* size);

/*
 * Which kernel plt_trace_rays launches for (lens, path_id, dir, prec) in this process:
 * PLT_KERNEL_JIT -- the float32 kernel specialised at run time for the path program
 * (NVRTC, all-transmission paths; compiled and cached by this call if needed);
 * PLT_KERNEL_PACKED -- the generic packed float32 kernel (ghost paths, or all-T paths when
 * NVRTC is unavailable); PLT_KERNEL_SCALAR -- the one-ray-per-thread float32 kernel
 * (developer switch PLT_TRACE_X1); PLT_KERNEL_FP64 -- PLT_FP64 traces.  All are within the
 * parity tolerances of the oracle, but their float32 results differ in the last bits, so a
 * caller that needs reproducibility across hosts checks this.
 * Errors: PLT_E_INVALID_ARG (null, bad enum, path id inconsistent with the lens), PLT_E_CUDA.
 */
typedef enum {
    PLT_KERNEL_JIT = 0,
    PLT_KERNEL_PACKED = 1,
    PLT_KERNEL_SCALAR = 2,
    PLT_KERNEL_FP64 = 3
} plt_kernel_kind;

PLT_API plt_status plt_trace_kernel(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                                    plt_kernel_kind* kind);

/*
 * Backward camera integrand with a procedural scene (Eq. 9,
 * P:259-269; the depth-of-field integrator).  For every valid hit of a
 * PLT_BACKWARD query (exit origin on the plane z = z_hits_mm in the lens frame, direction
 * towards -z) the ray continues in air to the scene plane z = scene->z_mm (t = (z_s -
 * z_hits)/w_z > 0 required); the scene radiance is a checkerboard of period `period_mm`:
 * L = 1 where floor(x/period) + floor(y/period) is even, `contrast` where it is odd.
 * film[i / spp] += llrint(I * L * weight_scale * 2^32) for ray i (pixel-stratified rays,
 * e.g. the sensor_grid law), skipping pixels >= `pixels`; IEEE double, exact int64 sum.
 * film: device, caller-owned, `pixels` int64, NOT cleared.  Errors: PLT_E_INVALID_ARG, PLT_E_CUDA.
 */
typedef struct {
    double z_mm;        /* scene plane (lens frame, object side: below the front vertex) */
    double period_mm;   /* checker square size, > 0 */
    double contrast;    /* radiance of the odd squares (even squares: 1) */
} plt_scene_plane;

PLT_API plt_status plt_shade_plane(const plt_scene_plane* scene, double z_hits_mm, const plt_hits* hits, int spp,
                                   int64_t pixels, float weight_scale, int64_t* film, int64_t n, void* cuda_stream);

/*
 * plt_shade_plane with the Monte-Carlo weight of pupil sampling (SURVEY.md §8(f) NEXT-3
 * remainder).  Eq. 9 integrates L T cos(theta) over the hemisphere at the sensor point;
 * when ray i's direction was drawn through a uniform point on a disc of area A parallel
 * to the sensor at axial distance dz (an exit pupil, or the rear clear aperture), its
 * solid-angle pdf is dz^2 / (A cos^3 theta), so the estimator weight is
 * (A / dz^2) cos^4 theta.  in_dz (device, n floats) holds the z-components w_z of the
 * SENSOR rays (cos theta = |w_z|); the caller folds A / dz^2 (and 1/spp) into
 * weight_scale: film[i / spp] += llrint(I * L * ((w_z^2)^2) * weight_scale * 2^32),
 * IEEE double in that order (bit-identical to oracle.shade_plane with in_dz).
 * Errors: PLT_E_INVALID_ARG (also in_dz == NULL), PLT_E_CUDA.
 */
/*
 * The pupil-sampling factor A / dz^2 of plt_shade_plane_weighted for directions drawn through
 * a uniform point of a disc of radius disc_r_mm at z = disc_z_mm, seen from a sensor at
 * z = sensor_z_mm: *weight = pi disc_r^2 / (sensor_z - disc_z)^2 (the caller multiplies its
 * own 1/spp into it).  Errors: PLT_E_INVALID_ARG (null, non-finite, r <= 0, disc on the sensor).
 */
PLT_API plt_status plt_pupil_weight(double sensor_z_mm, double disc_z_mm, double disc_r_mm, double* weight);

PLT_API plt_status plt_shade_plane_weighted(const plt_scene_plane* scene, double z_hits_mm, const plt_hits* hits,
                                            int spp, int64_t pixels, float weight_scale, const float* in_dz,
                                            int64_t* film, int64_t n, void* cuda_stream);

/*
 * Scene of several checkerboard cards at different depths (scenes
 * beyond one plane -- a depth-of-field target whose cards come into focus at different
 * sensor shifts).  Card k: plane z = z_mm (object side), axis-aligned rectangle
 * [x0_mm, x1_mm] x [y0_mm, y1_mm], checker period and odd-square contrast as
 * plt_scene_plane.  A valid backward exit ray takes the radiance of the card it meets
 * first -- smallest t = (z_k - z_hits)/w_z > 0 whose hit point lies inside the rectangle
 * (ties: lower k) -- or `background` if it meets none.  Weighting as
 * plt_shade_plane_weighted when in_dz != NULL, else as plt_shade_plane.  IEEE double,
 * exact int64 sum (bit-identical to oracle.shade_cards).  1 <= n_cards <= 8.
 * Errors: PLT_E_INVALID_ARG, PLT_E_CUDA.
 */
typedef struct {
    double z_mm, period_mm, contrast;
    double x0_mm, x1_mm, y0_mm, y1_mm;
} plt_scene_card;

PLT_API plt_status plt_shade_cards(const plt_scene_card* cards, int n_cards, double background, double z_hits_mm,
                                   const plt_hits* hits, int spp, int64_t pixels, float weight_scale,
                                   const float* in_dz, int64_t* film, int64_t n, void* cuda_stream);

/*
 * Free-space propagation to the plane z = z_target_mm (sensor-shift focusing with one
 * precomputed map): o' = o + ((z_t - z_in)/w_z) w in float32 (round-to-nearest,
 * one fma per coordinate), w and lambda copied.  in->plane_z_mm is z_in; out's arrays
 * (device, n each, may alias in's) receive the rays; out->plane_z_mm is not used.
 * The ray moves along its own line, forwards or backwards (t may be negative: a sensor
 * shifted past the map's input plane).  in->dz NULL: w_z = sign * sqrt(max(0, 1 - w_x^2 -
 * w_y^2)) with the sign of the query direction `dir` (+ for PLT_FORWARD, - for
 * PLT_BACKWARD) -- the same rule as plt_trace_rays -- and out->dz may then be NULL
 * too (the output stays in the (dx, dy) parameterisation).
 * Errors: PLT_E_INVALID_ARG (also a bad dir), PLT_E_CUDA.
 */
PLT_API plt_status plt_propagate_rays(const plt_rays* in, const plt_rays* out, double z_target_mm, plt_dir dir,
                                      int64_t n, void* cuda_stream);

/*
 * End-to-end query of a HOST-resident batch (the inference passage P:397-399 for rays that
 * live in host memory): for chunks of `chunk` rays (a multiple of 32), the library copies
 * the chunk's rays host -> device on its own copy stream, runs the exact trace (lens !=
 * NULL) and/or the map (map != NULL) on `cuda_stream` with their valid hits splatted into
 * splat->film (device, caller-owned, accumulated; splat may be NULL), and copies each
 * chunk's hits back into host_trace / host_map (nullable: not returned).  Chunk c+1's
 * copy overlaps chunk c's kernels (two device staging buffers from the library's pool,
 * ordered by events); nothing synchronises the host.  film_host (nullable, n_film int64)
 * receives the film after the last chunk.  The call returns once all work is enqueued: the
 * host buffers must stay valid until cuda_stream has completed it, and should be pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to overlap.
 * in: HOST SoA rays (dz may be NULL, A32); host_trace / host_map: HOST hit arrays
 * (mask_bits ceil(n/32) words; flags ignored).  Same results as plt_trace_rays_splat /
 * plt_eval_map_splat on the same rays (bit-identical hits and film).
 * Errors: PLT_E_INVALID_ARG (null, chunk not a positive multiple of 32, neither lens nor
 * map), the errors of the query calls, PLT_E_OOM, PLT_E_CUDA.
 */
PLT_API plt_status plt_query_host(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                                  const plt_map* map, const plt_rays* in, const plt_hits* host_trace,
                                  const plt_hits* host_map, const plt_splat_target* splat, int64_t* film_host,
                                  int64_t n, int64_t chunk, void* cuda_stream);

/*
 * Synthetic input rays on the device (SURVEY.md §8(d) "Synthetic inputs": Philox4x32-10
 * keyed by the seed, counted by the global ray index, so results are identical for any
 * batch split or GPU count).  Writes rays [start, start + n) of the law into out's device
 * arrays (n floats each; out->dz may be NULL: rays then carry (dx, dy) only, A32;
 * out->plane_z_mm is not used -- the rays lie on law->plane_z_mm).  Specification (also
 * implemented, independently, by plt_inputs/philox.py; the float32 rays are bit-identical):
 * ray i draws u_0..u_7 = (x + 0.5) 2^-32 from the 8 words of Philox4x32-10 with counter
 * (i mod 2^32, i div 2^32, b, 0x504C5452), b = 0, 1, key (seed mod 2^32, seed div 2^32),
 * and maps them by the law below in IEEE double with one rounding per operation (the
 * angle by an octant reduction and Taylor polynomials, plt_inputs/philox.py):
 *   DISC_CAP    origin uniform on the disc (disc_r, centre (disc_x0, 0)), direction uniform
 *               on the cap w_z >= cap_cos_min, lambda = lo + (hi - lo) u_4;
 *   COLLIMATED  origin as DISC_CAP, direction (dir_x, 0, dir_z);
 *   SENSOR_PUPIL origin uniform on the sensor_w x sensor_h rectangle, direction towards a
 *               point uniform on the disc of radius pupil_r at z = pupil_z;
 *   SENSOR_GRID as SENSOR_PUPIL with ray i in pixel i div spp of a width_px x height_px
 *               grid (row-major, row 0 at +y).
 * Errors: PLT_E_INVALID_ARG (null, bad kind, non-finite field, n < 0, start < 0, grid sizes
 * <= 0), PLT_E_CUDA.
 */
typedef enum { PLT_LAW_DISC_CAP = 0, PLT_LAW_COLLIMATED = 1, PLT_LAW_SENSOR_PUPIL = 2, PLT_LAW_SENSOR_GRID = 3 } plt_law_kind;

typedef struct {
    int kind;                          /* plt_law_kind                                         */
    int width_px, height_px, spp;      /* SENSOR_GRID                                          */
    double plane_z_mm;                 /* plane of the ray origins                             */
    double disc_r_mm, disc_x0_mm;      /* DISC_CAP, COLLIMATED: origin disc                    */
    double cap_cos_min;                /* DISC_CAP: cos of the cap half-angle                  */
    double dir_x, dir_z;               /* COLLIMATED: the fixed unit direction (x-z plane)     */
    double sensor_w_mm, sensor_h_mm;   /* SENSOR_*: sensor rectangle centred on the axis       */
    double pupil_z_mm, pupil_r_mm;     /* SENSOR_*: disc the directions aim at                 */
    double lambda_lo_nm, lambda_hi_nm; /* lambda = lo + (hi - lo) u (lo == hi: one wavelength) */
} plt_ray_law;

PLT_API plt_status plt_gen_rays(const plt_ray_law* law, uint64_t seed, int64_t start, const plt_rays* out, int64_t n,
                                void* cuda_stream);

/* out[i] = film[i] * 2^-32 * scale (float), for channels*height*width pixels. */
PLT_API plt_status plt_film_resolve(const plt_film_desc* film_desc, const int64_t* film, float* out,
                            double scale, void* cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* PLT_H_ */
