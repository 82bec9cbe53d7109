// abi.cpp -- the extern "C" entry points of include/plt.h.
//
// Every entry point converts host-layer exceptions into plt_status with a
// thread-local message, validates arguments synchronously, checks that the
// current device is an sm_100 part and enqueues its kernels on the caller's
// stream.  There is no CPU fallback.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "host.h"

namespace {

thread_local std::string g_err;

// NVTX range around every compute entry point (header-only NVTX3: a no-op unless a
// profiler injects itself), so ncu / nsys timelines name the ABI call of each kernel.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PLT_RANGE(name) NvtxRange plt_nvtx_range_(name)

plt_status set_err(plt_status c, const std::string& m) {
    g_err = m;
    return c;
}

#define PLT_GUARD_BEGIN \
    g_err.clear();      \
    try {
#define PLT_GUARD_END                                                   \
    }                                                                   \
    catch (const plt::Error& e) { return set_err(e.code, e.msg); }      \
    catch (const std::bad_alloc&) { return set_err(PLT_E_OOM, "out of host memory"); } \
    catch (const std::exception& e) { return set_err(PLT_E_INVALID_ARG, e.what()); }

plt_status cuda_status(int e, const char* where) {
    if (e == 0) return PLT_OK;
    return set_err(e == (int)cudaErrorMemoryAllocation ? PLT_E_OOM : PLT_E_CUDA,
                   std::string(where) + ": " + cudaGetErrorString((cudaError_t)e));
}

// The kernels are built for sm_100a only; refuse anything else loudly.
plt_status check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_err(PLT_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return set_err(PLT_E_CUDA, "libplt is built for sm_100a (B200); current device is sm_" +
                                       std::to_string(major) + std::to_string(minor));
    return PLT_OK;
}

bool rays_ok(const plt_rays* r) {
    // dz may be NULL: directions given by their (x, y) components (include/plt.h)
    return r && r->ox && r->oy && r->dx && r->dy && r->lambda_nm && std::isfinite(r->plane_z_mm);
}
bool hits_ok(const plt_hits* h) {
    return h && h->mask_bits && h->px && h->py && h->dx && h->dy && h->dz && h->throughput;
}

}  // namespace

extern "C" {

const char* plt_last_error(void) { return g_err.c_str(); }

const char* plt_version(void) { return "plt 0.1 sm_100a"; }

plt_status plt_lens_load(const char* text, size_t len, const plt_lens_opts* opts, plt_lens** out) {
    PLT_GUARD_BEGIN
    if (!text || !out) return set_err(PLT_E_INVALID_ARG, "text and out must be non-null");
    *out = plt::parse_lens(text, len, opts);
    return PLT_OK;
    PLT_GUARD_END
}

void plt_lens_free(plt_lens* lens) { delete lens; }

plt_status plt_lens_info(const plt_lens* lens, double lambda_nm, int* n_optical, int* stop_index,
                         double abcd[4], double* efl_mm, double* bfl_mm, double* sensor_z_mm) {
    PLT_GUARD_BEGIN
    if (!lens) return set_err(PLT_E_INVALID_ARG, "lens is null");
    if (!(lambda_nm >= 380.0 && lambda_nm <= 780.0))
        return set_err(PLT_E_INVALID_ARG, "lambda_nm outside [380, 780] nm (S:60-62)");
    double M[4];
    plt::lens_abcd(*lens, lambda_nm, M);
    if (n_optical) *n_optical = lens->n_optical;
    if (stop_index) *stop_index = lens->stop_index;
    if (abcd) std::memcpy(abcd, M, sizeof M);
    if (efl_mm) *efl_mm = M[2] != 0.0 ? -1.0 / M[2] : INFINITY;
    if (bfl_mm) *bfl_mm = M[2] != 0.0 ? -M[0] / M[2] : INFINITY;
    if (sensor_z_mm) *sensor_z_mm = lens->sensor_z;
    return PLT_OK;
    PLT_GUARD_END
}

plt_status plt_lens_pupils(const plt_lens* lens, double lambda_nm, double* ez, double* er, double* xz, double* xr) {
    PLT_GUARD_BEGIN
    if (!lens || !ez || !er || !xz || !xr) return set_err(PLT_E_INVALID_ARG, "null argument");
    double o[4];
    plt::lens_pupils(*lens, lambda_nm, o);
    *ez = o[0]; *er = o[1]; *xz = o[2]; *xr = o[3];
    return PLT_OK;
    PLT_GUARD_END
}

plt_status plt_enumerate_ghosts(const plt_lens* lens, int max_bounces, double min_throughput, uint64_t* ids,
                                int32_t* ij_pairs, int capacity, int* count) {
    PLT_GUARD_BEGIN
    if (!lens || !count) return set_err(PLT_E_INVALID_ARG, "lens and count must be non-null");
    if (max_bounces != 0 && max_bounces != 2 && max_bounces != 4)
        return set_err(PLT_E_UNSUPPORTED, "max_bounces must be 0, 2 or 4 (P:339: higher orders negligible)");
    auto v = plt::enumerate_ghosts(*lens, max_bounces, min_throughput);
    *count = (int)v.size();
    if (!ids || capacity < (int)v.size())
        return set_err(PLT_E_CAPACITY, "capacity " + std::to_string(capacity) + " < " + std::to_string(v.size()));
    for (size_t i = 0; i < v.size(); ++i) {
        ids[i] = v[i].first;
        if (ij_pairs) { ij_pairs[2 * i] = v[i].second.first; ij_pairs[2 * i + 1] = v[i].second.second; }
    }
    return PLT_OK;
    PLT_GUARD_END
}

static bool film_desc_ok(const plt_film_desc* fd) {
    return fd && fd->width_px > 0 && fd->height_px > 0 && fd->channels > 0 && fd->sensor_w_mm > 0 &&
           fd->sensor_h_mm > 0 && std::isfinite(fd->center_x_mm) && std::isfinite(fd->center_y_mm) &&
           (int64_t)fd->width_px * fd->height_px * fd->channels < ((int64_t)1 << 31);   // 32-bit pixel keys
}

// Validate a fused-splat target; on success *sc holds the kernel constants.
static plt_status splat_target(const plt_splat_target* t, plt::SplatCtx* sc) {
    *sc = plt::SplatCtx{};
    sc->film = nullptr;
    if (!t) return PLT_OK;
    if (!t->film || !film_desc_ok(t->film_desc)) return set_err(PLT_E_INVALID_ARG, "bad splat target (film / film_desc)");
    *sc = plt::make_splat_ctx(*t->film_desc, t->film, t->channel, t->weight_scale, t->dropped);
    return PLT_OK;
}

static plt_status trace_impl(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                             const plt_rays* in, const plt_hits* out, const plt_splat_target* splat, int64_t n,
                             void* cuda_stream);

plt_status plt_trace_rays(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                          const plt_rays* in, const plt_hits* out, int64_t n, void* cuda_stream) {
    return trace_impl(lens, path_id, dir, prec, in, out, nullptr, n, cuda_stream);
}

plt_status plt_trace_rays_splat(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                                const plt_rays* in, const plt_hits* out, const plt_splat_target* splat, int64_t n,
                                void* cuda_stream) {
    if (!splat) return set_err(PLT_E_INVALID_ARG, "splat target is null");
    return trace_impl(lens, path_id, dir, prec, in, out, splat, n, cuda_stream);
}

static plt_status trace_impl(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                             const plt_rays* in, const plt_hits* out, const plt_splat_target* splat, int64_t n,
                             void* cuda_stream) {
    PLT_RANGE(splat ? "plt_trace_rays_splat" : "plt_trace_rays");
    PLT_GUARD_BEGIN
    if (!lens) return set_err(PLT_E_INVALID_ARG, "lens is null");
    if (dir != PLT_FORWARD && dir != PLT_BACKWARD) return set_err(PLT_E_INVALID_ARG, "bad direction");
    if (prec != PLT_FP32 && prec != PLT_FP64) return set_err(PLT_E_INVALID_ARG, "bad precision");
    if (n < 0) return set_err(PLT_E_INVALID_ARG, "n < 0");
    auto cp = plt::compile_path(*lens, path_id, (int)dir);  // validates the path id
    if (n == 0) return PLT_OK;
    if (!rays_ok(in) || !hits_ok(out)) return set_err(PLT_E_INVALID_ARG, "null ray/hit pointer or non-finite plane z");
    if (n >= (int64_t)1 << 31) return set_err(PLT_E_INVALID_ARG, "n must be < 2^31 per call");
    plt::SplatCtx sc;
    plt_status s = splat_target(splat, &sc);
    if (s != PLT_OK) return s;
    s = check_device();
    if (s != PLT_OK) return s;
    if (prec == PLT_FP32)
        return cuda_status(plt::launch_trace_fp32(cp->pf, cp->pd, *in, *out, n, cuda_stream, sc), "trace_rays");
    return cuda_status(plt::launch_trace_fp64(cp->pd, *in, *out, n, cuda_stream, sc), "trace_rays(fp64)");
    PLT_GUARD_END
}

plt_status plt_trace_paths(const plt_lens* lens, const uint64_t* path_ids, int n_paths, plt_dir dir,
                           plt_precision prec, const plt_rays* in, const plt_hits* outs,
                           const plt_splat_target* splat, int64_t n, void* cuda_stream) {
    PLT_RANGE("plt_trace_paths");
    PLT_GUARD_BEGIN
    if (!lens) return set_err(PLT_E_INVALID_ARG, "lens is null");
    if (dir != PLT_FORWARD && dir != PLT_BACKWARD) return set_err(PLT_E_INVALID_ARG, "bad direction");
    if (prec != PLT_FP32 && prec != PLT_FP64) return set_err(PLT_E_INVALID_ARG, "bad precision");
    if (n < 0) return set_err(PLT_E_INVALID_ARG, "n < 0");
    if (n_paths < 0) return set_err(PLT_E_INVALID_ARG, "n_paths < 0");
    if (n_paths > 0 && (!path_ids || !outs)) return set_err(PLT_E_INVALID_ARG, "null path_ids / outs");
    std::vector<std::shared_ptr<plt::CompiledPath>> cps;
    for (int p = 0; p < n_paths; ++p) cps.push_back(plt::compile_path(*lens, path_ids[p], (int)dir));
    if (n == 0 || n_paths == 0) return PLT_OK;
    if (!rays_ok(in)) return set_err(PLT_E_INVALID_ARG, "null ray pointer or non-finite plane z");
    for (int p = 0; p < n_paths; ++p)
        if (!hits_ok(&outs[p])) return set_err(PLT_E_INVALID_ARG, "null hit pointer in outs[" + std::to_string(p) + "]");
    if (n >= (int64_t)1 << 31) return set_err(PLT_E_INVALID_ARG, "n must be < 2^31 per call");
    plt::SplatCtx sc;
    plt_status s = splat_target(splat, &sc);
    if (s != PLT_OK) return s;
    s = check_device();
    if (s != PLT_OK) return s;
    if (prec == PLT_FP32) {
        for (int p = 0; p < n_paths; ++p) {
            s = cuda_status(plt::launch_trace_fp32(cps[p]->pf, cps[p]->pd, *in, outs[p], n, cuda_stream, sc),
                            "trace_paths(fp32)");
            if (s != PLT_OK) return s;
        }
        return PLT_OK;
    }
    // the all-T program is the shared prefix; path p shares its steps [0, d_p), d_p = its
    // first reflection, when those steps and the frame are the same bytes
    auto pre = plt::compile_path(*lens, (uint64_t)1 << lens->n_optical, (int)dir);
    const plt::Program<double>& A = pre->pd;
    std::vector<const plt::Program<double>*> progs;
    std::vector<int> depth;
    for (int p = 0; p < n_paths; ++p) {
        const plt::Program<double>& P = cps[p]->pd;
        int d = 0;
        while (d < P.n_steps && !P.st[d].is_R) ++d;
        const bool same_frame = P.flip == A.flip && P.z_mirror == A.z_mirror && P.has_housing == A.has_housing &&
                                P.housing2 == A.housing2 && P.has_asph == A.has_asph;
        if (d >= P.n_steps || d > A.n_steps || !same_frame ||
            std::memcmp(P.st, A.st, sizeof(plt::Step<double>) * (size_t)d) != 0)
            d = 0;   // no reflection (all-T), or no common prefix: traced alone
        progs.push_back(&P);
        depth.push_back(d);
    }
    return cuda_status(plt::launch_trace_paths_fp64(A, progs, depth, *in, outs, n, cuda_stream, sc),
                       "trace_paths(fp64)");
    PLT_GUARD_END
}

plt_status plt_map_load(const plt_lens* lens, const void* blob, size_t len, plt_map** out) {
    PLT_GUARD_BEGIN
    if (!blob || !out) return set_err(PLT_E_INVALID_ARG, "blob and out must be non-null");
    *out = plt::parse_map(lens, (const uint8_t*)blob, len);
    return PLT_OK;
    PLT_GUARD_END
}

void plt_map_free(plt_map* map) { delete map; }

static plt_status eval_map_impl(const plt_map* map, const plt_rays* in, const plt_hits* out, float* raw_out,
                                const plt_splat_target* splat, int64_t n, void* cuda_stream);

plt_status plt_eval_map(const plt_map* map, const plt_rays* in, const plt_hits* out, float* raw_out, int64_t n,
                        void* cuda_stream) {
    return eval_map_impl(map, in, out, raw_out, nullptr, n, cuda_stream);
}

plt_status plt_eval_map_splat(const plt_map* map, const plt_rays* in, const plt_hits* out, float* raw_out,
                              const plt_splat_target* splat, int64_t n, void* cuda_stream) {
    if (!splat) return set_err(PLT_E_INVALID_ARG, "splat target is null");
    return eval_map_impl(map, in, out, raw_out, splat, n, cuda_stream);
}

static plt_status eval_map_impl(const plt_map* map, const plt_rays* in, const plt_hits* out, float* raw_out,
                                const plt_splat_target* splat, int64_t n, void* cuda_stream) {
    PLT_RANGE(splat ? "plt_eval_map_splat" : "plt_eval_map");
    PLT_GUARD_BEGIN
    if (!map) return set_err(PLT_E_INVALID_ARG, "map is null");
    if (n < 0) return set_err(PLT_E_INVALID_ARG, "n < 0");
    if (n == 0) return PLT_OK;
    if (!rays_ok(in) || !hits_ok(out)) return set_err(PLT_E_INVALID_ARG, "null ray/hit pointer");
    if (n >= (int64_t)1 << 31) return set_err(PLT_E_INVALID_ARG, "n must be < 2^31 per call");
    if (map->has_plane && std::fabs(in->plane_z_mm - map->plane_z) > 1e-6 * (1.0 + std::fabs(map->plane_z)))
        return set_err(PLT_E_INVALID_ARG, "rays lie on the plane z = " + std::to_string(in->plane_z_mm) +
                                              " mm but the map was trained on z = " + std::to_string(map->plane_z) +
                                              " mm (move them with plt_propagate_rays)");
    plt::SplatCtx sc;
    plt_status s = splat_target(splat, &sc);
    if (s != PLT_OK) return s;
    s = check_device();
    if (s != PLT_OK) return s;
    int dev = 0;
    cudaGetDevice(&dev);
    void* d_img = nullptr;
    {
        std::lock_guard<std::mutex> g(map->mu);
        auto it = map->dev_image.find(dev);
        if (it == map->dev_image.end()) {
            cudaError_t e = cudaMalloc(&d_img, map->image.size());
            if (e != cudaSuccess) return cuda_status((int)e, "eval_map weight upload");
            e = cudaMemcpy(d_img, map->image.data(), map->image.size(), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) { cudaFree(d_img); return cuda_status((int)e, "eval_map weight upload"); }
            map->dev_image[dev] = d_img;
        } else {
            d_img = it->second;
        }
    }
    return cuda_status(plt::launch_eval_map(d_img, map->layout, map->params, *in, *out, raw_out, n, cuda_stream, sc),
                       "eval_map");
    PLT_GUARD_END
}

plt_status plt_splat_sensor(const plt_film_desc* fd, int64_t* film, const plt_hits* hits, const uint8_t* channel,
                            float weight_scale, int64_t n, unsigned long long* dropped, void* cuda_stream) {
    PLT_RANGE("plt_splat_sensor");
    PLT_GUARD_BEGIN
    if (!fd || !film || !hits) return set_err(PLT_E_INVALID_ARG, "null film/hits");
    if (!film_desc_ok(fd)) return set_err(PLT_E_INVALID_ARG, "bad film description");
    if (n < 0) return set_err(PLT_E_INVALID_ARG, "n < 0");
    if (n == 0) return PLT_OK;
    if (!hits->mask_bits || !hits->px || !hits->py || !hits->dz || !hits->throughput)
        return set_err(PLT_E_INVALID_ARG, "null hit arrays");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    return cuda_status(plt::launch_splat(*fd, film, *hits, channel, weight_scale, n, dropped, cuda_stream), "splat_sensor");
    PLT_GUARD_END
}

plt_status plt_trace_jit_cubin(const plt_lens* lens, uint64_t path_id, plt_dir dir, void* buf, size_t capacity,
                               size_t* size) {
    PLT_GUARD_BEGIN
    if (!lens || !size) return set_err(PLT_E_INVALID_ARG, "lens and size must be non-null");
    if (dir != PLT_FORWARD && dir != PLT_BACKWARD) return set_err(PLT_E_INVALID_ARG, "bad direction");
    auto cp = plt::compile_path(*lens, path_id, (int)dir);
    std::string log;
    const std::string cubin = plt::trace_jit_cubin(cp->pf, &log);
    if (cubin.empty())
        return log.empty() ? set_err(PLT_E_UNSUPPORTED, "NVRTC is not available")
                           : set_err(PLT_E_VALIDATION, "trace JIT compilation failed: " + log);
    *size = cubin.size();
    if (!buf || capacity < cubin.size()) return buf ? set_err(PLT_E_CAPACITY, "buffer too small") : PLT_OK;
    std::memcpy(buf, cubin.data(), cubin.size());
    return PLT_OK;
    PLT_GUARD_END
}

plt_status plt_trace_kernel(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                            plt_kernel_kind* kind) {
    PLT_GUARD_BEGIN
    if (!lens || !kind) return set_err(PLT_E_INVALID_ARG, "lens and kind must be non-null");
    if (dir != PLT_FORWARD && dir != PLT_BACKWARD) return set_err(PLT_E_INVALID_ARG, "bad direction");
    if (prec != PLT_FP32 && prec != PLT_FP64) return set_err(PLT_E_INVALID_ARG, "bad precision");
    auto cp = plt::compile_path(*lens, path_id, (int)dir);
    if (prec == PLT_FP64) { *kind = PLT_KERNEL_FP64; return PLT_OK; }
    plt_status s = check_device();   // the JIT compiles for, and loads on, the current device
    if (s != PLT_OK) return s;
    *kind = (plt_kernel_kind)plt::trace_fp32_kind(cp->pf, nullptr);
    return PLT_OK;
    PLT_GUARD_END
}

static plt_status shade_impl(const plt_scene_plane* scene, double z_hits_mm, const plt_hits* hits, int spp,
                             int64_t pixels, float weight_scale, const float* in_dz, int64_t* film, int64_t n,
                             void* cuda_stream) {
    PLT_RANGE("plt_shade_plane");
    PLT_GUARD_BEGIN
    if (!scene || !hits || !film) return set_err(PLT_E_INVALID_ARG, "null scene/hits/film");
    if (!(scene->period_mm > 0) || !std::isfinite(scene->z_mm) || !std::isfinite(scene->contrast) ||
        !std::isfinite(z_hits_mm))
        return set_err(PLT_E_INVALID_ARG, "bad scene plane");
    if (spp <= 0 || pixels <= 0 || n < 0) return set_err(PLT_E_INVALID_ARG, "spp, pixels must be > 0 and n >= 0");
    if (n == 0) return PLT_OK;
    if (!hits->mask_bits || !hits->px || !hits->py || !hits->dx || !hits->dy || !hits->dz || !hits->throughput)
        return set_err(PLT_E_INVALID_ARG, "null hit arrays");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    const plt::ScenePlane sc{scene->z_mm, scene->period_mm, scene->contrast};
    return cuda_status(plt::launch_shade_plane(sc, z_hits_mm, *hits, spp, pixels, weight_scale, film, n, cuda_stream,
                                                  in_dz),
                       "shade_plane");
    PLT_GUARD_END
}

plt_status plt_shade_plane(const plt_scene_plane* scene, double z_hits_mm, const plt_hits* hits, int spp,
                           int64_t pixels, float weight_scale, int64_t* film, int64_t n, void* cuda_stream) {
    return shade_impl(scene, z_hits_mm, hits, spp, pixels, weight_scale, nullptr, film, n, cuda_stream);
}

plt_status plt_shade_cards(const plt_scene_card* cards, int n_cards, double background, double z_hits_mm,
                           const plt_hits* hits, int spp, int64_t pixels, float weight_scale, const float* in_dz,
                           int64_t* film, int64_t n, void* cuda_stream) {
    PLT_RANGE("plt_shade_cards");
    PLT_GUARD_BEGIN
    if (!cards || !hits || !film) return set_err(PLT_E_INVALID_ARG, "null cards/hits/film");
    if (n_cards < 1 || n_cards > plt::kMaxCards) return set_err(PLT_E_INVALID_ARG, "n_cards must be 1..8");
    plt::SceneCards sc{};
    sc.n = n_cards;
    sc.background = background;
    for (int k = 0; k < n_cards; ++k) {
        const plt_scene_card& c = cards[k];
        if (!(c.period_mm > 0) || !std::isfinite(c.z_mm) || !std::isfinite(c.contrast) || !(c.x1_mm >= c.x0_mm) ||
            !(c.y1_mm >= c.y0_mm))
            return set_err(PLT_E_INVALID_ARG, "bad scene card " + std::to_string(k));
        sc.z[k] = c.z_mm; sc.period[k] = c.period_mm; sc.contrast[k] = c.contrast;
        sc.x0[k] = c.x0_mm; sc.x1[k] = c.x1_mm; sc.y0[k] = c.y0_mm; sc.y1[k] = c.y1_mm;
    }
    if (!std::isfinite(background) || !std::isfinite(z_hits_mm)) return set_err(PLT_E_INVALID_ARG, "bad scene");
    if (spp <= 0 || pixels <= 0 || n < 0) return set_err(PLT_E_INVALID_ARG, "spp, pixels must be > 0 and n >= 0");
    if (n == 0) return PLT_OK;
    if (!hits->mask_bits || !hits->px || !hits->py || !hits->dx || !hits->dy || !hits->dz || !hits->throughput)
        return set_err(PLT_E_INVALID_ARG, "null hit arrays");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    return cuda_status(plt::launch_shade_cards(sc, z_hits_mm, *hits, spp, pixels, weight_scale, film, n, cuda_stream,
                                               in_dz),
                       "shade_cards");
    PLT_GUARD_END
}

plt_status plt_shade_plane_weighted(const plt_scene_plane* scene, double z_hits_mm, const plt_hits* hits, int spp,
                                    int64_t pixels, float weight_scale, const float* in_dz, int64_t* film, int64_t n,
                                    void* cuda_stream) {
    if (!in_dz && n > 0) return set_err(PLT_E_INVALID_ARG, "null in_dz (sensor-ray direction z-components)");
    return shade_impl(scene, z_hits_mm, hits, spp, pixels, weight_scale, in_dz, film, n, cuda_stream);
}

plt_status plt_pupil_weight(double sensor_z_mm, double disc_z_mm, double disc_r_mm, double* weight) {
    PLT_GUARD_BEGIN
    if (!weight) return set_err(PLT_E_INVALID_ARG, "weight is null");
    const double dz = sensor_z_mm - disc_z_mm;
    if (!std::isfinite(sensor_z_mm) || !std::isfinite(disc_z_mm) || !std::isfinite(disc_r_mm) || !(disc_r_mm > 0) ||
        dz == 0.0)
        return set_err(PLT_E_INVALID_ARG, "bad pupil disc");
    // Eq. 9 estimator of pupil sampling (plt.h plt_shade_plane_weighted): solid-angle pdf
    // dz^2 / (A cos^3 theta) with A = pi r^2; the cos^4 factor is applied per ray in-kernel
    *weight = 3.14159265358979323846 * disc_r_mm * disc_r_mm / (dz * dz);
    return PLT_OK;
    PLT_GUARD_END
}

plt_status plt_propagate_rays(const plt_rays* in, const plt_rays* out, double z_target_mm, plt_dir dir, int64_t n,
                              void* cuda_stream) {
    PLT_RANGE("plt_propagate_rays");
    PLT_GUARD_BEGIN
    if (dir != PLT_FORWARD && dir != PLT_BACKWARD) return set_err(PLT_E_INVALID_ARG, "bad direction");
    if (n < 0) return set_err(PLT_E_INVALID_ARG, "n < 0");
    if (n == 0) return PLT_OK;
    if (!rays_ok(in) || !out || !out->ox || !out->oy || !out->dx || !out->dy || (in->dz && !out->dz) || !out->lambda_nm ||
        !std::isfinite(z_target_mm))
        return set_err(PLT_E_INVALID_ARG, "null ray pointer or non-finite plane");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    return cuda_status(plt::launch_propagate(*in, *out, (float)z_target_mm, dir == PLT_BACKWARD ? -1.f : 1.f, n,
                                             cuda_stream),
                       "propagate_rays");
    PLT_GUARD_END
}

plt_status plt_gen_rays(const plt_ray_law* law, uint64_t seed, int64_t start, const plt_rays* out, int64_t n,
                        void* cuda_stream) {
    PLT_RANGE("plt_gen_rays");
    PLT_GUARD_BEGIN
    if (!law || !out) return set_err(PLT_E_INVALID_ARG, "null law / out");
    if (law->kind < PLT_LAW_DISC_CAP || law->kind > PLT_LAW_SENSOR_GRID) return set_err(PLT_E_INVALID_ARG, "bad law kind");
    const double f[] = {law->plane_z_mm, law->disc_r_mm, law->disc_x0_mm, law->cap_cos_min, law->dir_x, law->dir_z,
                        law->sensor_w_mm, law->sensor_h_mm, law->pupil_z_mm, law->pupil_r_mm, law->lambda_lo_nm,
                        law->lambda_hi_nm};
    for (double v : f)
        if (!std::isfinite(v)) return set_err(PLT_E_INVALID_ARG, "non-finite ray-law field");
    if (law->kind == PLT_LAW_SENSOR_GRID && (law->width_px <= 0 || law->height_px <= 0 || law->spp <= 0))
        return set_err(PLT_E_INVALID_ARG, "sensor grid sizes must be > 0");
    if (n < 0 || start < 0) return set_err(PLT_E_INVALID_ARG, "n and start must be >= 0");
    if (n == 0) return PLT_OK;
    if (!out->ox || !out->oy || !out->dx || !out->dy || !out->lambda_nm)
        return set_err(PLT_E_INVALID_ARG, "null ray array");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    return cuda_status(plt::launch_gen_rays(*law, seed, start, *out, n, cuda_stream), "gen_rays");
    PLT_GUARD_END
}

plt_status plt_film_resolve(const plt_film_desc* fd, const int64_t* film, float* out, double scale, void* cuda_stream) {
    PLT_RANGE("plt_film_resolve");
    PLT_GUARD_BEGIN
    if (!fd || !film || !out) return set_err(PLT_E_INVALID_ARG, "null film/out");
    if (fd->width_px <= 0 || fd->height_px <= 0 || fd->channels <= 0) return set_err(PLT_E_INVALID_ARG, "bad film description");
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    return cuda_status(plt::launch_resolve(*fd, film, out, scale, cuda_stream), "film_resolve");
    PLT_GUARD_END
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// plt_query_host: chunked host -> device -> query -> host pipeline (include/plt.h).
// ---------------------------------------------------------------------------------------
namespace {

// One library-owned, non-blocking copy stream per device (created on first use).
std::mutex g_copy_mu;
std::vector<cudaStream_t> g_copy_streams;

cudaError_t copy_stream(cudaStream_t* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(g_copy_mu);
    if ((int)g_copy_streams.size() <= dev) g_copy_streams.resize(dev + 1, nullptr);
    if (!g_copy_streams[dev]) {
        e = cudaStreamCreateWithFlags(&g_copy_streams[dev], cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
    }
    *out = g_copy_streams[dev];
    return cudaSuccess;
}

struct EventPool {   // events destroyed when the call returns (destruction is deferred by CUDA)
    std::vector<cudaEvent_t> ev;
    cudaError_t make(int k) {
        ev.resize(k, nullptr);
        for (auto& x : ev) {
            cudaError_t e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    ~EventPool() { for (auto x : ev) if (x) cudaEventDestroy(x); }
};

}  // namespace

extern "C" plt_status plt_query_host(const plt_lens* lens, uint64_t path_id, plt_dir dir, plt_precision prec,
                                     const plt_map* map, const plt_rays* in, const plt_hits* host_trace,
                                     const plt_hits* host_map, const plt_splat_target* splat, int64_t* film_host,
                                     int64_t n, int64_t chunk, void* cuda_stream) {
    PLT_RANGE("plt_query_host");
    PLT_GUARD_BEGIN
    if (!lens && !map) return set_err(PLT_E_INVALID_ARG, "neither lens nor map given");
    if (!rays_ok(in)) return set_err(PLT_E_INVALID_ARG, "null host ray pointer or non-finite plane z");
    if (n < 0 || chunk <= 0 || chunk % 32) return set_err(PLT_E_INVALID_ARG, "n >= 0 and chunk a positive multiple of 32");
    if (host_trace && !hits_ok(host_trace)) return set_err(PLT_E_INVALID_ARG, "null host_trace array");
    if (host_map && !hits_ok(host_map)) return set_err(PLT_E_INVALID_ARG, "null host_map array");
    if (film_host && (!splat || !splat->film || !splat->film_desc))
        return set_err(PLT_E_INVALID_ARG, "film_host needs a splat target");
    if (n == 0) return PLT_OK;
    plt_status s = check_device();
    if (s != PLT_OK) return s;
    const int64_t C = chunk < n ? chunk : ((n + 31) / 32) * 32;
    cudaStream_t cs = (cudaStream_t)cuda_stream, xs = nullptr;
    cudaError_t e = copy_stream(&xs);
    if (e != cudaSuccess) return cuda_status((int)e, "query_host copy stream");
    const bool has_dz = in->dz != nullptr;
    const int nin = has_dz ? 6 : 5;
    const int nq = (lens ? 1 : 0) + (map ? 1 : 0);
    // per staging slot: inputs, then per query 6 output arrays + mask words
    const size_t words = (size_t)(C / 32);
    const size_t slot_bytes = (size_t)C * 4 * nin + nq * ((size_t)C * 4 * 6 + words * 4);
    plt::ScratchGuard stage(cuda_stream);
    e = (cudaError_t)stage.alloc(2 * slot_bytes + 256);
    if (e != cudaSuccess) return cuda_status((int)e, "query_host staging");
    EventPool evs;
    e = evs.make(5);   // [0,1] inputs of slot b copied, [2,3] slot b consumed (compute + D2H), [4] copies done
    if (e != cudaSuccess) return cuda_status((int)e, "query_host events");
    // the staging memory is free for the copy stream once earlier work on cs is done
    e = cudaEventRecord(evs.ev[2], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(xs, evs.ev[2], 0);
    if (e == cudaSuccess) e = cudaEventRecord(evs.ev[3], cs);
    if (e != cudaSuccess) return cuda_status((int)e, "query_host ordering");
    for (int64_t lo = 0, c = 0; lo < n; lo += C, ++c) {
        const int64_t cn = (n - lo) < C ? (n - lo) : C;
        const int b = (int)(c & 1);
        char* base = (char*)stage.p + b * slot_bytes;
        float* din[6];
        for (int k = 0; k < nin; ++k) din[k] = (float*)(base + (size_t)k * C * 4);
        const float* hin[6] = {in->ox, in->oy, in->dx, in->dy, has_dz ? in->dz : in->lambda_nm, in->lambda_nm};
        // slot b is reusable once its previous chunk's kernels and D2H copies are done
        e = cudaStreamWaitEvent(xs, evs.ev[2 + b], 0);
        for (int k = 0; k < nin && e == cudaSuccess; ++k)
            e = cudaMemcpyAsync(din[k], hin[k] + lo, (size_t)cn * 4, cudaMemcpyHostToDevice, xs);
        if (e == cudaSuccess) e = cudaEventRecord(evs.ev[b], xs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, evs.ev[b], 0);
        if (e != cudaSuccess) return cuda_status((int)e, "query_host H2D");
        plt_rays dr{din[0], din[1], din[2], din[3], has_dz ? din[4] : nullptr, din[nin - 1], in->plane_z_mm};
        char* ob = base + (size_t)C * 4 * nin;
        plt_hits dh[2];
        for (int q = 0; q < nq; ++q) {
            char* o = ob + q * ((size_t)C * 4 * 6 + words * 4);
            dh[q] = plt_hits{(uint32_t*)(o + (size_t)C * 4 * 6), (float*)o, (float*)(o + (size_t)C * 4),
                             (float*)(o + (size_t)C * 8), (float*)(o + (size_t)C * 12), (float*)(o + (size_t)C * 16),
                             (float*)(o + (size_t)C * 20), nullptr};
        }
        plt_splat_target st{};
        if (splat) {   // the channel array (device, indexed like the rays) follows the chunk
            st = *splat;
            if (st.channel) st.channel += lo;
        }
        int q = 0;
        if (lens) {
            s = splat ? plt_trace_rays_splat(lens, path_id, dir, prec, &dr, &dh[q], &st, cn, cuda_stream)
                      : plt_trace_rays(lens, path_id, dir, prec, &dr, &dh[q], cn, cuda_stream);
            if (s != PLT_OK) return s;
            ++q;
        }
        if (map) {
            s = splat ? plt_eval_map_splat(map, &dr, &dh[q], nullptr, &st, cn, cuda_stream)
                      : plt_eval_map(map, &dr, &dh[q], nullptr, cn, cuda_stream);
            if (s != PLT_OK) return s;
        }
        // hits back to the host on the copy stream, after the kernels
        e = cudaEventRecord(evs.ev[2 + b], cs);
        bool d2h = false;
        for (int k = 0; k < nq && e == cudaSuccess; ++k) {
            const plt_hits* H = lens && k == 0 ? host_trace : host_map;
            if (!H) continue;
            if (!d2h) { e = cudaStreamWaitEvent(xs, evs.ev[2 + b], 0); d2h = true; }
            float* const dst[6] = {H->px, H->py, H->dx, H->dy, H->dz, H->throughput};
            float* const src[6] = {dh[k].px, dh[k].py, dh[k].dx, dh[k].dy, dh[k].dz, dh[k].throughput};
            for (int a = 0; a < 6 && e == cudaSuccess; ++a)
                e = cudaMemcpyAsync(dst[a] + lo, src[a], (size_t)cn * 4, cudaMemcpyDeviceToHost, xs);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(H->mask_bits + lo / 32, dh[k].mask_bits, (size_t)((cn + 31) / 32) * 4,
                                    cudaMemcpyDeviceToHost, xs);
        }
        if (d2h && e == cudaSuccess) e = cudaEventRecord(evs.ev[2 + b], xs);   // slot free after the D2H too
        if (e != cudaSuccess) return cuda_status((int)e, "query_host D2H");
    }
    // the caller's stream completes only after the last copies; then the staging is freed
    e = cudaEventRecord(evs.ev[4], xs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, evs.ev[4], 0);
    if (e == cudaSuccess && film_host) {
        const plt_film_desc& fd = *splat->film_desc;
        e = cudaMemcpyAsync(film_host, splat->film, (size_t)fd.channels * fd.height_px * fd.width_px * 8,
                            cudaMemcpyDeviceToHost, cs);
    }
    if (e != cudaSuccess) return cuda_status((int)e, "query_host");
    return cuda_status(stage.release(), "query_host staging");
    PLT_GUARD_END
}
