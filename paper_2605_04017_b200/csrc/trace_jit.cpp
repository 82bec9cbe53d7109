// trace_jit.cpp -- run-time specialisation of the packed float32 trace for one path program.
//
// The generic kernel (trace_kernel_x2) reads every step of the path program from the
// __grid_constant__ parameter inside the step loop: ~20 uniform constant loads, a loop
// counter and branches on the surface kind / interaction / glass form per step.  For a
// given (lens, path, direction) all of that is known on the host, so this module emits a
// kernel whose steps are literal compile-time constants -- the step loop is unrolled,
// the branches and loads fold away and lens constants become instruction immediates --
// and compiles it with NVRTC for sm_100a on first use (cached per program).  The device
// code is the same trace_dev.cuh the ahead-of-time kernels use; only the step policy
// differs.  NVRTC is loaded with dlopen: if it is missing, or compilation fails, the call
// uses the generic kernel (the same GPU computation, never a CPU path).
#include <dlfcn.h>
#include <nvrtc.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "plt_internal.h"

namespace plt {

namespace {

#include "jit_sources.inc"   // kJitSources[]: plt.h, plt_internal.h, splat_dev.cuh, trace_dev.cuh (no #includes)

struct Nvrtc {
    bool ok = false;
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
};

const Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        const char* env = std::getenv("PLT_NVRTC");
        // The toolkit's NVRTC (the release that built the ahead-of-time kernels) first: a bare
        // "libnvrtc.so.12" resolves to whichever copy the process already loaded -- e.g. the
        // older one bundled with torch, whose code for the same source measured ~9 % more
        // instructions (explicit FADD negations instead of folded FFMA2 operand modifiers).
        const char* names[] = {env, "/usr/local/cuda/lib64/libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so",
                               "libnvrtc.so.12"};
        void* h = nullptr;
        for (const char* nm : names)
            if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return r;
        r.create = (decltype(r.create))dlsym(h, "nvrtcCreateProgram");
        r.compile = (decltype(r.compile))dlsym(h, "nvrtcCompileProgram");
        r.cubin_size = (decltype(r.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
        r.cubin = (decltype(r.cubin))dlsym(h, "nvrtcGetCUBIN");
        r.log_size = (decltype(r.log_size))dlsym(h, "nvrtcGetProgramLogSize");
        r.log = (decltype(r.log))dlsym(h, "nvrtcGetProgramLog");
        r.destroy = (decltype(r.destroy))dlsym(h, "nvrtcDestroyProgram");
        r.ok = r.create && r.compile && r.cubin_size && r.cubin && r.log_size && r.log && r.destroy;
        return r;
    }();
    return n;
}

// Exact float literal (hexadecimal significand; C++17).
std::string lit(float v) {
    char b[64];
    std::snprintf(b, sizeof b, "%af", (double)v);
    return b;
}

const char* kPrelude =
    "#define PLT_JIT 1\n"
    "typedef signed char int8_t; typedef unsigned char uint8_t;\n"
    "typedef short int16_t; typedef unsigned short uint16_t;\n"
    "typedef int int32_t; typedef unsigned int uint32_t;\n"
    "typedef long long int64_t; typedef unsigned long long uint64_t;\n";

bool far_side_air(const Step<float>& st) {   // as step2's `air`: constant n = 1 behind the surface
    return st.gform == kCauchyForm && st.g[0] == 1.f && st.g[1] == 0.f && st.g[2] == 0.f;
}

// Is the ray in air before step s?  (starts in air; a T step enters the medium behind its
// surface, an R step or the stop leaves the medium unchanged)
bool in_air_before(const Program<float>& P, int s) {
    bool air = true;
    for (int k = 0; k < s; ++k)
        if (P.st[k].kind != kStop && !P.st[k].is_R) air = far_side_air(P.st[k]);
    return air;
}

bool verbose() {
    static const bool v = std::getenv("PLT_JIT_VERBOSE") != nullptr;
    return v;
}

// ---- eta polynomials (trace_dev.cuh EtaPoly) ---------------------------------------
// Index behind a step's surface at u = 1/lambda^2 (um^-2), from the same float
// coefficients the kernels use (glass_index2), evaluated in double.
double n_behind(const Step<float>& st, double u) {
    if (st.gform == kCauchyForm) return (double)st.g[0] + u * ((double)st.g[1] + u * (double)st.g[2]);
    const double l2 = 1.0 / u;
    double s = 1.0;
    for (int k = 0; k < 3; ++k) s += (double)st.g[k] * l2 / (l2 - (double)st.g[3 + k]);
    return std::sqrt(s);
}

// Step whose far side is the medium the ray is in before step s (-1: air).
int medium_before(const Program<float>& P, int s) {
    int m = -1;
    for (int k = 0; k < s; ++k)
        if (P.st[k].kind != kStop && !P.st[k].is_R) m = far_side_air(P.st[k]) ? -1 : k;
    return m;
}

// Fit eta(u) of step s as sum_k c_k v^k, v = (u - kEtaU0) kEtaUS (the constants of
// trace_dev.cuh), by interpolation at the Chebyshev nodes of the lowest degree D <= 10
// whose float-rounded coefficients stay within 1.2e-7 relative of eta on a dense grid of
// u in [1.6, 7.0]; false if none does.
// Cauchy / Abbe glasses need degree 3 on 378-791 nm; Sellmeier glasses up to ~9 (their
// infrared term is a pole of eta(u) at u = 0, just outside the interval).
constexpr int kMaxEtaDeg = 10;
bool fit_eta(const Program<float>& P, int s, std::vector<float>& c) {
    // the device computes v = fma(u, kEtaUS, -kEtaU0 * kEtaUS) with these float constants
    const float us_f = 1.f / 2.7f, off_f = -4.3f * us_f;
    const double us = (double)us_f, off = (double)off_f;
    const int m = medium_before(P, s);
    auto eta = [&](double v) {
        const double u = (v - off) / us;
        const double n1 = m < 0 ? 1.0 : n_behind(P.st[m], u);
        const double n2 = far_side_air(P.st[s]) ? 1.0 : n_behind(P.st[s], u);
        return n1 / n2;
    };
    for (int D = 0; D <= kMaxEtaDeg; ++D) {
        double A[kMaxEtaDeg + 1][kMaxEtaDeg + 2];
        for (int k = 0; k <= D; ++k) {
            const double x = std::cos(M_PI * (k + 0.5) / (D + 1));
            double p = 1.0;
            for (int j = 0; j <= D; ++j) { A[k][j] = p; p *= x; }
            A[k][D + 1] = eta(x);
        }
        for (int i = 0; i <= D; ++i) {           // Gaussian elimination with partial pivoting
            int piv = i;
            for (int r = i + 1; r <= D; ++r) if (std::fabs(A[r][i]) > std::fabs(A[piv][i])) piv = r;
            for (int j = 0; j <= D + 1; ++j) std::swap(A[i][j], A[piv][j]);
            for (int r = 0; r <= D; ++r) {
                if (r == i) continue;
                const double f = A[r][i] / A[i][i];
                for (int j = i; j <= D + 1; ++j) A[r][j] -= f * A[i][j];
            }
        }
        c.assign(D + 1, 0.f);
        for (int i = 0; i <= D; ++i) c[i] = (float)(A[i][D + 1] / A[i][i]);
        double worst = 0.0;
        for (int g = 0; g <= 4000; ++g) {
            const double v = -1.0 + g / 2000.0;
            double p = c[D];
            for (int k = D - 1; k >= 0; --k) p = p * v + c[k];
            worst = std::fmax(worst, std::fabs(p / eta(v) - 1.0));
        }
        if (worst <= 1.2e-7) return true;
    }
    return false;
}

// Polynomial eta for every interaction step of P, or empty if any step does not fit
// (the kernel then evaluates the glass formulas exactly).
std::vector<std::vector<float>> eta_polys(const Program<float>& P) {
    std::vector<std::vector<float>> out(P.n_steps);
    for (int s = 0; s < P.n_steps; ++s) {
        if (P.st[s].kind == kStop) continue;
        if (!fit_eta(P, s, out[s])) return {};
    }
    return out;
}

std::string gen_phase(const Program<float>& P, int s0, int s1, const std::vector<std::vector<float>>& polys) {
    std::string c = "        do {\n";
    for (int s = s0; s < s1; ++s) {
        const Step<float>& st = P.st[s];
        const char* n1 = in_air_before(P, s) ? "true" : "false";
        const bool poly = !polys.empty() && st.kind != kStop;
        c += "            if (!__any_sync(0xffffffffu, any2(alive))) break;\n";
        c += "            { constexpr Step<float> st{" + lit(st.z) + ", " + lit(st.R) + ", " + lit(st.twoR) + ", " +
             lit(st.invR) + ", " + lit(st.a2) + ", " + lit(st.band_a) + ", " + lit(st.sdir) + ", {";
        for (int k = 0; k < 6; ++k) c += lit(st.g[k]) + (k < 5 ? ", " : "");
        c += "}, " + std::to_string(st.kind) + ", " + std::to_string(st.is_R) + ", " + std::to_string(st.gform) +
             ", 0, {";
        for (int k = 0; k < 5; ++k) c += lit(st.asph[k]) + (k < 4 ? ", " : "");
        c += "}, " + lit(st.coat_n) + ", " + lit(st.coat_kpi) + "};\n";
        if (poly) {
            const std::vector<float>& e = polys[s];
            c += "              constexpr EtaPoly<" + std::to_string(e.size() - 1) + "> ep{{";
            for (size_t k = 0; k < e.size(); ++k) c += lit(e[k]) + (k + 1 < e.size() ? ", " : "");
            c += "}};\n              step2<true, Hdr, " + std::string(n1) + ", EtaPoly<" + std::to_string(e.size() - 1) +
                 ">>(st, H, ox, oy, oz, wx, wy, wz, I, ncur, r.u, r.l2, alive, near, rho2o, ep, v); }\n";
        } else {
            c += "              step2<true, Hdr, " + std::string(n1) +
                 ">(st, H, ox, oy, oz, wx, wy, wz, I, ncur, r.u, r.l2, alive, near, rho2o); }\n";
        }
    }
    c += "        } while (0);\n";
    return c;
}

int jit_min_blocks() {   // blocks per SM the specialised kernel is register-limited to (tuning knob)
    static const int v = [] {
        const char* e = std::getenv("PLT_JIT_MINB");
        return e ? std::atoi(e) : 4;
    }();
    return v;
}

std::string gen_source(const Program<float>& P) {
    const bool compact = P.split > 0 && P.split < P.n_steps;
    std::string src = kPrelude;
    src += "#define PLT_JIT_MINB " + std::to_string(jit_min_blocks()) + "\n";
    // features the program does not use are compiled out entirely (their mere presence, even
    // constant-folded, changes the generated code: measured 0.610 vs 0.629 ms on C2)
    bool coat = false, asph = false;
    for (int i = 0; i < P.n_steps; ++i) { coat |= P.st[i].coat_n > 0.f; asph |= P.st[i].kind == kAsphere; }
    // eta polynomials: not for coated programs (the film needs n before and behind)
    static const bool poly_off = [] { const char* e = std::getenv("PLT_JIT_ETA_POLY"); return e && e[0] == '0'; }();
    const std::vector<std::vector<float>> polys = (coat || poly_off) ? std::vector<std::vector<float>>{} : eta_polys(P);
    if (verbose()) {
        std::string d;
        for (const auto& e : polys) d += e.empty() ? "-" : std::to_string(e.size() - 1);
        std::fprintf(stderr, "plt: trace JIT eta(lambda): %s\n",
                     polys.empty() ? "exact glass formulas" : ("polynomial degrees per step " + d).c_str());
    }
    if (!coat) src += "#define PLT_NO_COAT 1\n";
    if (!asph) src += "#define PLT_NO_ASPH 1\n";
    if (const char* e = std::getenv("PLT_JIT_DEFINES")) src += std::string(e) + "\n";   // developer A/B knob
    for (const char* part : kJitSources) src += part;
    src += "\nnamespace plt {\nstruct JitSteps {\n"
           "    __device__ __forceinline__ static bool compact(const Program<float>&) { return ";
    src += compact ? "true" : "false";
    src += "; }\n    struct Hdr { int has_housing; float housing2, band_h; };\n"
           "    __device__ __forceinline__ static void run(const Program<float>&, Ray2& r, int phase) {\n"
           "        constexpr Hdr H{" + std::to_string(P.has_housing) + ", " + lit(P.housing2) + ", " + lit(P.band_h) +
           "};\n"
           "        f2 ox = r.ox, oy = r.oy, oz = r.oz, wx = r.wx, wy = r.wy, wz = r.wz, I = r.I, ncur = r.ncur;\n"
           "        m2 alive = r.alive, near = r.near;\n"
           "        f2 rho2o = fma2(ox, ox, oy * oy);\n";
    if (!polys.empty()) {
        src += "        const f2 v = fma2(r.u, mk(kEtaUS), mk(-kEtaU0 * kEtaUS));\n";
        // rays outside the fitted wavelength range go to the exact float64 re-trace
        src += "        if (phase == 0) near = near | (alive & (lt(v, mk(-1.f)) | lt(mk(1.f), v)));\n";
    }
    src += "        if (phase == 0) {\n";
    src += gen_phase(P, 0, compact ? P.split : P.n_steps, polys);
    src += "        } else {\n";
    src += gen_phase(P, compact ? P.split : P.n_steps, P.n_steps, polys);
    src += "        }\n"
           "        r.ox = ox; r.oy = oy; r.oz = oz; r.wx = wx; r.wy = wy; r.wz = wz; r.I = I; r.ncur = ncur;\n"
           "        r.alive = alive; r.near = near;\n    }\n};\n}  // namespace plt\n"
           "extern \"C\" __global__ void __launch_bounds__(256, PLT_JIT_MINB) plt_trace_jit(\n"
           "        const __grid_constant__ plt::Program<float> P, plt_rays in, plt_hits out, int64_t n,\n"
           "        plt::Scratch scr, const __grid_constant__ plt::SplatCtx sc) {\n"
           "    plt::trace_x2_body<plt::JitSteps>(P, in, out, n, scr, sc);\n}\n";
    return src;
}

struct Entry {
    bool tried = false;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
};

std::mutex g_mu;
std::map<std::string, Entry> g_cache;

std::string key_of(const Program<float>& P) {
    const size_t bytes = offsetof(Program<float>, st) + sizeof(Step<float>) * (size_t)P.n_steps;
    return std::string(reinterpret_cast<const char*>(&P), bytes);
}

}  // namespace

std::string trace_jit_source(const Program<float>& P) { return gen_source(P); }

// Compile (or fetch) the specialised kernel for P; nullptr if unavailable.
void* trace_jit_kernel(const Program<float>& P) {
    static const bool off = [] {
        const char* e = std::getenv("PLT_TRACE_JIT");
        return e && std::strcmp(e, "0") == 0;
    }();
    if (off || P.n_steps <= 0) return nullptr;
    const std::string key = key_of(P);
    std::lock_guard<std::mutex> g(g_mu);
    Entry& e = g_cache[key];
    if (e.tried) return (void*)e.kernel;
    e.tried = true;
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) {
        if (verbose()) std::fprintf(stderr, "plt: NVRTC not found; generic trace kernel\n");
        return nullptr;
    }
    const std::string src = gen_source(P);
    nvrtcProgram prog;
    if (nv.create(&prog, src.c_str(), "plt_trace_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return nullptr;
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true", "-default-device"};
    const nvrtcResult rc = nv.compile(prog, 5, opts);
    if (rc != NVRTC_SUCCESS || verbose()) {
        size_t ls = 0;
        nv.log_size(prog, &ls);
        std::vector<char> log(ls + 1, 0);
        nv.log(prog, log.data());
        if (rc != NVRTC_SUCCESS || ls > 1)
            std::fprintf(stderr, "plt: trace JIT %s:\n%s\n", rc == NVRTC_SUCCESS ? "log" : "FAILED", log.data());
    }
    if (rc != NVRTC_SUCCESS) { nv.destroy(&prog); return nullptr; }
    size_t cs = 0;
    nv.cubin_size(prog, &cs);
    std::vector<char> cubin(cs);
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    if (cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&e.kernel, e.lib, "plt_trace_jit") != cudaSuccess) {
        cudaGetLastError();
        e.kernel = nullptr;
        return nullptr;
    }
    if (verbose()) std::fprintf(stderr, "plt: trace JIT compiled (%zu-byte cubin, %d steps)\n", cs, P.n_steps);
    return (void*)e.kernel;
}

// Compile P's kernel to a cubin without a GPU (tests / inspection); "" on failure.
std::string trace_jit_cubin(const Program<float>& P, std::string* log_out) {
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) return {};
    const std::string src = gen_source(P);
    nvrtcProgram prog;
    if (nv.create(&prog, src.c_str(), "plt_trace_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return {};
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true", "-default-device"};
    const nvrtcResult rc = nv.compile(prog, 5, opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    nv.log(prog, &log[0]);
    if (log_out) *log_out = log;
    std::string out;
    if (rc == NVRTC_SUCCESS) {
        size_t cs = 0;
        nv.cubin_size(prog, &cs);
        out.resize(cs);
        nv.cubin(prog, &out[0]);
    }
    nv.destroy(&prog);
    return out;
}

}  // namespace plt
