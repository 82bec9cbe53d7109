// host.h -- host-side lens / map objects behind the opaque ABI handles.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "plt_internal.h"

namespace plt {

// Glass models (paper silent on dispersion): constant, Cauchy, Abbe (n_d, V_d)
// mapped to a two-term Cauchy law that is exact at d and reproduces n_F - n_C = (n_d-1)/V_d,
// and Sellmeier.
struct Glass {
    enum Model { kConst = 0, kCauchy = 1, kAbbe = 2, kSellmeier = 3 } model = kConst;
    double c[6] = {1.0, 0, 0, 0, 0, 0};
    double index(double lambda_nm) const;
    // Coefficients for the device evaluator: Cauchy form (A, B, C) or Sellmeier (B1..3, C1..3).
    void device_form(int* gform, double g[6]) const;
};

struct Surface {
    double z = 0, R = 0, a = 0;
    bool stop = false;
    Glass before, after;
    // even asphere: conic k and A4, A6, A8, A10
    bool asph = false;
    double k = 0, A[4] = {0, 0, 0, 0};
    // single-layer AR coating (NEXT-4): index, thickness in um (0 = bare)
    double coat_n = 0, coat_d_um = 0;
};

// Thrown inside the host layer, converted to plt_status at the ABI boundary.
struct Error {
    plt_status code;
    std::string msg;
};

struct CompiledPath {
    Program<float> pf;
    Program<double> pd;
};

}  // namespace plt

struct plt_lens {
    std::string name;
    std::vector<plt::Surface> surf;
    plt_lens_opts opts{};
    double sensor_z = 0;   // resolved forward output plane
    int n_optical = 0;
    int stop_index = -1;   // index among ALL surfaces, -1 if none
    mutable std::mutex mu;
    mutable std::map<std::pair<uint64_t, int>, std::shared_ptr<plt::CompiledPath>> cache;
};

struct plt_map {
    uint32_t direction = 0;
    uint64_t path_id = 0;
    bool has_plane = false;   // blob version >= 2: the input plane the map was trained on
    double plane_z = 0;       // (eval_map rejects rays on any other plane)
    plt::MapLayout layout{};
    plt::MapParams params{};
    std::vector<uint8_t> image;            // packed host weight image (layout.total_bytes)
    mutable std::mutex mu;
    mutable std::map<int, void*> dev_image;  // device ordinal -> device copy (lazy)
    ~plt_map();
};

namespace plt {

plt_lens* parse_lens(const char* text, size_t len, const plt_lens_opts* opts);  // throws Error
void lens_abcd(const plt_lens& L, double lambda_nm, double M[4]);
void lens_pupils(const plt_lens& L, double lambda_nm, double out[4]);   // z_ent, r_ent, z_exit, r_exit
std::shared_ptr<CompiledPath> compile_path(const plt_lens& L, uint64_t path_id, int dir);  // throws
std::vector<std::pair<uint64_t, std::pair<int, int>>> enumerate_ghosts(const plt_lens& L, int max_bounces,
                                                                       double min_throughput);
plt_map* parse_map(const plt_lens* lens, const uint8_t* blob, size_t len);  // throws Error

}  // namespace plt
