// gen_rays.cu -- counter-based synthetic rays on the device (plt_gen_rays).
//
// The workloads of BASELINE.json (C3: 805 M camera rays at the 32768-spp scale, C5: up to
// 2^30 rays) are generated where they are consumed: ray i of a batch is a pure function
// of (seed, i) -- Philox4x32-10 (Salmon et al., SC'11) keyed by the seed, counted by the
// global ray index -- so a batch of any size is produced in HBM at memory speed, sharded
// over ranks without any scatter, and any sample of it can be regenerated on the host.
// The specification (plt.h, plt_inputs/philox.py) fixes every double operation and its
// order; the kernel spells each one with an explicit round-to-nearest intrinsic so no
// fused multiply-add changes a bit, and the float32 rays equal the host generator's.
#include <cuda_runtime.h>
#include <cstdint>

#include "plt_internal.h"

namespace plt {

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u, kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
constexpr uint32_t kTag = 0x504C5452u;   // 'PLTR'
constexpr int kThreads = 256;

struct Law {
    int kind, width_px, height_px, spp;
    double plane_z, disc_r, disc_x0, cap_cos_min, dir_x, dir_z, sensor_w, sensor_h, pupil_z, pupil_r;
    double lam_lo, lam_span;   // lambda = lo + span u
    double cell_w, cell_h;     // sensor_grid pixel pitch W / Wpx, H / Hpx
};

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kM0, c[0]), lo0 = kM0 * c[0];
        const uint32_t hi1 = __umulhi(kM1, c[2]), lo1 = kM1 * c[2];
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += kW0; k1 += kW1;   // the bump after the 10th round is unused
    }
}

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// (cos 2 pi u, sin 2 pi u): octant reduction + Taylor polynomials + octant-centre rotation
__device__ __forceinline__ void angle(double u, double& co, double& si) {
    const double t = dm(u, 8.0);
    const double k = floor(t);
    const double th = dm(ds(ds(t, k), 0.5), 0.78539816339744830962);
    const double t2 = dm(th, th);
    double ps = 1.6059043836821614599e-10;
    ps = da(dm(ps, t2), -2.5052108385441718775e-08);
    ps = da(dm(ps, t2), 2.7557319223985890653e-06);
    ps = da(dm(ps, t2), -0.00019841269841269841270);
    ps = da(dm(ps, t2), 0.0083333333333333333333);
    ps = da(dm(ps, t2), -0.16666666666666666667);
    const double s = da(th, dm(dm(th, t2), ps));
    double pc = -1.1470745597729724714e-11;
    pc = da(dm(pc, t2), 2.0876756987868098979e-09);
    pc = da(dm(pc, t2), -2.7557319223985890653e-07);
    pc = da(dm(pc, t2), 2.4801587301587301587e-05);
    pc = da(dm(pc, t2), -0.0013888888888888888889);
    pc = da(dm(pc, t2), 0.041666666666666666667);
    pc = da(dm(pc, t2), -0.5);
    const double c = da(1.0, dm(t2, pc));
    const double A = 0.92387953251128673848, B = 0.38268343236508978178;
    const int ki = (int)k;
    // octant centres (k + 1/2) pi/4
    const double ck = (ki == 0 || ki == 7) ? A : (ki == 1 || ki == 6) ? B : (ki == 2 || ki == 5) ? -B : -A;
    const double sk = (ki == 0 || ki == 3) ? B : (ki == 1 || ki == 2) ? A : (ki == 4 || ki == 7) ? -B : -A;
    co = ds(dm(c, ck), dm(s, sk));
    si = da(dm(s, ck), dm(c, sk));
}

__global__ void __launch_bounds__(kThreads) gen_rays_kernel(const __grid_constant__ Law L, uint32_t k0, uint32_t k1,
                                                            int64_t start, plt_rays out, int64_t n) {
    for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < n; j += (int64_t)gridDim.x * kThreads) {
        const uint64_t i = (uint64_t)(start + j);
        double u[8];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)b, kTag};
            philox(c, k0, k1);
#pragma unroll
            for (int q = 0; q < 4; ++q) u[4 * b + q] = dm(da((double)c[q], 0.5), 2.3283064365386962890625e-10);
        }
        double ox, oy, dx, dy, dz;
        if (L.kind == PLT_LAW_DISC_CAP || L.kind == PLT_LAW_COLLIMATED) {
            const double r = dm(L.disc_r, __dsqrt_rn(u[0]));
            double c, s;
            angle(u[1], c, s);
            ox = da(L.disc_x0, dm(r, c));
            oy = dm(r, s);
            if (L.kind == PLT_LAW_DISC_CAP) {
                const double wz = ds(1.0, dm(u[2], ds(1.0, L.cap_cos_min)));
                const double sz = __dsqrt_rn(fmax(0.0, ds(1.0, dm(wz, wz))));
                double c2, s2;
                angle(u[3], c2, s2);
                dx = dm(sz, c2); dy = dm(sz, s2); dz = wz;
            } else {
                dx = L.dir_x; dy = 0.0; dz = L.dir_z;
            }
        } else {
            if (L.kind == PLT_LAW_SENSOR_PUPIL) {
                ox = dm(ds(u[0], 0.5), L.sensor_w);
                oy = dm(ds(u[1], 0.5), L.sensor_h);
            } else {
                const int64_t pix = (int64_t)(i / (uint64_t)L.spp);
                const double ix = (double)(pix % L.width_px), iy = (double)(pix / L.width_px);
                ox = da(dm(-0.5, L.sensor_w), dm(da(ix, u[0]), L.cell_w));
                oy = ds(dm(0.5, L.sensor_h), dm(da(iy, u[1]), L.cell_h));
            }
            const double r = dm(L.pupil_r, __dsqrt_rn(u[2]));
            double c, s;
            angle(u[3], c, s);
            const double vx = ds(dm(r, c), ox), vy = ds(dm(r, s), oy), vz = ds(L.pupil_z, L.plane_z);
            const double inv = __ddiv_rn(1.0, __dsqrt_rn(da(da(dm(vx, vx), dm(vy, vy)), dm(vz, vz))));
            dx = dm(vx, inv); dy = dm(vy, inv); dz = dm(vz, inv);
        }
        const double lam = da(L.lam_lo, dm(L.lam_span, u[4]));
        const_cast<float*>(out.ox)[j] = __double2float_rn(ox);
        const_cast<float*>(out.oy)[j] = __double2float_rn(oy);
        const_cast<float*>(out.dx)[j] = __double2float_rn(dx);
        const_cast<float*>(out.dy)[j] = __double2float_rn(dy);
        if (out.dz) const_cast<float*>(out.dz)[j] = __double2float_rn(dz);
        const_cast<float*>(out.lambda_nm)[j] = __double2float_rn(lam);
    }
}

}  // namespace

int launch_gen_rays(const plt_ray_law& law, uint64_t seed, int64_t start, const plt_rays& out, int64_t n,
                    void* stream) {
    Law L{};
    L.kind = law.kind;
    L.width_px = law.width_px; L.height_px = law.height_px; L.spp = law.spp;
    L.plane_z = law.plane_z_mm; L.disc_r = law.disc_r_mm; L.disc_x0 = law.disc_x0_mm;
    L.cap_cos_min = law.cap_cos_min; L.dir_x = law.dir_x; L.dir_z = law.dir_z;
    L.sensor_w = law.sensor_w_mm; L.sensor_h = law.sensor_h_mm; L.pupil_z = law.pupil_z_mm; L.pupil_r = law.pupil_r_mm;
    L.lam_lo = law.lambda_lo_nm;
    L.lam_span = law.lambda_hi_nm - law.lambda_lo_nm;   // one rounding, as the host generator
    if (law.kind == PLT_LAW_SENSOR_GRID) {
        L.cell_w = law.sensor_w_mm / law.width_px;
        L.cell_h = law.sensor_h_mm / law.height_px;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sms * 16;   // 16 x 256 threads per SM, grid-stride beyond
    if (blocks > cap) blocks = cap;
    gen_rays_kernel<<<(int)(blocks < 1 ? 1 : blocks), kThreads, 0, (cudaStream_t)stream>>>(
        L, (uint32_t)seed, (uint32_t)(seed >> 32), start, out, n);
    return (int)cudaGetLastError();
}

}  // namespace plt
