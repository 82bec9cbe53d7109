/*
 * oracle.c -- plain, slow, float64 CPU oracle of the per-ray lens transport query.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path (paper_2605_04017_b200/).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * O1..O13 / A1..A30 = SURVEY.md §8(c) steps and readings (restated in DESIGN.md).
 *
 *   orc_glass_index  O1   glass index n(lambda)      (paper silent)
 *   orc_trace        O2-O8 composite operator T^P = S_K o ... o S_1 (Eq. 5-7)
 *                          validity: output iff sigma_{K+1} is the output plane
 *   orc_map_eval     O9-O10 factorised network {y} = f(x) if g(x)=1 else {},
 *                          tanh MLP, symmetry canonicalisation (Eq. 10)
 *   orc_splat        O11  film[c][iy][ix] += I*|w_z|*scale (Eq. 8; Listing 1)
 *
 * Everything is written in the order the paper/SURVEY state it; no blocking,
 * fusion or re-ordering.  Arithmetic is IEEE double, no fast-math.
 */
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* O1 glass index (lambda in nm).                                            */
/* model 0: constant n                     c = {n}                            */
/* model 1: Cauchy  n = A + B/l^2 + C/l^4  c = {A, B[um^2], C[um^4]}  */
/* model 2: Abbe    (n_d, V_d) -> Cauchy A + B/l^2 with                       */
/*          B = (n_d-1) / (V_d (l_F^-2 - l_C^-2)),  A = n_d - B / l_d^2       */
/* model 3: Sellmeier n^2 = 1 + sum B_i l^2/(l^2 - C_i)  c = {B1..3, C1..3}   */
/* ------------------------------------------------------------------------- */
double orc_glass_index(int model, const double* c, double lambda_nm)
{
    const double l = lambda_nm * 1e-3; /* micrometres */
    const double l2 = l * l;
    if (model == 0) return c[0];
    if (model == 1) return c[0] + c[1] / l2 + c[2] / (l2 * l2);
    if (model == 2) {
        const double lF = 0.4861327, lC = 0.6562725, ld = 0.5875618;
        const double B = (c[0] - 1.0) / (c[1] * (1.0 / (lF * lF) - 1.0 / (lC * lC)));
        const double A = c[0] - B / (ld * ld);
        return A + B / l2;
    }
    if (model == 3) {
        double n2 = 1.0;
        for (int i = 0; i < 3; ++i) n2 += c[i] * l2 / (l2 - c[3 + i]);
        return sqrt(n2);
    }
    return NAN;
}

/* Surface record (flat double array, stride ORC_STRIDE):                     */
/*  [0] z vertex  [1] R signed (0 = plane)  [2] a clear semi-aperture          */
/*  [3] is_stop   [4] glass-before model  [5..10] coeffs                       */
/*  [11] glass-after model  [12..17] coeffs                                    */
/*  [18] is_asph  [19] conic k  [20..23] A4, A6, A8, A10 (even asphere)        */
/*  [24] coating index n_c (0 = bare)  [25] coating thickness d (um)          */
#define ORC_STRIDE 26

/* Lens-level parameters: [0] housing radius (0 = none) [1] z of output plane  */
/* [2] rect W (0 = none) [3] rect H [4] rect cx [5] rect cy                    */

#define EPS_T 1e-6 /* self-hit epsilon, mm */

static inline double dot3(const double* a, const double* b)
{
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* Even asphere: sag(rho) = c rho^2 / (1 + sqrt(q))          */
/* + A4 rho^4 + A6 rho^6 + A8 rho^8 + A10 rho^10 with q = 1 - (1 + k) c^2 rho^2, and      */
/* g = (d sag / d rho) / rho = c / sqrt(q) + 4 A4 rho^2 + 6 A6 rho^4 + 8 A8 rho^6 + 10 A10 rho^8. */
/* Returns 0 outside the conic's domain (q < 0).                                          */
static int asph_sag(const double* f, double c, double r2, double* sag, double* g, double* q_out)
{
    const double k = f[19], A4 = f[20], A6 = f[21], A8 = f[22], A10 = f[23];
    const double q = 1.0 - (1.0 + k) * c * c * r2;
    *q_out = q;
    if (q < 0.0) return 0;
    const double sq = sqrt(q);
    *sag = c * r2 / (1.0 + sq) + A4 * r2 * r2 + A6 * r2 * r2 * r2 + A8 * r2 * r2 * r2 * r2 +
           A10 * r2 * r2 * r2 * r2 * r2;
    *g = c / sq + 4.0 * A4 * r2 + 6.0 * A6 * r2 * r2 + 8.0 * A8 * r2 * r2 * r2 + 10.0 * A10 * r2 * r2 * r2 * r2;
    return 1;
}

/*
 * Trace one ray along path id (forward sense: the ray travels +z at entry).
 * Returns 1 if valid.  Margins: m[0] geometric edge margin (mm), m[1] min |kappa|
 * (TIR discriminant), m[2] min sphere discriminant (mm^2), m[3] min |w_z|.
 */
static int trace_one(const double* S, int n_surf, const double* L, uint64_t path_id,
                     double ox, double oy, double oz, double dx, double dy, double dz,
                     double lambda, double out[6], double m[4], int* steps)
{
    /* O2 path decoding: K = floor(log2 id); interaction k is R <=> bit k-1 set. */
    int K = 63;
    while (K > 0 && !((path_id >> K) & 1ull)) --K;

    double o[3] = {ox, oy, oz};
    double nrm = sqrt(dx * dx + dy * dy + dz * dz);
    double w[3] = {dx / nrm, dy / nrm, dz / nrm};
    double I = 1.0, ncur = 1.0;
    int s = 0, dir = +1, k = 0;
    m[0] = INFINITY; m[1] = INFINITY; m[2] = INFINITY; m[3] = INFINITY;

    /* O3 state machine: loop while the ray is inside the surface list.  *steps counts the
       surface steps begun (stop crossings included) plus 1 for the output plane, i.e. how
       much of the path's work the ray needed before it terminated (bookkeeping only). */
    *steps = 0;
    while (s >= 0 && s < n_surf) {
        ++*steps;
        const double* f = S + (size_t)s * ORC_STRIDE;
        const double zs = f[0], R = f[1], a = f[2];
        const int is_stop = f[3] != 0.0;

        /* O4 direction sanity */
        if (fabs(w[2]) < m[3]) m[3] = fabs(w[2]);
        if (!(w[2] * dir > 0.0)) return 0;

        /* O5 intersection, vertex-local */
        const double lx = o[0], ly = o[1], lz = o[2] - zs;
        const int asph = !is_stop && f[18] != 0.0;
        double t, ga = 0.0;   /* asphere: g at the hit */
        if (asph) {
            /* Newton on F(t) = (lz + t wz) - sag(rho(t)), F'(t) = wz - g (x wx + y wy), from the
               tangent plane z = vertex (the plain algorithm; no base-sphere shortcut). */
            const double c = (R == 0.0) ? 0.0 : 1.0 / R;
            t = -lz / w[2];
            int ok = 0;
            double Fp = 0.0;
            for (int it = 0; it < 100; ++it) {
                const double x = lx + t * w[0], y = ly + t * w[1], z = lz + t * w[2];
                double sag, g, q;
                if (!asph_sag(f, c, x * x + y * y, &sag, &g, &q)) return 0;
                const double F = z - sag;
                Fp = w[2] - g * (x * w[0] + y * w[1]);
                if (Fp == 0.0) return 0;
                const double dt = F / Fp;
                t -= dt;
                if (fabs(dt) <= 1e-14 * (1.0 + fabs(t))) { ok = 1; break; }
            }
            if (!ok) return 0;
            if (fabs(Fp) < m[2]) m[2] = fabs(Fp);      /* grazing hit (double root) margin */
            {
                const double x = lx + t * w[0], y = ly + t * w[1];
                double sag, q;
                if (!asph_sag(f, c, x * x + y * y, &sag, &ga, &q)) return 0;
            }
        } else if (R == 0.0 || is_stop) {
            t = -lz / w[2];
        } else {
            const double b = lx * w[0] + ly * w[1] + (lz - R) * w[2];
            const double c = lx * lx + ly * ly + lz * (lz - 2.0 * R);
            const double disc = b * b - c;
            if (fabs(disc) < m[2]) m[2] = fabs(disc);
            if (disc < 0.0) return 0;
            const double sq = sqrt(disc);
            const double q = (b >= 0.0) ? (-b - sq) : (-b + sq);
            if (q == 0.0) return 0;
            const double t0 = q, t1 = c / q;
            const int use_closer = (w[2] > 0.0) != (R < 0.0); /* pbrt cap rule */
            t = use_closer ? fmin(t0, t1) : fmax(t0, t1);
        }
        if (!(t > EPS_T)) return 0;
        const double h[3] = {o[0] + t * w[0], o[1] + t * w[1], o[2] + t * w[2]};

        /* O6 aperture (clear semi-aperture; optional housing cylinder, endpoint test) */
        const double rho = sqrt(h[0] * h[0] + h[1] * h[1]);
        if (fabs(rho - a) < m[0]) m[0] = fabs(rho - a);
        if (rho > a) return 0;
        if (L[0] > 0.0) {
            if (fabs(rho - L[0]) < m[0]) m[0] = fabs(rho - L[0]);
            if (rho > L[0]) return 0;
        }
        o[0] = h[0]; o[1] = h[1]; o[2] = h[2];

        if (is_stop) { s += dir; continue; }  /* the stop is not an interaction */

        /* O7 interaction k+1 */
        if (k >= K) return 0;              /* sequence exhausted: sigma_{K+1} not the output plane */
        const int is_R = (int)((path_id >> k) & 1ull);
        double nv[3];
        if (asph) {   /* gradient of z - sag(rho): (-g x, -g y, 1), normalised */
            const double nn = sqrt(ga * ga * (h[0] * h[0] + h[1] * h[1]) + 1.0);
            nv[0] = -ga * h[0] / nn; nv[1] = -ga * h[1] / nn; nv[2] = 1.0 / nn;
        } else if (R == 0.0) { nv[0] = 0.0; nv[1] = 0.0; nv[2] = 1.0; }
        else { nv[0] = h[0] / R; nv[1] = h[1] / R; nv[2] = (h[2] - zs - R) / R; }
        if (dot3(nv, w) > 0.0) { nv[0] = -nv[0]; nv[1] = -nv[1]; nv[2] = -nv[2]; }
        const double cosi = -dot3(nv, w);
        const double n1 = ncur;
        const double n2 = (dir > 0) ? orc_glass_index((int)f[11], f + 12, lambda)
                                    : orc_glass_index((int)f[4], f + 5, lambda);
        const double eta = n1 / n2;
        const double kappa = 1.0 - eta * eta * (1.0 - cosi * cosi);
        if (fabs(kappa) < m[1]) m[1] = fabs(kappa);
        double Rf, cost = 0.0;
        if (kappa < 0.0) {
            Rf = 1.0;  /* total internal reflection */
        } else if (f[24] > 0.0) {
            /* single thin film n_c, d between n1 and n2: amplitude      */
            /* coefficients r_1c, r_c2 per polarisation and the film phase 2 beta =           */
            /* 4 pi n_c d cos_c / lambda give R = (a^2 + b^2 + 2ab cos 2beta) /                */
            /* (1 + a^2 b^2 + 2ab cos 2beta) (Airy summation, lossless film)                  */
            cost = sqrt(kappa);
            const double nc = f[24], d = f[25], lam_um = lambda * 1e-3;
            const double sc2 = (n1 / nc) * (n1 / nc) * (1.0 - cosi * cosi);
            const double cosc = sqrt(fmax(0.0, 1.0 - sc2));
            const double cb = cos(4.0 * M_PI * nc * d * cosc / lam_um);
            const double as = (n1 * cosi - nc * cosc) / (n1 * cosi + nc * cosc);
            const double bs = (nc * cosc - n2 * cost) / (nc * cosc + n2 * cost);
            const double ap = (nc * cosi - n1 * cosc) / (nc * cosi + n1 * cosc);
            const double bp = (n2 * cosc - nc * cost) / (n2 * cosc + nc * cost);
            const double Rs = (as * as + bs * bs + 2.0 * as * bs * cb) / (1.0 + as * as * bs * bs + 2.0 * as * bs * cb);
            const double Rp = (ap * ap + bp * bp + 2.0 * ap * bp * cb) / (1.0 + ap * ap * bp * bp + 2.0 * ap * bp * cb);
            Rf = 0.5 * (Rs + Rp);
        } else {
            cost = sqrt(kappa);
            const double rs = (n1 * cosi - n2 * cost) / (n1 * cosi + n2 * cost);
            const double rp = (n2 * cosi - n1 * cost) / (n2 * cosi + n1 * cost);
            Rf = 0.5 * (rs * rs + rp * rp);  /* unpolarised */
        }
        if (!is_R) {
            if (kappa < 0.0) return 0;     /* TIR on a T step absorbs */
            const double g = eta * cosi - cost;
            w[0] = eta * w[0] + g * nv[0];
            w[1] = eta * w[1] + g * nv[1];
            w[2] = eta * w[2] + g * nv[2];
            I *= (1.0 - Rf);
            ncur = n2;
        } else {
            const double wn = dot3(w, nv);
            w[0] = w[0] - 2.0 * wn * nv[0];
            w[1] = w[1] - 2.0 * wn * nv[1];
            w[2] = w[2] - 2.0 * wn * nv[2];
            I *= Rf;
            dir = -dir;
        }
        ++k;
        s += dir;
    }
    if (dir < 0) return 0;                 /* left through the front */
    if (k != K) return 0;                  /* sequence not fully consumed */

    /* O8 output plane */
    ++*steps;
    if (fabs(w[2]) < m[3]) m[3] = fabs(w[2]);
    if (!(w[2] > 0.0)) return 0;
    const double t = (L[1] - o[2]) / w[2];
    if (!(t > 0.0)) return 0;
    const double px = o[0] + t * w[0], py = o[1] + t * w[1];
    if (L[2] > 0.0) {
        const double ex = fabs(px - L[4]) - 0.5 * L[2];
        const double ey = fabs(py - L[5]) - 0.5 * L[3];
        if (fabs(ex) < m[0]) m[0] = fabs(ex);
        if (fabs(ey) < m[0]) m[0] = fabs(ey);
        if (ex > 0.0 || ey > 0.0) return 0;
    }
    out[0] = px; out[1] = py; out[2] = w[0]; out[3] = w[1]; out[4] = w[2]; out[5] = I;
    return 1;
}

/* Batched entry point over [0, n).  Inputs are the float32 rays widened to double by the
   caller (or exact doubles in tests).  Invalid rays get zero outputs. */
void orc_trace(const double* S, int n_surf, const double* L, uint64_t path_id,
               int64_t n, const double* ox, const double* oy, double plane_z,
               const double* dx, const double* dy, const double* dz, const double* lambda_nm,
               uint8_t* valid, double* out /* n x 6 */, double* margins /* n x 4 */,
               int32_t* steps /* n, nullable: steps begun before termination */)
{
    for (int64_t i = 0; i < n; ++i) {
        double o6[6] = {0, 0, 0, 0, 0, 0}, m4[4];
        int st = 0;
        int v = trace_one(S, n_surf, L, path_id, ox[i], oy[i], plane_z,
                          dx[i], dy[i], dz[i], lambda_nm[i], o6, m4, &st);
        if (steps) steps[i] = st;
        valid[i] = (uint8_t)v;
        if (!v) memset(o6, 0, sizeof o6);
        memcpy(out + 6 * i, o6, sizeof o6);
        memcpy(margins + 4 * i, m4, sizeof m4);
    }
}

/* ------------------------------------------------------------------------- */
/* O9 MLP forward: h0 = x; h_l = tanh(W_l h_{l-1} + b_l); y = W_{L+1} h_L + b   */
/* Weights are given as doubles (the bf16 values of the blob widened).        */
/* dims[0..nl] ; W concatenated row-major per layer; b concatenated.          */
/* ------------------------------------------------------------------------- */
static void mlp_forward(int nl, const int* dims, const double* W, const double* B,
                        const double* x, double* y)
{
    double cur[64], nxt[64];
    for (int i = 0; i < dims[0]; ++i) cur[i] = x[i];
    size_t wo = 0, bo = 0;
    for (int l = 0; l < nl; ++l) {
        const int fi = dims[l], fo = dims[l + 1];
        for (int o = 0; o < fo; ++o) {
            double acc = B[bo + o];
            for (int i = 0; i < fi; ++i) acc += W[wo + (size_t)o * fi + i] * cur[i];
            nxt[o] = (l + 1 < nl) ? tanh(acc) : acc;   /* tanh hidden, linear output */
        }
        wo += (size_t)fi * fo;
        bo += fo;
        for (int o = 0; o < fo; ++o) cur[o] = nxt[o];
    }
    for (int o = 0; o < dims[nl]; ++o) y[o] = cur[o];
}

void orc_mlp_forward(int nl, const int* dims, const double* W, const double* B,
                     int64_t n, const double* x /* n x dims[0] */, double* y /* n x dims[nl] */)
{
    for (int64_t i = 0; i < n; ++i)
        mlp_forward(nl, dims, W, B, x + (size_t)i * dims[0], y + (size_t)i * dims[nl]);
}

/* ------------------------------------------------------------------------- */
/* O10 map wrapper: canonicalise (Eq. 10) -> normalise -> classifier */
/* g; valid <=> logit >= 0 -> regressor f (only if valid) ->        */
/* de-normalise -> undo reflection, rotate back -> w unit, I clamped.   */
/* norm = in_lo[4], in_hi[4], out_mid[6], out_half[6].                          */
/* raw (nullable) = n x 7: logit, y[6] (regressor raw outputs, 0 if invalid).   */
/* ------------------------------------------------------------------------- */
void orc_map_eval(int ncl, const int* cdims, const double* cW, const double* cB,
                  int nrl, const int* rdims, const double* rW, const double* rB,
                  const double* norm, int64_t n,
                  const double* ox, const double* oy, const double* dx, const double* dy,
                  const double* dz, const double* lambda_nm,
                  uint8_t* valid, double* out /* n x 6 */, double* raw /* n x 7 or NULL */)
{
    const double *lo = norm, *hi = norm + 4, *mid = norm + 8, *half = norm + 14;
    for (int64_t i = 0; i < n; ++i) {
        const double px = ox[i], py = oy[i], wx = dx[i], wy = dy[i], wz = dz[i];
        /* canonicalise: rotate p onto +x, reflect so w'_y >= 0 */
        const double r = sqrt(px * px + py * py);
        double c, s;
        if (r > 0.0) { c = px / r; s = py / r; }
        else {
            const double phi = (wx == 0.0 && wy == 0.0) ? 0.0 : atan2(wy, wx);
            c = cos(phi); s = sin(phi);
        }
        double wpx = c * wx + s * wy;
        double wpy = -s * wx + c * wy;
        const int flip = wpy < 0.0;
        if (flip) wpy = -wpy;
        const double xin[4] = {r, wpx, wpy, lambda_nm[i]};
        double xh[4];
        for (int d = 0; d < 4; ++d) {
            double v = 2.0 * (xin[d] - lo[d]) / (hi[d] - lo[d]) - 1.0;
            xh[d] = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        }
        double logit;
        mlp_forward(ncl, cdims, cW, cB, xh, &logit);
        double o6[6] = {0, 0, 0, 0, 0, 0}, y[6] = {0, 0, 0, 0, 0, 0};
        const int v = logit >= 0.0;
        if (v) {
            mlp_forward(nrl, rdims, rW, rB, xh, y);
            double q[6];
            for (int d = 0; d < 6; ++d) q[d] = mid[d] + half[d] * y[d];
            if (flip) { q[1] = -q[1]; q[3] = -q[3]; }
            o6[0] = c * q[0] - s * q[1];
            o6[1] = s * q[0] + c * q[1];
            double ox_ = c * q[2] - s * q[3], oy_ = s * q[2] + c * q[3], oz_ = q[4];
            const double wn = sqrt(ox_ * ox_ + oy_ * oy_ + oz_ * oz_);
            o6[2] = ox_ / wn; o6[3] = oy_ / wn; o6[4] = oz_ / wn;
            o6[5] = q[5] < 0.0 ? 0.0 : (q[5] > 1.0 ? 1.0 : q[5]);
        }
        valid[i] = (uint8_t)v;
        memcpy(out + 6 * i, o6, sizeof o6);
        if (raw) {
            raw[7 * i] = logit;
            for (int d = 0; d < 6; ++d) raw[7 * i + 1 + d] = y[d];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O11 splat: ix = floor((p_x - c_x + W/2)/W * width),                          */
/*            iy = floor((H/2 - (p_y - c_y))/H * height)  (row 0 at +y);         */
/* film[c][iy][ix] += llrint(I * |w_z| * scale * 2^32) (int64 fixed point).     */
/* Invalid or off-film hits are skipped and counted.                            */
/* ------------------------------------------------------------------------- */
int64_t orc_splat(int width, int height, int channels, double W, double H, double cx, double cy,
                  int64_t* film, int64_t n, const uint8_t* valid, const float* px, const float* py,
                  const float* dz, const float* I, const uint8_t* channel, float scale)
{
    int64_t dropped = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        const double fx = ((double)px[i] - cx + W / 2.0) / W * (double)width;
        const double fy = (H / 2.0 - ((double)py[i] - cy)) / H * (double)height;
        const double fxf = floor(fx), fyf = floor(fy);
        if (!(fxf >= 0.0 && fxf < (double)width && fyf >= 0.0 && fyf < (double)height)) { ++dropped; continue; }
        const int c = channel ? (int)channel[i] : 0;
        if (c < 0 || c >= channels) { ++dropped; continue; }
        const double wgt = (double)I[i] * fabs((double)dz[i]) * (double)scale * 4294967296.0;
        film[((int64_t)c * height + (int64_t)fyf) * width + (int64_t)fxf] += llrint(wgt);
    }
    return dropped;
}

/* ------------------------------------------------------------------------- */
/* O14 backward camera integrand with a procedural checkerboard scene plane   */
/* (Eq. 9): exit ray (origin on z = z_hits,   */
/* direction w) continues to z = z_scene; L = 1 on even squares, contrast on  */
/* odd ones; film[i / spp] += llrint(I * L * scale * 2^32).                   */
/* ------------------------------------------------------------------------- */
void orc_shade_plane(double z_scene, double period, double contrast, double z_hits, int spp, int64_t pixels,
                     float scale, int64_t* film, int64_t n, const uint8_t* valid, const float* px, const float* py,
                     const float* dx, const float* dy, const float* dz, const float* I, const float* in_dz)
{
    /* in_dz (nullable): z-components of the SENSOR rays; when given, each contribution is
     * weighted by cos^4(theta) = (w_z^2)^2, the Monte-Carlo weight of directions drawn
     * through uniform points on a disc parallel to the sensor (Eq. 9 with the pdf
     * dz^2 / (A cos^3 theta); A / dz^2 is the caller's scale). */
    for (int64_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        const double t = (z_scene - z_hits) / (double)dz[i];
        const int64_t pix = i / spp;
        if (!(t > 0.0) || pix >= pixels) continue;
        const double x = (double)px[i] + t * (double)dx[i];
        const double y = (double)py[i] + t * (double)dy[i];
        const int64_t q = (int64_t)floor(x / period) + (int64_t)floor(y / period);
        const double L = (q & 1) ? contrast : 1.0;
        double IL = (double)I[i] * L;
        if (in_dz) { const double c = (double)in_dz[i], c2 = c * c; IL = IL * (c2 * c2); }
        film[pix] += llrint(IL * (double)scale * 4294967296.0);
    }
}

/* ------------------------------------------------------------------------- */
/* O14b scene cards (scenes beyond one plane): the ray     */
/* takes the radiance of the first card it meets -- smallest t = (z_k - z_hits) */
/* / w_z > 0 with the hit inside the card's rectangle (ties: lower k) -- else   */
/* `background`; cards[7k..7k+6] = z, period, contrast, x0, x1, y0, y1.  The    */
/* pupil weight as orc_shade_plane.                                            */
/* ------------------------------------------------------------------------- */
void orc_shade_cards(const double* cards, int n_cards, double background, double z_hits, int spp, int64_t pixels,
                     float scale, int64_t* film, int64_t n, const uint8_t* valid, const float* px, const float* py,
                     const float* dx, const float* dy, const float* dz, const float* I, const float* in_dz)
{
    for (int64_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        const int64_t pix = i / spp;
        if (pix >= pixels) continue;
        double L = background, best = 0.0;
        int found = 0;
        for (int k = 0; k < n_cards; ++k) {
            const double* c = cards + 7 * k;
            const double t = (c[0] - z_hits) / (double)dz[i];
            if (!(t > 0.0) || (found && !(t < best))) continue;
            const double x = (double)px[i] + t * (double)dx[i];
            const double y = (double)py[i] + t * (double)dy[i];
            if (x < c[3] || x > c[4] || y < c[5] || y > c[6]) continue;
            const int64_t q = (int64_t)floor(x / c[1]) + (int64_t)floor(y / c[1]);
            L = (q & 1) ? c[2] : 1.0;
            best = t;
            found = 1;
        }
        double IL = (double)I[i] * L;
        if (in_dz) { const double cz = (double)in_dz[i], c2 = cz * cz; IL = IL * (c2 * c2); }
        film[pix] += llrint(IL * (double)scale * 4294967296.0);
    }
}
