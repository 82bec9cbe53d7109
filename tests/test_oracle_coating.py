"""Pins of the oracle's single-layer anti-reflection coating: the
ideal quarter wave (n_c = sqrt(n), lambda = lambda0, normal incidence) reflects nothing,
a vanishing film and a half-wave (absentee) film reproduce the bare surface, and at
oblique incidence the Airy formula equals an independent characteristic-matrix (transfer
matrix) computation for s and p.  CPU only."""
import math

import numpy as np

import oracle

N = 1.5
LAM = 550.0


def slab(coat=None):
    tok = f" coat:{coat[0]!r},{coat[1]!r}" if coat else ""
    return f"name slab\n0 2.0 n:{N} 40{tok}\n0 0.0 air 40{tok}\n"


def ray(theta_deg, lam=LAM):
    t = math.radians(theta_deg)
    return {"ox": np.zeros(1), "oy": np.zeros(1), "dx": np.array([math.sin(t)]), "dy": np.zeros(1),
            "dz": np.array([math.cos(t)]), "lambda_nm": np.array([lam]), "plane_z": -5.0}


def throughput(text, theta=0.0, lam=LAM):
    lens = oracle.load_lens(text, {"sensor_z_mm": 10.0})
    t = oracle.trace(lens, 1 << 2, 0, ray(theta, lam))
    assert t["valid"][0]
    return float(t["I"][0])


def test_ideal_quarter_wave_transmits_everything():
    assert abs(throughput(slab((math.sqrt(N), LAM))) - 1.0) < 1e-15


def test_vanishing_and_absentee_films_are_the_bare_surface():
    bare = throughput(slab())
    assert abs(bare - (1 - ((N - 1) / (N + 1)) ** 2) ** 2) < 1e-15
    assert abs(throughput(slab((1.38, 1e-9))) - bare) < 1e-12          # d ~ 0
    assert abs(throughput(slab((1.38, 2 * LAM)), lam=LAM) - bare) < 1e-12  # d = lambda/(2 n_c): half wave


def _tmm_R(n1, nc, n2, d_um, lam_um, theta1):
    """Independent characteristic-matrix reflectance of one film, s and p averaged."""
    s1 = n1 * math.sin(theta1)
    c1 = math.cos(theta1)
    cc = np.sqrt(1 - (s1 / nc) ** 2 + 0j)
    c2 = np.sqrt(1 - (s1 / n2) ** 2 + 0j)
    delta = 2 * math.pi * nc * d_um * cc / lam_um
    out = []
    for pol in ("s", "p"):
        eta = (lambda n, c: n * c) if pol == "s" else (lambda n, c: n / c)
        e1, ec, e2 = eta(n1, c1), eta(nc, cc), eta(n2, c2)
        M = np.array([[np.cos(delta), 1j * np.sin(delta) / ec], [1j * ec * np.sin(delta), np.cos(delta)]])
        B, Cc = M @ np.array([1.0, e2])
        r = (e1 * B - Cc) / (e1 * B + Cc)
        out.append(abs(r) ** 2)
    return 0.5 * sum(out)


def test_oblique_film_matches_the_transfer_matrix():
    nc, lam0 = 1.38, 500.0
    d_um = lam0 * 1e-3 / (4 * nc)
    for theta in (0.0, 20.0, 35.0, 50.0):
        t = math.radians(theta)
        R1 = _tmm_R(1.0, nc, N, d_um, LAM * 1e-3, t)                     # air -> glass, through the film
        t2 = math.asin(math.sin(t) / N)
        R2 = _tmm_R(N, nc, 1.0, d_um, LAM * 1e-3, t2)                    # glass -> air, through the film
        assert abs(throughput(slab((nc, lam0)), theta) - (1 - R1) * (1 - R2)) < 1e-13
