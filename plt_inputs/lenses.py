"""Lens prescriptions used as synthetic inputs.

This module holds DATA only: prescription text in the repo's line-oriented
``.lens`` format and a text-level length scaler.  It performs none of the
method's arithmetic (no glass evaluation, no tracing, no paraxial optics);
both the float64 oracle (``oracle/``) and the CUDA library parse the text
independently.

The paper does not publish its prescriptions (fig:path-tracing
header names "Wide-angle 22mm lens. Nakamura.", "24mm lens. Canon", "59mm lens.
Optical Designer").  The stand-ins are the public Kolb/pbrt tables recalled in
SURVEY.md Appendix A (A.1 double-Gauss 50 mm, A.2 Nakamura 22 mm) and the
scaled variants of A.3.

Format (one surface per line, front to back; ``#`` starts a comment)::

    name <identifier>
    <radius_mm> <thickness_mm> <glass> <aperture_diameter_mm>

``glass`` is the medium AFTER the surface: ``air`` | ``stop`` |
``n:<n>`` (constant index) | ``abbe:<n_d>,<V_d>`` | ``cauchy:<A>,<B>,<C>``
(B in um^2, C in um^4) | ``sellmeier:<B1>,<B2>,<B3>,<C1>,<C2>,<C3>`` (C in um^2).
A bare numeric Kolb row ``radius thickness n_d aperture [V_d]`` is also
accepted (n_d = 0 -> stop, n_d = 1 -> air, V_d present -> Abbe glass).
A radius of 0 means a planar surface.  The stop is planar by definition.
"""

SINGLET = """\
# C1: N-BK7 equiconvex singlet behind a front stop (SURVEY.md A.3, config C1)
name singlet_nbk7
0       5.0   stop                                                                 16.0
50.0    5.0   sellmeier:1.03961212,0.231792344,1.01046945,0.00600069867,0.0200179144,103.560653  25.0
-50.0   0.0   air                                                                  25.0
"""

# Kolb, Mitchell & Hanrahan 1995 Table 1 scaled x0.5 (pbrt-v3 dgauss.50mm)
DGAUSS50 = """\
# double-Gauss 50 mm (SURVEY.md Appendix A.1); glass = Abbe (n_d, V_d)
name dgauss50
29.475   3.76   abbe:1.670,47.1  25.2
84.83    0.12   air              25.2
19.275   4.025  abbe:1.670,47.1  23.0
40.77    3.275  abbe:1.699,30.1  23.0
12.75    5.705  air              18.0
0        4.5    stop             17.1
-14.495  1.18   abbe:1.603,38.0  17.0
40.77    6.065  abbe:1.658,57.3  20.0
-20.385  0.19   air              20.0
437.065  3.22   abbe:1.717,48.0  20.0
-39.73   0.0    air              20.0
"""

# pbrt-v3 wide.22mm (Nakamura); V_d assumed per glass as listed there
WIDE22 = """\
# wide-angle 22 mm "Nakamura" (SURVEY.md Appendix A.2); glass = Abbe (n_d, V_d)
name wide22
35.98738   1.21638  abbe:1.54,59.7    23.716
11.69718   9.9957   air               17.996
13.08714   5.12622  abbe:1.772,49.6   12.364
-22.63294  1.76924  abbe:1.617,54.0    9.812
71.05802   0.8184   air                9.152
0          2.27766  stop               8.756
-9.58584   2.43254  abbe:1.617,54.0    8.184
-11.28864  0.11506  air                9.152
-166.7765  3.09606  abbe:1.713,53.8   10.648
-7.5911    1.32682  abbe:1.805,25.4   11.44
-16.7662   3.98068  air               12.276
-7.70286   1.21638  abbe:1.617,54.0   13.42
-11.97328  0.0      air               17.996
"""


def scale_lens_text(text: str, s: float, name: str) -> str:
    """Scale every length column (radius, thickness, aperture) of a .lens text by ``s``.

    Pure text/data manipulation used to build the SURVEY.md A.3 stand-ins
    (24 mm = A.2 x 1.08974, 59 mm = A.1 x 1.17161); glass columns untouched.
    """
    out = []
    for line in text.splitlines():
        body = line.split("#", 1)[0].strip()
        if not body:
            out.append(line)
            continue
        tok = body.split()
        if tok[0] == "name":
            out.append(f"name {name}")
            continue
        r, t, g, d = float(tok[0]), float(tok[1]), tok[2], float(tok[3])
        out.append(f"{r * s!r} {t * s!r} {g} {d * s!r}")
    return "\n".join(out) + "\n"


WIDE24 = scale_lens_text(WIDE22, 1.08974, "wide24")      # SURVEY.md A.3 (EFL ~24.000 mm)
DGAUSS59 = scale_lens_text(DGAUSS50, 1.17161, "dgauss59")  # SURVEY.md A.3 (EFL ~59.000 mm)

LENSES = {
    "singlet": SINGLET,
    "dgauss50": DGAUSS50,
    "wide22": WIDE22,
    "wide24": WIDE24,
    "dgauss59": DGAUSS59,
}


def random_lens_text(seed: int) -> tuple:
    """A seeded random air-spaced lens for fuzz parity tests: 2-3 elements, each a singlet
    or a cemented doublet, a stop between two of them; radii |R| in [25, 150] mm of either
    sign, clear semi-apertures <= 0.55 |R| (so every cap is a proper spherical cap), glass
    2-6 mm, air 0.5-5 mm; glasses Abbe (n_d 1.48-1.85, V_d 25-65), Cauchy or the N-BK7
    Sellmeier.  Returns (text, front semi-aperture mm, z of the last vertex mm).  DATA only:
    no optics is evaluated here."""
    import numpy as np
    rng = np.random.default_rng([int(seed), 0x1E75])
    bk7 = "sellmeier:1.03961212,0.231792344,1.01046945,0.00600069867,0.0200179144,103.560653"

    def glass():
        k = rng.integers(0, 3)
        if k == 0:
            return f"abbe:{rng.uniform(1.48, 1.85):.4f},{rng.uniform(25, 65):.1f}"
        if k == 1:
            return f"cauchy:{rng.uniform(1.45, 1.75):.4f},{rng.uniform(0.003, 0.012):.5f},0"
        return bk7

    semi = float(rng.uniform(6.0, 11.0))
    rows, z = [], 0.0
    n_el = int(rng.integers(2, 4))
    stop_after = int(rng.integers(0, n_el - 1))
    for e in range(n_el):
        n_surf = 2 if rng.random() < 0.6 else 3            # singlet or cemented doublet
        for s in range(n_surf):
            R = float(rng.uniform(25.0, 150.0)) * (1 if rng.random() < 0.5 else -1)
            R = max(abs(R), semi / 0.55) * np.sign(R)
            last = s == n_surf - 1
            if last:
                t, g = float(rng.uniform(0.5, 5.0)), "air"
            else:
                t, g = float(rng.uniform(2.0, 6.0)), glass()
            rows.append([R, t, g, 2.0 * semi])
        if e == stop_after:
            rows.append([0.0, float(rng.uniform(1.0, 4.0)), "stop", 2.0 * semi * 0.8])
    rows[-1][1] = 0.0
    for r in rows[:-1]:
        z += r[1]
    text = "name fuzz_%d\n" % seed + "".join(f"{r[0]:.4f} {r[1]:.4f} {r[2]} {r[3]:.4f}\n" for r in rows)
    return text, semi, z
