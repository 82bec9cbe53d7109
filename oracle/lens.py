"""Oracle-side lens model, paraxial ABCD (O13), path ids (O2) and ghost enumeration (O12).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Independent of the CUDA
library's C++ parser: this file re-reads the same prescription text.

Conventions: mm and nm; +z from object to image side;
surfaces listed front to back, first vertex at z = 0, z_{k+1} = z_k + t_k;
the glass column is the medium AFTER the surface; air (n = 1) before surface
1; a stop has glass_after = glass_before.  Backward mode mirrors the lens
(z' = z_S - z, R' = -R, order reversed, before/after swapped).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

GLASS_CONST, GLASS_CAUCHY, GLASS_ABBE, GLASS_SELLMEIER = 0, 1, 2, 3
AIR = (GLASS_CONST, (1.0, 0, 0, 0, 0, 0))


@dataclass
class Surface:
    z: float
    R: float
    a: float
    is_stop: bool
    glass_before: tuple = AIR
    glass_after: tuple = AIR
    # even asphere: sag(rho) = c rho^2 / (1 + sqrt(1 - (1 + k) c^2 rho^2))
    #   + A4 rho^4 + A6 rho^6 + A8 rho^8 + A10 rho^10, c = 1/R (0 for R = 0)
    asph: bool = False
    k: float = 0.0
    A: tuple = (0.0, 0.0, 0.0, 0.0)
    # single-layer anti-reflection coating: index n_c, thickness d (um);
    # a quarter wave at lambda0: d = lambda0 / (4 n_c).  coat_n = 0: bare surface
    coat_n: float = 0.0
    coat_d_um: float = 0.0


@dataclass
class OracleLens:
    name: str
    surfaces: list
    opts: dict = field(default_factory=dict)

    @property
    def optical(self):
        return [s for s in self.surfaces if not s.is_stop]

    @property
    def n_optical(self) -> int:
        return len(self.optical)


def _glass_token(tok: str, vd: str | None = None):
    t = tok.strip().lower()
    if t == "air":
        return AIR
    if t == "stop":
        return None
    if ":" in t:
        kind, args = t.split(":", 1)
        v = [float(x) for x in args.split(",")]
        if kind == "n":
            return (GLASS_CONST, (v[0], 0, 0, 0, 0, 0))
        if kind == "abbe":
            return (GLASS_ABBE, (v[0], v[1], 0, 0, 0, 0))
        if kind == "cauchy":
            v = (v + [0.0, 0.0])[:3]
            return (GLASS_CAUCHY, (v[0], v[1], v[2], 0, 0, 0))
        if kind == "sellmeier":
            return (GLASS_SELLMEIER, tuple(v[:6]))
        raise ValueError(f"unknown glass {tok!r}")
    nd = float(t)  # bare Kolb n_d
    if nd == 0.0:
        return None
    if nd == 1.0:
        return AIR
    if vd is not None:
        return (GLASS_ABBE, (nd, float(vd), 0, 0, 0, 0))
    return (GLASS_CONST, (nd, 0, 0, 0, 0, 0))


def _coat_token(tok: str):
    """'coat:n_c,lambda0_nm' -> (n_c, quarter-wave thickness in um)."""
    n_c, lam0 = [float(x) for x in tok.split(":", 1)[1].split(",")][:2]
    return n_c, lam0 * 1e-3 / (4.0 * n_c)


def _asph_token(tok: str):
    """'asph:k,A4,A6,A8,A10' (missing trailing coefficients are 0)."""
    v = [float(x) for x in tok.split(":", 1)[1].split(",")]
    v = (v + [0.0] * 5)[:5]
    return v[0], tuple(v[1:])


def parse_lens(text: str, opts: dict | None = None) -> OracleLens:
    """Parse the repo's .lens table (or a JSON document with a 'surfaces' list).
    Table rows: radius thickness glass aperture_diameter [V_d] [asph:k,A4,A6,A8,A10];
    JSON surfaces may carry "conic" and "aspheric": [A4, A6, A8, A10]."""
    rows, name = [], "lens"
    if text.lstrip().startswith("{"):
        doc = json.loads(text)
        name = doc.get("name", name)
        for s in doc["surfaces"]:
            coat = None
            if "coating" in s:
                n_c, lam0 = float(s["coating"]["n"]), float(s["coating"]["lambda0_nm"])
                coat = (n_c, lam0 * 1e-3 / (4.0 * n_c))
            asph = None
            if "conic" in s or "aspheric" in s:
                A = tuple((list(map(float, s.get("aspheric", []))) + [0.0] * 4)[:4])
                asph = (float(s.get("conic", 0.0)), A)
            rows.append((float(s["radius_mm"]), float(s["thickness_mm"]),
                         _glass_token(str(s["glass"])), 2.0 * float(s["semi_aperture_mm"]), asph, coat))
    else:
        for line in text.splitlines():
            body = line.split("#", 1)[0].strip()
            if not body:
                continue
            tok = body.split()
            if tok[0] == "name":
                name = tok[1]
                continue
            asph, coat = None, None
            while len(tok) > 4 and tok[-1].lower().startswith(("asph:", "coat:")):
                if tok[-1].lower().startswith("asph:"):
                    asph = _asph_token(tok[-1])
                else:
                    coat = _coat_token(tok[-1])
                tok = tok[:-1]
            vd = tok[4] if len(tok) > 4 else None
            rows.append((float(tok[0]), float(tok[1]), _glass_token(tok[2], vd), float(tok[3]), asph, coat))
    surfaces, z, prev = [], 0.0, AIR
    for (r, t, g, d, asph, coat) in rows:
        stop = g is None
        after = prev if stop else g
        sf = Surface(z=z, R=0.0 if stop else r, a=0.5 * d, is_stop=stop, glass_before=prev, glass_after=after)
        if asph is not None and not stop:
            sf.asph, sf.k, sf.A = True, asph[0], asph[1]
        if coat is not None and not stop:
            sf.coat_n, sf.coat_d_um = coat
        surfaces.append(sf)
        prev = after
        z += t
    lens = OracleLens(name=name, surfaces=surfaces, opts=dict(opts or {}))
    return lens


def glass_index(g, lam_nm: float) -> float:
    """O1 via the C oracle (single implementation of the glass formulas)."""
    from . import _lib
    return _lib.glass_index(g[0], g[1], lam_nm)


def mirrored(lens: OracleLens) -> list:
    """C0 backward mode: z' = z_S - z, R' = -R (and A' = -A: the mirrored sag is -sag),
    order reversed, before/after swapped."""
    zS = lens.surfaces[-1].z
    out = []
    for s in reversed(lens.surfaces):
        out.append(Surface(z=zS - s.z, R=-s.R if s.R != 0.0 else 0.0, a=s.a, is_stop=s.is_stop,
                           glass_before=s.glass_after, glass_after=s.glass_before,
                           asph=s.asph, k=s.k, A=tuple(-x for x in s.A),   # sag' = -sag
                           coat_n=s.coat_n, coat_d_um=s.coat_d_um))
    return out


def surface_array(surfs: list) -> np.ndarray:
    a = np.zeros((len(surfs), 26), dtype=np.float64)
    for i, s in enumerate(surfs):
        a[i, 0], a[i, 1], a[i, 2], a[i, 3] = s.z, s.R, s.a, 1.0 if s.is_stop else 0.0
        a[i, 4] = s.glass_before[0]
        a[i, 5:11] = s.glass_before[1]
        a[i, 11] = s.glass_after[0]
        a[i, 12:18] = s.glass_after[1]
        a[i, 18] = 1.0 if s.asph else 0.0
        a[i, 19] = s.k
        a[i, 20:24] = s.A
        a[i, 24], a[i, 25] = s.coat_n, s.coat_d_um
    return a


# ---------------------------------------------------------------------------
# O13 ABCD paraxial matrices
# ray vector (h, u) with u = slope; refraction [[1,0],[(n1-n2)/(n2 R), n1/n2]];
# translation [[1,d],[0,1]]
# ---------------------------------------------------------------------------
def refraction_matrix(n1: float, n2: float, R: float) -> np.ndarray:
    c = 0.0 if R == 0.0 else (n1 - n2) / (n2 * R)
    return np.array([[1.0, 0.0], [c, n1 / n2]])


def translation_matrix(d: float) -> np.ndarray:
    return np.array([[1.0, d], [0.0, 1.0]])


def abcd_vertex_to_vertex(lens: OracleLens, lam_nm: float) -> np.ndarray:
    """System matrix from just before the first vertex to just after the last vertex."""
    M = np.eye(2)
    surfs = lens.surfaces
    for k, s in enumerate(surfs):
        if k > 0:
            M = translation_matrix(s.z - surfs[k - 1].z) @ M
        n1 = glass_index(s.glass_before, lam_nm)
        n2 = glass_index(s.glass_after, lam_nm)
        M = refraction_matrix(n1, n2, s.R) @ M
    return M


def efl_bfl(lens: OracleLens, lam_nm: float):
    """EFL = -1/C, BFL = -A/C measured from the last vertex (air on both ends)."""
    M = abcd_vertex_to_vertex(lens, lam_nm)
    A, C = M[0, 0], M[1, 0]
    return -1.0 / C, -A / C


def paraxial_focus_z(lens: OracleLens, lam_nm: float) -> float:
    return lens.surfaces[-1].z + efl_bfl(lens, lam_nm)[1]


def abcd_input_to_plane(lens: OracleLens, lam_nm: float, z_in: float, z_out: float) -> np.ndarray:
    M = abcd_vertex_to_vertex(lens, lam_nm)
    return translation_matrix(z_out - lens.surfaces[-1].z) @ M @ translation_matrix(lens.surfaces[0].z - z_in)


def pupils(lens: OracleLens, lam_nm: float):
    """Paraxial entrance and exit pupils (images of the aperture stop through the front and
    rear groups; SURVEY §8(f) NEXT-3 exit-pupil sampling).  Returns (z_ent, r_ent, z_exit,
    r_exit) in the lens frame.  Rear group: M from the stop plane to the last vertex; the
    stop's image lies s' = -B/D behind the last vertex with magnification det(M)/D = 1/D
    (air).  Front group: N from the first vertex to the stop plane; the object plane
    conjugate to the stop (A s + B = 0 for N T(s)) is at z = z_first + B/A, imaged onto the
    stop with magnification A."""
    surfs = lens.surfaces
    k = next((i for i, x in enumerate(surfs) if x.is_stop), None)
    if k is None:
        raise ValueError("lens has no aperture stop")
    zs, a = surfs[k].z, surfs[k].a

    def group(ss, z_from):
        M, z = np.eye(2), z_from
        for x in ss:
            M = translation_matrix(x.z - z) @ M
            M = refraction_matrix(glass_index(x.glass_before, lam_nm), glass_index(x.glass_after, lam_nm), x.R) @ M
            z = x.z
        return M, z

    rear = [x for x in surfs[k + 1:] if not x.is_stop]
    if rear:
        M, zl = group(rear, zs)
        z_exit, r_exit = zl - M[0, 1] / M[1, 1], a / abs(M[1, 1])
    else:
        z_exit, r_exit = zs, a
    front = [x for x in surfs[:k] if not x.is_stop]
    if front:
        N, zl = group(front, front[0].z)
        N = translation_matrix(zs - zl) @ N
        z_ent, r_ent = front[0].z + N[0, 1] / N[0, 0], a / abs(N[0, 0])
    else:
        z_ent, r_ent = zs, a
    return z_ent, r_ent, z_exit, r_exit


# ---------------------------------------------------------------------------
# O2 path ids (sentinel, LSB-first) and O12 ghost enumeration
# ---------------------------------------------------------------------------
def decode_path(path_id: int):
    """K = floor(log2 id); interaction k (1-based) is 'R' iff bit k-1 is set."""
    if path_id <= 0:
        raise ValueError("path id must be positive")
    K = path_id.bit_length() - 1
    return ["R" if (path_id >> k) & 1 else "T" for k in range(K)]


def encode_path(seq) -> int:
    pid = 1 << len(seq)
    for k, L in enumerate(seq):
        if L == "R":
            pid |= 1 << k
    return pid


def all_t_id(m: int) -> int:
    return 1 << m


def ghost_id(m: int, i: int, j: int) -> int:
    """Two-bounce ghost reflecting at optical surface i then j (1 <= j < i <= m)."""
    return (1 << (m + 2 * (i - j))) + (1 << (i - 1)) + (1 << (2 * i - j - 1))


def _walk_normal_incidence(lens: OracleLens, path_id: int, lam_nm: float):
    """Walk the optical-surface sequence of a path id; return throughput at normal incidence
    (product of R = ((n1-n2)/(n1+n2))^2 or 1-R per interaction) or None if inconsistent."""
    opt = lens.optical
    m = len(opt)
    seq = decode_path(path_id)
    s, d, ncur, I = 0, +1, 1.0, 1.0
    for L in seq:
        if not (0 <= s < m):
            return None
        surf = opt[s]
        n2 = glass_index(surf.glass_after if d > 0 else surf.glass_before, lam_nm)
        if surf.coat_n > 0.0:   # thin film at normal incidence (same Airy formula as the trace)
            nc = surf.coat_n
            a, b = (ncur - nc) / (ncur + nc), (nc - n2) / (nc + n2)
            cb = math.cos(4.0 * math.pi * nc * surf.coat_d_um / (lam_nm * 1e-3))
            R0 = (a * a + b * b + 2 * a * b * cb) / (1 + a * a * b * b + 2 * a * b * cb)
        else:
            R0 = ((ncur - n2) / (ncur + n2)) ** 2
        if L == "T":
            I *= 1.0 - R0
            ncur = n2
        else:
            I *= R0
            d = -d
        s += d
    if d < 0 or s != m:
        return None
    return I


def ghost4_id(m: int, i: int, j: int, k: int, l: int) -> int:
    """Four-bounce path reflecting at optical surfaces i, j, k, l in that order
    (1 <= j < i <= m, j < k <= m, 1 <= l < k): interactions forward to i, back to j,
    forward to k, back to l, forward out."""
    K = m + 2 * (i - j) + 2 * (k - l)
    r1 = i - 1
    r2 = r1 + (i - j)
    r3 = r2 + (k - j)
    r4 = r3 + (k - l)
    return (1 << K) | (1 << r1) | (1 << r2) | (1 << r3) | (1 << r4)


def enumerate_ghosts(lens: OracleLens, max_bounces: int = 2, min_throughput: float = 0.0,
                     lam_nm: float = 587.5618):
    """O12: all (i, j), 1 <= j < i <= m, ascending by id; optional normal-incidence prune.
    max_bounces = 0 returns the all-T path only; 2 returns the all-T path plus ghosts;
    4 adds the four-bounce paths (i, j, k, l) of ghost4_id, their pair given as (i, j)."""
    m = lens.n_optical
    items = [(all_t_id(m), (0, 0))]

    def keep(pid):
        if min_throughput <= 0.0:
            return True
        thr = _walk_normal_incidence(lens, pid, lam_nm)
        return thr is not None and thr >= min_throughput

    if max_bounces >= 2:
        for i in range(2, m + 1):
            for j in range(1, i):
                pid = ghost_id(m, i, j)
                if keep(pid):
                    items.append((pid, (i, j)))
    if max_bounces >= 4:
        for j in range(1, m):
            for i in range(j + 1, m + 1):
                for k in range(j + 1, m + 1):
                    for l in range(1, k):
                        pid = ghost4_id(m, i, j, k, l)
                        if keep(pid):
                            items.append((pid, (i, j)))
    items.sort()
    return [p for p, _ in items], [ij for _, ij in items]
