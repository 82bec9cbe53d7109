"""Pins for oracle O1 (glass), O13 (ABCD) and O2/O12 (path ids, ghosts) -- CPU only."""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.lens import (GLASS_ABBE, GLASS_CAUCHY, GLASS_CONST, GLASS_SELLMEIER, decode_path,
                         encode_path, ghost_id, refraction_matrix, translation_matrix)
from plt_inputs import configs as C
from plt_inputs.lenses import LENSES

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
NBK7 = (GLASS_SELLMEIER, (1.03961212, 0.231792344, 1.01046945, 0.00600069867, 0.0200179144, 103.560653))
LF, LD, LC = 486.1327, 587.5618, 656.2725


def n_of(g, lam):
    return oracle.glass_index(g, lam)


def test_nbk7_catalog():
    g = G["nbk7_sellmeier"]
    nd, nF, nC = n_of(NBK7, LD), n_of(NBK7, LF), n_of(NBK7, LC)
    assert abs(nd - g["n_d"]) < g["tol_n"]
    assert abs(nF - g["n_F"]) < g["tol_n"]
    assert abs(nC - g["n_C"]) < g["tol_n"]
    assert abs((nd - 1) / (nF - nC) - g["V_d"]) < g["tol_V"]


@pytest.mark.parametrize("nd,vd", [(1.670, 47.1), (1.617, 54.0), (1.805, 25.4)])
def test_abbe_reproduces_nd_and_vd(nd, vd):
    g = (GLASS_ABBE, (nd, vd, 0, 0, 0, 0))
    assert abs(n_of(g, LD) - nd) < 1e-12
    assert abs((n_of(g, LD) - 1) / (n_of(g, LF) - n_of(g, LC)) - vd) < 1e-9


def test_cauchy_spec_example_and_monotone():
    c = G["cauchy_example"]
    g = (GLASS_CAUCHY, (c["A"], c["B_um2"], 0, 0, 0, 0))
    assert abs(n_of(g, c["lambda_nm"]) - c["n"]) < c["tol"]
    lams = np.linspace(380, 780, 81)
    for gg in (g, NBK7, (GLASS_ABBE, (1.7, 30.0, 0, 0, 0, 0))):
        ns = [n_of(gg, l) for l in lams]
        assert all(a > b for a, b in zip(ns, ns[1:])) and min(ns) >= 1.0
    assert n_of((GLASS_CONST, (1.5168, 0, 0, 0, 0, 0)), 550) == 1.5168


def _thick_lens(n, R1, R2, t):
    # independent closed form: lensmaker thick-lens formula
    inv_f = (n - 1) * (1 / R1 - 1 / R2 + (n - 1) * t / (n * R1 * R2))
    f = 1 / inv_f
    bfl = f * (1 - (n - 1) * t / (n * R1))
    return f, bfl


def test_singlet_efl_bfl_lensmaker():
    lens = oracle.load_lens(LENSES["singlet"])
    for key, lam in (("F", LF), ("d", LD), ("C", LC)):
        efl, bfl = oracle.efl_bfl(lens, lam)
        f, b = _thick_lens(n_of(NBK7, lam), 50.0, -50.0, 5.0)
        assert abs(efl - f) < 1e-9 and abs(bfl - b) < 1e-9
        assert abs(efl - G["singlet_efl_mm"][key]) < 2e-6
        assert abs(bfl - G["singlet_bfl_mm"][key]) < 2e-6
        M = oracle.abcd_vertex_to_vertex(lens, lam)
        assert abs(np.linalg.det(M) - 1.0) < 1e-12


def test_dgauss_and_wide_efl():
    d = oracle.load_lens(LENSES["dgauss50"])
    efl, bfl = oracle.efl_bfl(d, LD)
    assert abs(efl - G["dgauss50_efl_mm"]["value"]) < G["dgauss50_efl_mm"]["tol"]
    assert abs(bfl - G["dgauss50_bfl_mm"]["value"]) < G["dgauss50_bfl_mm"]["tol"]
    w = oracle.load_lens(LENSES["wide22"])
    assert abs(oracle.efl_bfl(w, LD)[0] - G["wide22_efl_mm"]["value"]) < G["wide22_efl_mm"]["tol"]
    assert w.n_optical == 12 and d.n_optical == 10
    for lens in (d, w):
        assert abs(np.linalg.det(oracle.abcd_vertex_to_vertex(lens, 500.0)) - 1.0) < 1e-12


def test_abcd_matrix_examples():
    ex = G["abcd_translation_example"]
    h, u = translation_matrix(ex["d"]) @ np.array([ex["h"], ex["u"]])
    assert abs(h - ex["h_out"]) < 1e-15 and abs(u - ex["u_out"]) < 1e-15
    P = refraction_matrix(1.0, 1.5, 0.0)
    assert np.allclose(P, [[1, 0], [0, 1 / 1.5]], atol=0, rtol=0)
    assert abs(np.linalg.det(refraction_matrix(1.2, 1.7, 33.0)) - 1.2 / 1.7) < 1e-15


def test_path_encoding_and_printed_ids():
    for pid in (1, 2, 5, 4096, 65616, 131092, (1 << 30) | 12345):
        assert encode_path(decode_path(pid)) == pid
    for key in ("path_65616", "path_131092"):
        g = G[key]
        pid = int(key.split("_")[1])
        assert ghost_id(g["m"], g["i"], g["j"]) == pid
        seq = decode_path(pid)
        assert len(seq) == g["K"] == g["m"] + 2 * (g["i"] - g["j"])
        assert [k + 1 for k, L in enumerate(seq) if L == "R"] == [g["i"], 2 * g["i"] - g["j"]]


def _slab_text(nsurf):
    rows = ["name flat"]
    for k in range(nsurf):
        rows.append(f"0 2.0 {'n:1.5' if k % 2 == 0 else 'air'} 20")
    return "\n".join(rows) + "\n"


def test_enumerate_counts_parity_ascending():
    lens = oracle.load_lens(_slab_text(4), {"sensor_z_mm": 50.0})
    ids, ij = oracle.enumerate_ghosts(lens, 2)
    assert len(ids) == G["enumerate_4_surfaces_2_bounces"]["count"]
    assert ids == sorted(ids) and len(set(ids)) == len(ids)
    for name in ("dgauss50", "wide22"):
        L = oracle.load_lens(LENSES[name])
        ids, ij = oracle.enumerate_ghosts(L, 2)
        m = L.n_optical
        assert len(ids) == 1 + m * (m - 1) // 2
        assert ids[0] == 1 << m and ids == sorted(ids)
        for pid in ids:
            assert decode_path(pid).count("R") % 2 == 0
    # brute force: every bit string of length K with exactly two R whose surface walk is consistent
    L = oracle.load_lens(_slab_text(5), {"sensor_z_mm": 50.0})
    m = 5
    brute = set()
    for K in range(m, m + 2 * m):
        for a in range(K):
            for b in range(a + 1, K):
                pid = (1 << K) | (1 << a) | (1 << b)
                if oracle.lens._walk_normal_incidence(L, pid, LD) is not None:
                    brute.add(pid)
    ids, _ = oracle.enumerate_ghosts(L, 2)
    assert brute == set(ids[1:])


def test_ghost_prune_is_monotone():
    L = oracle.load_lens(LENSES["wide22"])
    all_ids, _ = oracle.enumerate_ghosts(L, 2, 0.0)
    prev = set(all_ids)
    for thr in (1e-6, 1e-5, 1e-4, 1e-3):
        ids, _ = oracle.enumerate_ghosts(L, 2, thr)
        assert set(ids) <= prev
        prev = set(ids)
    # normal-incidence throughput of a slab ghost (2,1): T1 R2 R1 T2 with R = 0.04
    slab = oracle.load_lens(_slab_text(2), {"sensor_z_mm": 50.0})
    thr = oracle.lens._walk_normal_incidence(slab, ghost_id(2, 2, 1), LD)
    assert abs(thr - 0.96 * 0.04 * 0.04 * 0.96) < 1e-15


def test_four_bounce_enumeration_is_complete_and_consistent():
    """O12 with max_bounces = 4: the four-bounce ids are exactly the
    bit strings with four R whose surface walk enters at the front and leaves at the back
    (brute force over every such string), and their count follows the closed form
    sum_j (m - j) * sum_{k > j} (k - 1)."""
    L = oracle.load_lens(_slab_text(4), {"sensor_z_mm": 50.0})
    m = 4
    brute = set()
    for K in range(m, m + 4 * m):
        for bits in itertools.combinations(range(K), 4):
            pid = (1 << K) | sum(1 << b for b in bits)
            if oracle.lens._walk_normal_incidence(L, pid, LD) is not None:
                brute.add(pid)
    ids4, _ = oracle.enumerate_ghosts(L, 4)
    ids2, _ = oracle.enumerate_ghosts(L, 2)
    four = set(ids4) - set(ids2)
    assert four == brute
    assert len(four) == sum((m - j) * sum(k - 1 for k in range(j + 1, m + 1)) for j in range(1, m))
    # normal-incidence throughput of a four-bounce path through a 2-surface slab: T R R R R T
    slab = oracle.load_lens(_slab_text(2), {"sensor_z_mm": 50.0})
    pid = oracle.lens.ghost4_id(2, 2, 1, 2, 1)
    assert abs(oracle.lens._walk_normal_incidence(slab, pid, LD) - 0.96 * 0.04 ** 4 * 0.96) < 1e-18
