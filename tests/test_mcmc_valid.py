"""Pins of the valid-region MCMC sampler (tests/mcmc_valid.py) on a case with a
closed-form valid region: collimated axial light on the C1 singlet, whose only limiting
aperture is the 8 mm front stop -- the valid set on the entry disc is the disc r <= 8 for
every wavelength.  The chains must stay valid and be uniform on it: r^2 / 64 ~ U(0, 1),
lambda ~ U(400, 700), the polar angle uniform."""
import numpy as np

import oracle
from plt_inputs.lenses import LENSES

from mcmc_valid import sample_valid, to_rays


def test_mcmc_is_uniform_on_a_known_valid_disc():
    ol = oracle.load_lens(LENSES["singlet"])
    law = {"kind": "collimated", "plane_z": -5.0, "disc_r": 12.0, "disc_x0": 0.0, "angle_deg": 0.0}
    s = sample_valid(ol, oracle.all_t_id(ol.n_optical), 0, law, (400.0, 700.0), 60_000, seed=3, chains=2000,
                     burn_in=100, thin=2)
    t = oracle.trace(ol, oracle.all_t_id(ol.n_optical), 0, to_rays(s, law))
    assert t["valid"].all()
    u = (s[:, 0] ** 2 + s[:, 1] ** 2) / 64.0
    assert u.max() <= 1.0 + 1e-6
    qs = np.quantile(u, [0.1, 0.25, 0.5, 0.75, 0.9])
    assert np.allclose(qs, [0.1, 0.25, 0.5, 0.75, 0.9], atol=0.02), qs
    lq = np.quantile(s[:, 2], [0.1, 0.5, 0.9])
    assert np.allclose(lq, [430.0, 550.0, 670.0], atol=6.0), lq
    ang = np.arctan2(s[:, 1], s[:, 0])
    h, _ = np.histogram(ang, bins=8, range=(-np.pi, np.pi))
    assert h.min() > 0.9 * h.mean() and h.max() < 1.1 * h.mean()
