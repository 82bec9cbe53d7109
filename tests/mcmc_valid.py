"""Markov-chain Monte Carlo sampler of a path's valid input region ("To
accelerate data generation, we employ a Markov Chain Monte Carlo sampler with a binary
visibility target function"), for training the maps of ghost paths whose valid fraction
is too small for uniform sampling (tests/fit_flare_maps.py --mcmc-below).

TEST INFRASTRUCTURE: visibility comes from the float64 oracle (oracle.trace), never from
the CUDA path.  The target is the indicator of the valid set inside the law's domain, so
its stationary distribution is uniform over the valid region -- the paper's "uniformly
sample (p_in, w_in) within the valid region".  Many independent chains advance in
lock-step (one batched oracle call per step); a random-walk proposal is accepted iff it
stays in the domain and is valid; the step size adapts during burn-in towards ~30 %
acceptance.

State for the "collimated" flare law (fixed direction): (p_x, p_y, lambda) on the entry
disc x [lam_lo, lam_hi].
"""
from __future__ import annotations

import math

import numpy as np

import oracle


def _rays(state, law):
    n = state.shape[0]
    a = math.radians(law["angle_deg"])
    return {"ox": state[:, 0].astype(np.float32), "oy": state[:, 1].astype(np.float32),
            "dx": np.full(n, math.sin(a), np.float32), "dy": np.zeros(n, np.float32),
            "dz": np.full(n, math.cos(a), np.float32), "lambda_nm": state[:, 2].astype(np.float32),
            "plane_z": float(law["plane_z"])}


def _in_domain(state, law, lam):
    x0 = law.get("disc_x0", 0.0)
    r2 = (state[:, 0] - x0) ** 2 + state[:, 1] ** 2
    return (r2 <= law["disc_r"] ** 2) & (state[:, 2] >= lam[0]) & (state[:, 2] <= lam[1])


def valid_of(olens, path_id, direction, state, law, threads):
    return oracle.trace(olens, path_id, direction, _rays(state, law), threads=threads)["valid"]


def sample_valid(olens, path_id: int, direction: int, law: dict, lam: tuple, n_samples: int, seed: int,
                 chains: int = 4096, burn_in: int = 200, thin: int = 4, seed_tries: int = 1 << 22,
                 threads: int = 1):
    """n_samples states (p_x, p_y, lambda) distributed uniformly over the valid region of
    `path_id` within the collimated law's domain (entry disc x wavelength interval).
    Raises RuntimeError if no valid seed is found among `seed_tries` uniform draws."""
    if law["kind"] != "collimated":
        raise ValueError("mcmc sampler implemented for the collimated flare law")
    rng = np.random.default_rng([int(seed), 0x3C3C])
    x0, R = law.get("disc_x0", 0.0), law["disc_r"]
    # seeds: uniform draws until enough valid starting points
    seeds = np.zeros((0, 3))
    tried = 0
    while seeds.shape[0] < chains and tried < seed_tries:
        m = 1 << 18
        rr = R * np.sqrt(rng.random(m))
        ph = 2 * np.pi * rng.random(m)
        st = np.stack([x0 + rr * np.cos(ph), rr * np.sin(ph), lam[0] + (lam[1] - lam[0]) * rng.random(m)], 1)
        seeds = np.concatenate([seeds, st[valid_of(olens, path_id, direction, st, law, threads)]])
        tried += m
    if seeds.shape[0] == 0:
        raise RuntimeError(f"path {path_id}: no valid ray among {tried} uniform draws")
    state = seeds[rng.integers(0, seeds.shape[0], chains)]
    step = np.array([0.05 * R, 0.05 * R, 0.05 * (lam[1] - lam[0])])
    out, t = [], 0
    while sum(o.shape[0] for o in out) < n_samples:
        prop = state + step * rng.standard_normal(state.shape)
        ok = _in_domain(prop, law, lam)
        if ok.any():
            v = np.zeros(chains, bool)
            v[ok] = valid_of(olens, path_id, direction, prop[ok], law, threads)
            ok &= v
        state[ok] = prop[ok]
        acc = ok.mean()
        if t < burn_in:                       # adapt towards ~30 % acceptance
            step *= math.exp(0.5 * (acc - 0.3))
        elif (t - burn_in) % thin == 0:
            out.append(state.copy())
        t += 1
    return np.concatenate(out)[:n_samples]


def to_rays(state, law):
    """Ray dict (plt_inputs layout) of sampled states."""
    return _rays(state, law)
