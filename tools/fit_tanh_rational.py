"""Fit the odd rational tanh(x) ~= x P(x^2) / Q(x^2) (P degree 4, Q degree 4 with Q(0) = 1)
on [0, X_MAX] that eval_map's accurate classifier units evaluate on the FMA pipe (packed
FFMA2) with ONE MUFU reciprocal, instead of ex2 + rcp.

Linearised least squares on tanh Q - x P = 0 (Sanathanan-Koerner reweighting by 1/|Q| and a
Lawson-style weight update towards the minimax error), in float64; then the float32
evaluation as the kernel does it (clamp to +-X_MAX, Horner with fused multiply-adds,
correctly rounded reciprocal) is checked on a dense grid of [-12, 12].  Prints the
coefficients as C hex-float literals.

    python tools/fit_tanh_rational.py
"""
import numpy as np

X_MAX = 8.5
NP, NQ = 5, 4          # P: p0..p4 (degree 4 in x^2); Q: 1, q1..q4


def fit(iters=60):
    x = np.unique(np.concatenate([np.linspace(0.0, X_MAX, 20001),
                                  X_MAX * (1.0 - np.cos(np.linspace(0.0, np.pi / 2, 5001)))]))[1:]
    t, s = np.tanh(x), x * x
    sk = np.ones_like(x)        # Sanathanan-Koerner weight 1/|Q_prev|
    lw = np.ones_like(x)        # Lawson weight (minimax), damped
    best = None
    for it in range(iters):
        w = sk * lw
        A = np.concatenate([x[:, None] * s[:, None] ** np.arange(NP)[None, :],
                            -t[:, None] * s[:, None] ** np.arange(1, NQ + 1)[None, :]], 1)
        sol, *_ = np.linalg.lstsq(A * w[:, None], t * w, rcond=None)
        p, q = sol[:NP], np.concatenate([[1.0], sol[NP:]])
        Q, P = np.polyval(q[::-1], s), np.polyval(p[::-1], s)
        if np.any(Q <= 0):
            break
        err = x * P / Q - t
        m = np.abs(err).max()
        if best is None or m < best[0]:
            best = (m, p.copy(), q.copy())
        sk = 1.0 / np.abs(Q)
        if it >= 5:             # after the SK iterations settle, move towards equi-oscillation
            lw = lw * (np.abs(err) / m + 1e-3) ** 0.25
            lw /= lw.max()
    return best


def eval_f32(p, q, x):
    f = np.float32
    p, q = p.astype(f), q.astype(f)
    x = np.clip(x.astype(f), -f(X_MAX), f(X_MAX))
    s = (x * x).astype(f)
    P = np.full_like(s, p[-1])
    for c in p[-2::-1]:
        P = (P.astype(np.float64) * s + c).astype(f)        # fma: one rounding
    Q = np.full_like(s, q[-1])
    for c in q[-2::-1]:
        Q = (Q.astype(np.float64) * s + c).astype(f)
    r = (1.0 / Q.astype(np.float64)).astype(f)
    return ((x * P).astype(f) * r).astype(f)


def main():
    m, p, q = fit()
    xs = np.linspace(-12.0, 12.0, 4000001)
    e = np.abs(eval_f32(p, q, xs).astype(np.float64) - np.tanh(xs))
    print(f"float64 fit max |error| {m:.3e}; float32 evaluation max |error| {e.max():.3e} at x = {xs[e.argmax()]:.4f}")
    fl = lambda v: float(np.float32(v)).hex().replace("0x1.", "0x1.") + "f"
    print("P (p0..p4):", ", ".join(fl(v) for v in p))
    print("Q (q1..q4):", ", ".join(fl(v) for v in q[1:]))


if __name__ == "__main__":
    main()
