"""O2-stereo: float64 numpy solve of the census + tensor-TGV stereo energy (TEST INFRASTRUCTURE ONLY, see
oracle/__init__.py).

The independent-precision reference of the depth-map module (paper §IV; readings S-1 … S-13,
DESIGN.md §13): the integer census signatures and Hamming costs come from ``stereo_oracle.c`` (exact,
pinned), everything else is written here from the readings in float64 with whole-array operations —
the tensor T = e·nnᵀ + n⊥n⊥ᵀ, e = exp(−γ|∇I_R|^β) (S-5), forward differences with Neumann
boundary and their negative adjoints (S-7), the Chambolle–Pock iterations on (d, w) with the α-ball
projections in the textbook form p / max(1, |p|/α) and the coupling prox as a division (S-8; the fp32
side uses the equivalent product forms of S-13), over-relaxation θ_CP = 1, the data step as an exact
argmin over the integer disparities with the parabola step (S-9), θ geometric from θ₀ to θ_end.
"""
from __future__ import annotations

import numpy as np


def _gx(a):
    g = np.zeros_like(a)
    g[:, :-1] = a[:, 1:] - a[:, :-1]
    return g


def _gy(a):
    g = np.zeros_like(a)
    g[:-1, :] = a[1:, :] - a[:-1, :]
    return g


def _gx_adj(v):
    """Adjoint of _gx: ⟨_gx(a), v⟩ = ⟨a, _gx_adj(v)⟩ (= − divergence)."""
    r = np.zeros_like(v)
    r[:, :-1] -= v[:, :-1]
    r[:, 1:] += v[:, :-1]
    return r


def _gy_adj(v):
    r = np.zeros_like(v)
    r[:-1, :] -= v[:-1, :]
    r[1:, :] += v[:-1, :]
    return r


def tensor_f64(I, beta=1.0, gamma=4.0):
    """(T11, T12, T22) [3, H, W] float64: central differences with clamped borders (S-5), T = I where
    |∇I| < 1e-6."""
    A = np.asarray(I, np.float64)
    P = np.pad(A, 1, mode="edge")
    gx = (P[1:-1, 2:] - P[1:-1, :-2]) / 2.0
    gy = (P[2:, 1:-1] - P[:-2, 1:-1]) / 2.0
    m = np.hypot(gx, gy)
    small = m < 1e-6
    ms = np.where(small, 1.0, m)
    nx, ny = gx / ms, gy / ms
    e = np.exp(-gamma * ms ** beta)
    T11 = e * nx * nx + ny * ny
    T12 = e * nx * ny - ny * nx
    T22 = e * ny * ny + nx * nx
    return np.stack([np.where(small, 1.0, T11), np.where(small, 0.0, T12), np.where(small, 1.0, T22)])


def stereo_f64(IL, IR, D, cost, win=5, outer=10, inner=10, lam=0.5, alpha1=1.0, alpha2=5.0, beta=1.0,
               gamma=4.0, theta0=1.0, theta_end=0.01, tau=None, sigma=None):
    """Solve one pair.  cost: [H, W, D] integer Hamming costs (S-3).  Returns (d, w, a) float64."""
    rho = np.asarray(cost, np.float64)
    H, W = rho.shape[:2]
    tau = 1.0 / np.sqrt(12.0) if tau is None else float(tau)
    sigma = 1.0 / np.sqrt(12.0) if sigma is None else float(sigma)
    T11, T12, T22 = tensor_f64(IR, beta, gamma)
    a = np.argmin(rho, axis=2).astype(np.float64)          # winner-take-all, ties → smallest d (S-8)
    d = a.copy()
    db = d.copy()
    w = np.zeros((2, H, W))
    wb = w.copy()
    p = np.zeros((2, H, W))
    q = np.zeros((4, H, W))
    ks = np.arange(D, dtype=np.float64)
    for o in range(outer):
        theta = theta0 if outer <= 1 else theta0 * (theta_end / theta0) ** (o / (outer - 1))
        for _ in range(inner):
            # dual ascent: K(d̄, w̄) = (T∇d̄ − w̄, ∇w̄), projections onto the α₁ / α₂ balls (S-6)
            gx, gy = _gx(db), _gy(db)
            p = p + sigma * np.stack([T11 * gx + T12 * gy - wb[0], T12 * gx + T22 * gy - wb[1]])
            p = p / np.maximum(1.0, np.sqrt((p ** 2).sum(0)) / alpha1)
            q = q + sigma * np.stack([_gx(wb[0]), _gy(wb[0]), _gx(wb[1]), _gy(wb[1])])
            q = q / np.maximum(1.0, np.sqrt((q ** 2).sum(0)) / alpha2)
            # primal descent with Kᵀ(p, q) = (∇ᵀ(T p), −p + ∇ᵀq); prox of 1/(2θ)(d − a)² for d
            tp1, tp2 = T11 * p[0] + T12 * p[1], T12 * p[0] + T22 * p[1]
            kd = _gx_adj(tp1) + _gy_adj(tp2)
            kw = np.stack([-p[0] + _gx_adj(q[0]) + _gy_adj(q[1]), -p[1] + _gx_adj(q[2]) + _gy_adj(q[3])])
            dn = (d - tau * kd + (tau / theta) * a) / (1.0 + tau / theta)
            wn = w - tau * kw
            db, wb = 2.0 * dn - d, 2.0 * wn - w
            d, w = dn, wn
        # data step: exact argmin over k of 1/(2θ)(d − k)² + λρ_k, then the parabola (S-9)
        E = (d[..., None] - ks) ** 2 / (2.0 * theta) + lam * rho
        k = np.argmin(E, axis=2)
        a = k.astype(np.float64)
        inner_k = (k > 0) & (k < D - 1)
        kc = np.clip(k, 1, D - 2)
        Em = np.take_along_axis(E, (kc - 1)[..., None], 2)[..., 0]
        E0 = np.take_along_axis(E, kc[..., None], 2)[..., 0]
        Ep = np.take_along_axis(E, (kc + 1)[..., None], 2)[..., 0]
        den = Em - 2.0 * E0 + Ep
        ok = inner_k & (den > 0)
        delta = np.clip(np.where(ok, (Em - Ep) / (2.0 * np.where(ok, den, 1.0)), 0.0), -0.5, 0.5)
        a = a + delta
    return d, w, a
