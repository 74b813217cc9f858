"""Pins of the depth-map estimation oracle (oracle/stereo_oracle.c; paper §IV).

  * census: the worked 3×3 example (tests/golden/stereo_examples.txt), constant images, exact
    invariance under strictly increasing intensity maps (the census is an order statistic);
  * cost volume: identical images give zero cost at d = 0, complementary signatures the maximum, and a
    textured image shifted by a known amount is matched at that shift by winner-take-all;
  * tensor: closed forms, det T = exp(−γ|∇I|^β), the unit eigenvector orthogonal to ∇I;
  * TGV operators: ⟨K(d,w), (p,q)⟩ = ⟨(d,w), Kᵀ(p,q)⟩ (the divergences are the negative adjoints);
  * data step: with λ = 0 the parabola through the exact quadratic returns d itself;
  * whole solve: a constant-disparity pair is recovered to 0.1 px, a slanted plane to a median < 0.5 px
    (S:400-401), and λ → ∞ reproduces winner-take-all up to the sub-pixel step.
"""
import math
import os

import numpy as np
import pytest

import oracle
from synth.stereo import plane_pair

GOLD = os.path.join(os.path.dirname(__file__), "golden", "stereo_examples.txt")


def _golden(kind):
    out = []
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        k, cite, rest = line.split(None, 2)
        if k == kind:
            lhs, rhs = rest.split("->")
            out.append((cite, [float(v) for v in lhs.split()], [float(v) for v in rhs.split()]))
    return out


@pytest.mark.parametrize("cite,inp,exp", _golden("census"))
def test_census_worked_example(cite, inp, exp):
    win = int(inp[0])
    patch = np.array(inp[1:], np.float32).reshape(win, win)
    sig = oracle.census(patch, win=win)
    assert int(sig[win // 2, win // 2]) == int(exp[0]), cite


@pytest.mark.parametrize("cite,inp,exp", _golden("tensor"))
def test_tensor_worked_examples(cite, inp, exp):
    gx, gy, gamma, beta = inp
    # an image whose central difference at the centre pixel is (gx, gy): a linear ramp
    y, x = np.mgrid[0:5, 0:5].astype(np.float64)
    I = (gx * x + gy * y).astype(np.float32)
    T = oracle.tensor(I, beta=beta, gamma=gamma)[2, 2]
    assert np.allclose(T, exp, atol=1e-7), (cite, T)


def test_census_invariances():
    rng = np.random.default_rng(0)
    I = rng.uniform(size=(20, 30)).astype(np.float32)
    assert (oracle.census(np.full((8, 8), 0.3, np.float32)) == 0).all()
    s = oracle.census(I)
    for phi in (lambda v: v ** 2.2, lambda v: np.sqrt(v), lambda v: 0.1 + 0.5 * v):
        assert np.array_equal(oracle.census(phi(I).astype(np.float32)), s)
    # 5×5: 24 bits, bit k set iff neighbour k < centre
    assert s.max() < (1 << 24)
    y, x = 7, 11
    nb = [I[np.clip(y + dy, 0, 19), np.clip(x + dx, 0, 29)] for dy in range(-2, 3) for dx in range(-2, 3)
          if (dx, dy) != (0, 0)]
    assert s[y, x] == sum(1 << k for k, v in enumerate(nb) if v < I[y, x])


def test_cost_volume_properties():
    IL, IR, _ = plane_pair(32, 80, c=6.0)
    sL, sR = oracle.census(IL), oracle.census(IR)
    assert (oracle.cost_volume(sR, sR, 8)[..., 0] == 0).all()
    cv = oracle.cost_volume(sL, sR, 16)
    assert (cv[:, -3:, 5:] == 24).all()                      # x + d outside the image
    assert (cv[4:-4, 4:-24].argmin(-1) == 6).mean() > 0.95   # textured pair shifted by 6 px
    a = np.array([[0.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 0.0]], np.float32)
    s1 = oracle.census(a, win=3)[1, 1]
    s2 = oracle.census(1.0 - a, win=3)[1, 1]
    assert s1 == 0xFF and s2 == 0 and bin(int(s1) ^ int(s2)).count("1") == 8


def test_tensor_structure():
    rng = np.random.default_rng(1)
    I = rng.uniform(size=(24, 24)).astype(np.float32)
    T = oracle.tensor(I, beta=1.0, gamma=4.0).astype(np.float64)
    gy, gx = np.gradient(I.astype(np.float64))
    g = np.hypot(gx, gy)
    inner = (slice(1, -1), slice(1, -1))
    det = T[..., 0] * T[..., 2] - T[..., 1] ** 2
    assert np.allclose(det[inner], np.exp(-4.0 * g[inner]), atol=2e-6)
    # eigenvalue 1 has an eigenvector orthogonal to ∇I: T·n⊥ = n⊥
    n_perp = np.stack([-gy, gx], -1) / np.maximum(g, 1e-12)[..., None]
    Tn = np.stack([T[..., 0] * n_perp[..., 0] + T[..., 1] * n_perp[..., 1],
                   T[..., 1] * n_perp[..., 0] + T[..., 2] * n_perp[..., 1]], -1)
    assert np.abs(Tn - n_perp)[inner].max() <= 1e-6


@pytest.mark.parametrize("seed", range(5))
def test_tgv_adjointness(seed):
    rng = np.random.default_rng(seed)
    H, W = 13, 17
    T = oracle.tensor(rng.uniform(size=(H, W)).astype(np.float32))
    d = rng.normal(size=(H, W)).astype(np.float32)
    w = rng.normal(size=(2, H, W)).astype(np.float32)
    p = rng.normal(size=(2, H, W)).astype(np.float32)
    q = rng.normal(size=(4, H, W)).astype(np.float32)
    u, v = oracle.tgv_K(T, d, w)
    kd, kw = oracle.tgv_KT(T, p, q)
    lhs = (u.astype(np.float64) * p).sum() + (v.astype(np.float64) * q).sum()
    rhs = (d.astype(np.float64) * kd).sum() + (w.astype(np.float64) * kw).sum()
    assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs) + 1)


def test_data_step_closed_form():
    rho = np.zeros(16, np.float32)
    for d in (3.25, 7.5, 9.9):
        a = oracle.data_step(d, np.random.default_rng(0).uniform(size=16).astype(np.float32), 1.0, 0.0)
        assert abs(a - d) <= 1e-5
    # λ = 0 and a flat cost: the nearest integer ± the parabola; at the ends no parabola
    assert oracle.data_step(0.2, rho, 1.0, 0.0) == 0.0
    assert oracle.data_step(15.4, rho, 1.0, 0.0) == 15.0
    # c = 0: the cost argmin (ties: smallest), parabola of the costs
    r = np.array([5, 4, 1, 3, 6], np.float32)
    assert abs(oracle.data_step(0.0, r, 0.0, 1.0) - (2 + (4.0 - 3.0) / (2 * ((4.0 - 2.0) + 3.0)))) <= 1e-6


def test_constant_disparity_recovered():
    IL, IR, dt = plane_pair(48, 96, c=7.0)
    d, w, a = oracle.stereo(IL, IR, D=32, outer=10, inner=20)
    err = np.abs(d - 7.0)[4:-4, 4:-40]
    assert np.median(err) <= 0.1 and np.percentile(err, 95) <= 0.3
    assert np.median(np.abs(w)) <= 0.05


@pytest.mark.parametrize("abc", [(0.05, 0.02, 5.0), (-0.04, 0.0, 12.0)])
def test_slanted_plane(abc):
    IL, IR, dt = plane_pair(48, 96, *abc)
    d, w, a = oracle.stereo(IL, IR, D=32, outer=10, inner=20)
    err = np.abs(d - dt.numpy())[4:-4, 4:-40]
    assert np.median(err) < 0.5
    assert np.isfinite(d).all()


def test_large_lambda_is_wta():
    IL, IR, dt = plane_pair(32, 64, 0.03, 0.0, 4.0)
    d, w, a = oracle.stereo(IL, IR, D=24, outer=3, inner=5, lam=1e5)
    cv = oracle.cost_volume(oracle.census(IL), oracle.census(IR), 24)
    is_min = cv == cv.min(-1, keepdims=True)                  # every cost minimiser (ties allowed)
    k = np.arange(24)
    near = np.abs(a[..., None] - k) <= 0.5 + 1e-6
    assert (near & is_min).any(-1).all()


# --- the float64 numpy solve (oracle/stereo64.py), the independent-precision reference of the GPU solve ---

def test_stereo64_operators_adjoint_and_tensor_closed_form():
    """Pins of stereo64's own pieces: its difference operators are adjoint (⟨∇a, v⟩ = ⟨a, ∇ᵀv⟩ to 1e-12)
    and its tensor matches the closed form: det T = exp(−γ|∇I|^β), T n⊥ = n⊥, T = I on a flat image."""
    from oracle import stereo64 as S64
    rng = np.random.default_rng(3)
    a = rng.normal(size=(11, 13))
    v = rng.normal(size=(11, 13))
    assert abs((S64._gx(a) * v).sum() - (a * S64._gx_adj(v)).sum()) <= 1e-12
    assert abs((S64._gy(a) * v).sum() - (a * S64._gy_adj(v)).sum()) <= 1e-12
    y, x = np.mgrid[0:9, 0:9].astype(np.float64)
    I = 0.03 * x + 0.04 * y                                   # |∇I| = 0.05 inside
    T11, T12, T22 = S64.tensor_f64(I, beta=1.0, gamma=4.0)
    det = T11 * T22 - T12 * T12
    assert abs(det[4, 4] - np.exp(-4.0 * 0.05)) <= 1e-12
    npx, npy = -0.8, 0.6                                      # n⊥ of n = (0.6, 0.8)
    assert abs(T11[4, 4] * npx + T12[4, 4] * npy - npx) <= 1e-12
    assert abs(T12[4, 4] * npx + T22[4, 4] * npy - npy) <= 1e-12
    F = S64.tensor_f64(np.full((5, 5), 0.3))
    assert np.array_equal(F, np.stack([np.ones((5, 5)), np.zeros((5, 5)), np.ones((5, 5))]))


def test_stereo64_matches_fp32_oracle():
    """The float64 numpy solve (textbook division forms, whole-array operators) and the fp32 C oracle
    (S-13 product forms, per-pixel loops) agree to 1e-4 px after 10 × 20 iterations on a slanted plane,
    and both recover the plane (a dropped term or sign in either breaks one of the two)."""
    from oracle.stereo64 import stereo_f64
    IL, IR, dt = plane_pair(48, 96, 0.02, 0.01, 7.0)
    IL, IR = IL.numpy(), IR.numpy()
    d32, w32, a32 = oracle.stereo(IL, IR, D=24, outer=10, inner=20)
    cost = oracle.cost_volume(oracle.census(IL), oracle.census(IR), 24)
    d64, w64, a64 = stereo_f64(IL, IR, 24, cost, outer=10, inner=20)
    assert np.abs(d32 - d64).max() <= 1e-4
    assert np.abs(w32 - w64).max() <= 1e-4
    assert np.median(np.abs(d64 - dt.numpy())[4:-4, 4:-40]) < 0.5
