"""Pins of the oracle's operators and single steps against the paper's worked examples
(tests/golden/worked_examples.txt), adjointness, the operator-norm bound and brute-force energy.
SURVEY §8(c) pin rows 'Gradient / divergence', 'Dual step', 'Primal step', 'Relax', 'Energy'."""
import numpy as np
import pytest

import oracle
import oracle.dense as dn
from synth import random_instance, dense_box


def vidx(x, y, z):
    return x + 8 * y + 64 * z


def one_block(W_on=(), W_all=None):
    c = np.zeros((1, 3), np.int32)
    W = np.zeros((1, 512), np.float32) if W_all is None else np.full((1, 512), W_all, np.float32)
    for v in W_on:
        W[0, vidx(*v)] = 1.0
    return c, W, oracle.neighbours(c)


# ------------------------------------------------------------------------------- gradient (Eq. 3)

def test_gradient_worked_example():
    c, W, nbr = one_block([(3, 3, 3), (4, 3, 3)])
    u = np.zeros((1, 512))
    u[0, vidx(3, 3, 3)] = 0.4
    u[0, vidx(4, 3, 3)] = 0.7
    g = oracle.gradient(nbr, W, u)
    assert abs(g[0, 0, vidx(3, 3, 3)] - 0.3) < 1e-12
    assert g[1, 0, vidx(3, 3, 3)] == 0 and g[2, 0, vidx(3, 3, 3)] == 0
    assert g[0, 0, vidx(4, 3, 3)] == 0                         # S:210 (u_{i+1} ∈ Ω̄)


def test_gradient_zero_across_unallocated_block_and_omega_bar():
    c = np.array([[0, 0, 0], [1, 0, 0]], np.int32)
    W = np.ones((2, 512), np.float32)
    nbr = oracle.neighbours(c)
    u = np.random.default_rng(0).normal(size=(2, 512))
    g = oracle.gradient(nbr, W, u)
    # x = 7 of block 0 → x = 0 of block 1 (allocated): difference
    assert g[0, 0, vidx(7, 2, 2)] == u[1, vidx(0, 2, 2)] - u[0, vidx(7, 2, 2)]
    # x = 7 of block 1 → unallocated (2,0,0): 0 (Eq. 3 "i = V_x", reading c-7)
    assert g[0, 1, vidx(7, 2, 2)] == 0
    # +y of y = 7 → unallocated
    assert g[1, 0, vidx(2, 7, 2)] == 0
    W[1, vidx(0, 2, 2)] = 0
    g = oracle.gradient(nbr, W, u)
    assert g[0, 0, vidx(7, 2, 2)] == 0 and np.all(g[:, 1, vidx(0, 2, 2)] == 0)


# ----------------------------------------------------------------------------- divergence (Eq. 4)

def test_divergence_worked_examples():
    c, W, nbr = one_block(W_all=1.0)
    p = np.zeros((3, 1, 512))
    i = vidx(4, 4, 4)
    im = vidx(3, 4, 4)
    p[0, 0, i] = 0.2
    p[0, 0, im] = 0.5
    d = oracle.divergence(nbr, W, p)
    assert abs(d[0, i] - (-0.3)) < 1e-12
    W2 = W.copy()
    W2[0, i] = 0
    assert oracle.divergence(nbr, W2, p)[0, i] == 0           # S:219 centre ∈ Ω̄
    W3 = W.copy()
    W3[0, im] = 0
    assert abs(oracle.divergence(nbr, W3, p)[0, i] - 0.2) < 1e-15   # S:220 left ∈ Ω̄ → p_i


@pytest.mark.parametrize("seed", range(100))
def test_adjointness_random_masks(seed):
    # <∇u, p> + <u, div p> = 0 over 100 random 16^3 grids (2x2x2 blocks), Ω density 10-90 %
    g = np.random.default_rng(seed)
    dens = 0.1 + 0.8 * (seed / 99.0)
    s = dense_box(2, 2, 2, seed=seed, w_density=dens)
    # drop a random block now and then so unallocated neighbours occur too
    keep = np.ones(8, bool)
    if seed % 3 == 0:
        keep[g.integers(0, 8)] = False
    c = s.coords.numpy()[keep]
    W = s.W.numpy()[keep]
    nbr = oracle.neighbours(c)
    u = g.normal(size=(c.shape[0], 512))
    p = g.normal(size=(3, c.shape[0], 512))
    gr = oracle.gradient(nbr, W, u)
    dv = oracle.divergence(nbr, W, p)
    lhs = float(np.sum(gr * p))
    rhs = float(np.sum(u * dv))
    scale = float(np.sum(np.abs(gr * p)) + np.sum(np.abs(u * dv))) + 1e-300
    assert abs(lhs + rhs) <= 1e-12 * scale


def test_operator_norm_bound():
    # ‖∇_Ω‖² ≤ 12 (the CP step condition τσ‖∇‖² ≤ 1 with τσ = 1/12): power iteration on −div∇
    for s, lo in ((dense_box(2, 2, 2, seed=1), 11.0), (random_instance(60, seed=4, extent=3), 0.0)):
        c, W = s.coords.numpy(), s.W.numpy()
        nbr = oracle.neighbours(c)
        x = np.random.default_rng(0).normal(size=(c.shape[0], 512))
        lam = 0.0
        for _ in range(300):
            y = -oracle.divergence(nbr, W, oracle.gradient(nbr, W, x))
            lam = float(np.sum(x * y) / np.sum(x * x))
            x = y / np.linalg.norm(y)
        assert lo <= lam <= 12.0 + 1e-9


# ------------------------------------------------------------------------ single steps via 1 iteration

def _state(n=1):
    return np.zeros((n, 512)), np.zeros((n, 512)), np.zeros((3, n, 512))


def test_dual_step_worked_examples():
    c, W, nbr = one_block([(3, 3, 3), (4, 3, 3)])
    f = np.zeros((1, 512), np.float32)
    u, ub, p = _state()
    ub[0, vidx(4, 3, 3)] = 1.0                                  # ∇ū(v) = (1, 0, 0)
    v = vidx(3, 3, 3)
    _, _, p1 = oracle.regularise(c, f, W, 1.0, 0.0, 1 / 6, 0.5, 1, state=(u, ub, p), nbr=nbr)
    assert np.allclose(p1[:, 0, v], [0.5, 0, 0], atol=0, rtol=0)
    _, _, p2 = oracle.regularise(c, f, W, 1.0, 0.01, 1 / 6, 0.5, 1, state=(u, ub, p), nbr=nbr)
    assert abs(p2[0, 0, v] - 0.5 / 1.005) < 1e-9                             # Huber ε = 0.01
    u, ub, p = _state()
    p[:, 0, v] = [3.0, 4.0, 0.0]                                             # p̃ = (3, 4, 0)
    _, _, p3 = oracle.regularise(c, f, W, 1.0, 0.0, 1 / 6, 0.5, 1, state=(u, ub, p), nbr=nbr)
    assert np.allclose(p3[:, 0, v], [0.6, 0.8, 0.0], atol=1e-15)


def test_primal_step_worked_examples():
    c, W, nbr = one_block([(3, 3, 3)])                          # isolated: div p = 0
    v = vidx(3, 3, 3)
    f = np.zeros((1, 512), np.float32)
    f[0, v] = 0.2
    u, ub, p = _state()
    u[0, v] = 0.5
    uL2, _, _ = oracle.regularise(c, f, W, 0.8, 0.0, 1 / 6, 0.5, 1, data_term=1, state=(u, ub, p), nbr=nbr)
    assert abs(uL2[0, v] - 0.46470588) < 1e-7
    uL1, _, _ = oracle.regularise(c, f, W, 0.8, 0.0, 1 / 6, 0.5, 1, data_term=0, state=(u, ub, p), nbr=nbr)
    assert abs(uL1[0, v] - 0.36666667) < 1e-7                                # r = 0.3 > t = 0.1333
    u[0, v] = f[0, v]
    for dt in (0, 1):                                                        # S:237 fixed point
        uf, _, _ = oracle.regularise(c, f, W, 0.8, 0.0, 1 / 6, 0.5, 1, data_term=dt, state=(u, ub, p), nbr=nbr)
        assert uf[0, v] == np.float64(np.float32(0.2))


def test_relax_worked_examples():
    c, W, nbr = one_block([(3, 3, 3)])
    v = vidx(3, 3, 3)
    f = np.zeros((1, 512), np.float32)
    f[0, v] = 1.0
    u, ub, p = _state()
    u[0, v] = 0.4                       # L1 with t = 0.25·0.4·1 = 0.1: u' = 0.4 + 0.1 = 0.5
    u1, ub1, _ = oracle.regularise(c, f, W, 0.4, 0.0, 0.25, 0.25, 1, theta=1.0, state=(u, ub, p), nbr=nbr)
    assert abs(u1[0, v] - 0.5) < 1e-7 and abs(ub1[0, v] - 0.6) < 1e-7
    u0, ub0, _ = oracle.regularise(c, f, W, 0.4, 0.0, 0.25, 0.25, 1, theta=0.0, state=(u, ub, p), nbr=nbr)
    assert ub0[0, v] == u0[0, v]                                             # S:247 θ = 0


def test_omega_bar_dual_is_zero():
    c, W, nbr = one_block([(3, 3, 3)])
    f = np.zeros((1, 512), np.float32)
    u, ub, p = _state()
    p[:, 0, :] = 0.3
    _, _, p1 = oracle.regularise(c, f, W, 1.0, 0.0, 0.2, 0.2, 1, state=(u, ub, p), nbr=nbr)
    mask = W[0] == 0
    assert np.all(p1[:, 0, mask] == 0)


# ---------------------------------------------------------------------------------------- energy

def test_energy_worked_examples():
    c, W, nbr = one_block(W_all=3.0)
    f = np.full((1, 512), 0.37, np.float32)
    P, _ = oracle.energy(nbr, f, W, f.astype(np.float64), 0.8, 0.0)
    assert P == 0.0
    c, W, nbr = one_block([(3, 3, 3), (4, 3, 3)])
    u = np.zeros((1, 512))
    u[0, vidx(4, 3, 3)] = 1.0
    for lam in (0.1, 5.0):
        P, _ = oracle.energy(nbr, u.astype(np.float32), W, u, lam, 0.0)
        assert P == 1.0


def _numpy_energy(s, u, lam, eps, data_term):
    lo, alloc, (ud, fd, Wd) = dn.to_dense(s.coords.numpy(), u, s.f.numpy().astype(np.float64),
                                         s.W.numpy().astype(np.float64))
    om = alloc & (Wd > 0)
    g = dn.gradient(ud, om)
    nrm = np.sqrt(g[0] ** 2 + g[1] ** 2 + g[2] ** 2)
    if eps > 0:
        H = np.where(nrm <= eps, nrm ** 2 / (2 * eps), nrm - eps / 2)
    else:
        H = nrm
    r = ud - fd
    D = lam * Wd * np.abs(r) if data_term == 0 else 0.5 * lam * Wd * r * r
    return float(np.sum(np.where(om, H + D, 0.0)))


@pytest.mark.parametrize("eps,dt", [(0.0, 0), (0.05, 0), (0.0, 1), (0.05, 1)])
def test_energy_brute_force(eps, dt):
    s = random_instance(50, seed=7, extent=3)
    u = np.random.default_rng(1).normal(size=(50, 512))
    lam = float(np.float32(0.7))
    P, _ = oracle.energy(oracle.neighbours(s.coords), s.f, s.W, u, lam, float(np.float32(eps)), dt)
    ref = _numpy_energy(s, u, lam, float(np.float32(eps)), dt)
    assert abs(P - ref) <= 1e-10 * abs(ref)


@pytest.mark.parametrize("dt", [0, 1])
def test_weak_duality_random(dt):
    s = random_instance(40, seed=9, extent=3)
    nbr = oracle.neighbours(s.coords)
    g = np.random.default_rng(2)
    for _ in range(5):
        u = g.normal(size=(40, 512))
        p = g.normal(size=(3, 40, 512))
        p /= np.maximum(1.0, np.sqrt((p ** 2).sum(0)))[None]
        P, D = oracle.energy(nbr, s.f, s.W, u, 0.5, 0.02, dt, p=p)
        assert D <= P + 1e-9 * abs(P)
