"""Pins of the whole oracle iteration (SURVEY §8(c) rows 'Whole iteration (exact)', '(closed form,
1-D embedded)', '(dense equivalence)', 'Convergence behaviour').  CPU only."""
import math

import numpy as np
import pytest

import oracle
import oracle.dense as dn
from synth import dense_box, line_indices, line_scene, random_instance

F32 = lambda x: float(np.float32(x))


# ------------------------------------------------------------------ O1 (hashed blocks) == O2 (dense)

CASES = [
    dict(box=(2, 2, 2), w_density=1.0, lam=0.5, eps=0.0, data_term=0, init=0),
    dict(box=(3, 2, 1), w_density=0.6, lam=0.3, eps=0.05, data_term=0, init=0),
    dict(box=(2, 1, 2), w_density=0.8, lam=1.2, eps=0.0, data_term=1, init=0),
    dict(box=(2, 2, 1), w_density=0.5, lam=0.7, eps=0.02, data_term=1, init=1),
    dict(box=(1, 2, 2), w_density=0.9, lam=0.4, eps=0.0, data_term=0, init=1),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_hvg_equals_dense_brute_force(case, prec):
    s = dense_box(*case["box"], seed=11, w_density=case["w_density"], lam=case["lam"], eps=case["eps"],
                  data_term=case["data_term"], init=case["init"], iters=25)
    u1, _, _ = oracle.regularise_scene(s, precision=prec)
    u2 = dn.regularise(s.coords.numpy(), s.f.numpy(), s.W.numpy(), s.lam, s.eps, s.tau, s.sigma, s.iters,
                       data_term=s.data_term, init=s.init, dtype=np.float64 if prec == "f64" else np.float32)
    assert np.array_equal(u1, u2)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_hvg_equals_dense_random_block_sets(seed):
    # irregular allocation: missing blocks act as Ω̄; caller order is random
    s = random_instance(45, seed=seed, extent=3, w_density=0.75, iters=30, eps=0.01 * seed,
                        data_term=seed % 2)
    for prec, dt in (("f64", np.float64), ("f32", np.float32)):
        u1, _, _ = oracle.regularise_scene(s, precision=prec)
        u2 = dn.regularise(s.coords.numpy(), s.f.numpy(), s.W.numpy(), s.lam, s.eps, s.tau, s.sigma, s.iters,
                           data_term=s.data_term, dtype=dt)
        assert np.array_equal(u1, u2)


# --------------------------------------------------------------------------- exact invariants

def test_constant_f_is_preserved_bitwise():
    # constant f on a connected Ω → u = f (within 1e-9).  TV-L1 keeps it bitwise; the L2 prox
    # (f + t f)/(1 + t) rounds to within one ulp in fp32.
    s = dense_box(2, 2, 1, seed=1, w_density=1.0, lam=0.3, iters=50)
    s.f[:] = 0.3125
    u, _, _ = oracle.regularise_scene(s, precision="f32")
    assert np.all(u == np.float32(0.3125))
    s.data_term = 1
    u, _, _ = oracle.regularise_scene(s, precision="f64")
    assert np.abs(u - 0.3125).max() <= 1e-9
    u, _, _ = oracle.regularise_scene(s, precision="f32")
    assert np.abs(u - 0.3125).max() <= 1e-7


def test_omega_bar_untouched_and_pinned_voxels(tiny_scene, tiny_oracle):
    s = tiny_scene
    f, W = s.f.numpy(), s.W.numpy()
    for key in ("u32", "u64"):
        u = tiny_oracle[key]
        bar = W == 0
        assert np.array_equal(u[bar], f[bar].astype(u.dtype))          # S:270 Ω̄ bitwise = f
        # L1 warm start: λW ≥ 3+√3 ⇒ u ≡ f (|div p| ≤ 3+√3 for ‖p‖₂ ≤ 1; the λ→∞ case)
        pin = (W > 0) & (s.lam * W >= 3 + math.sqrt(3))
        assert pin.sum() > 0.5 * (W > 0).sum()
        assert np.array_equal(u[pin], f[pin].astype(u.dtype))
        assert np.abs(u - f).max() > 0.01                              # the rest does move


def test_pinned_voxels_equal_f_at_every_checkpoint(tiny_scene):
    s = tiny_scene
    nbr = oracle.neighbours(s.coords)
    f, W = s.f.numpy(), s.W.numpy()
    pin = (W > 0) & (s.lam * W >= 3 + math.sqrt(3))
    state = None
    for _ in range(4):
        state = oracle.regularise_scene(s, precision="f32", iters=3, state=state, nbr=nbr)
        assert np.array_equal(state[0][pin], f[pin])


def test_feasibility_every_iteration(tiny_stress_scene):
    s = tiny_stress_scene
    nbr = oracle.neighbours(s.coords)
    state = None
    for _ in range(10):
        state = oracle.regularise_scene(s, precision="f64", iters=1, state=state, nbr=nbr)
        assert np.sqrt((state[2] ** 2).sum(0)).max() <= 1 + 1e-9


def test_disjoint_components_independent():
    # S:273 / S:553: two Ω components separated by a W = 0 slab; perturbing one leaves the other bitwise equal
    s = dense_box(3, 1, 1, seed=2, w_density=1.0, lam=0.4, iters=40)
    W = s.W.numpy()
    W[1, :] = 0                                                     # middle block unobserved
    s2 = dense_box(3, 1, 1, seed=2, w_density=1.0, lam=0.4, iters=40)
    s2.W[:] = s.W
    s2.f[0] += 0.25 * np.random.default_rng(0).normal(size=512).astype(np.float32)
    u1, _, _ = oracle.regularise_scene(s, precision="f32")
    u2, _, _ = oracle.regularise_scene(s2, precision="f32")
    assert np.array_equal(u1[2], u2[2]) and not np.array_equal(u1[0], u2[0])


def test_sign_symmetry():
    # f → −f ⇒ u → −u bitwise (the iteration is odd in (f, u, ū, p))
    s = random_instance(30, seed=3, extent=2, iters=40, eps=0.01)
    u1, _, _ = oracle.regularise_scene(s, precision="f32")
    s.f = -s.f
    u2, _, _ = oracle.regularise_scene(s, precision="f32")
    assert np.array_equal(u1, -u2)


def test_permutation_and_translation_invariance():
    s = random_instance(40, seed=4, extent=3, iters=30)
    u1, _, _ = oracle.regularise_scene(s, precision="f32")
    perm = np.random.default_rng(0).permutation(40)
    s2 = random_instance(40, seed=4, extent=3, iters=30)
    s2.coords = s.coords[perm] + 1000
    s2.f = s.f[perm]
    s2.W = s.W[perm]
    u2, _, _ = oracle.regularise_scene(s2, precision="f32")
    assert np.array_equal(u1[perm], u2)


def test_resume_is_bitwise_equal_to_one_run():
    s = random_instance(30, seed=5, extent=2, iters=0, eps=0.02)
    nbr = oracle.neighbours(s.coords)
    a = oracle.regularise_scene(s, precision="f32", iters=17, nbr=nbr)
    a = oracle.regularise_scene(s, precision="f32", iters=13, state=a, nbr=nbr)
    b = oracle.regularise_scene(s, precision="f32", iters=30, nbr=nbr)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_zero_iterations_returns_initial_state():
    s = random_instance(10, seed=6, extent=2)
    u, ub, p = oracle.regularise_scene(s, iters=0)
    assert np.array_equal(u, s.f.numpy().astype(np.float64)) and not p.any()
    s.init = 1
    u, _, _ = oracle.regularise_scene(s, iters=0)
    W = s.W.numpy()
    assert np.all(u[W > 0] == 0) and np.array_equal(u[W == 0], s.f.numpy()[W == 0].astype(np.float64))


# ------------------------------------------------------------- closed forms of the 1-D embedding

def _line_u(s, prec="f64"):
    u, _, _ = oracle.regularise_scene(s, precision=prec)
    return np.array([u[b, v] for b, v in line_indices(s)])


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("lam,kept", [(0.2, True), (0.1, False)])
def test_tvl1_step_closed_form(axis, lam, kept):
    # TV-L1 1-D step at m of n with uniform W: kept iff λW·min(m, n−m) > 1, else the minority side
    # is flattened to the majority value (contrast-invariant; SURVEY finding 8)
    n, m, c = 24, 8, 5.0
    f = np.where(np.arange(n) < m, 0.0, c)
    s = line_scene(f, 1.0, axis=axis, lam=lam, iters=20000)
    u = _line_u(s)
    want = f if kept else np.full(n, c)
    assert np.abs(u - want).max() < 1e-4


@pytest.mark.parametrize("lam,kept", [(0.7, True), (0.3, False)])
def test_tvl1_bump_closed_form(lam, kept):
    # interior bump of width L: kept iff λW·L > 2
    n, a, L, c = 24, 9, 4, 2.0
    f = np.where((np.arange(n) >= a) & (np.arange(n) < a + L), c, 0.0)
    s = line_scene(f, 1.0, axis=1, lam=lam, iters=20000)
    u = _line_u(s)
    want = f if kept else np.zeros(n)
    assert np.abs(u - want).max() < 1e-4


@pytest.mark.parametrize("c,w", [(0.3, 1.0), (0.1, 1.0), (0.6, 2.0)])
def test_rof_step_closed_form(c, w):
    # L2 (ROF, paper Eq. 8 prox of (λW/2)(u−f)²): if c·λW > 1/m + 1/(n−m) the plateaus are
    # 1/(λW m) and c − 1/(λW (n−m)); otherwise u is the constant mean
    n, m = 24, 8
    lam = F32(1.0 if w == 1.0 else 0.5)
    lw = lam * w
    f = np.where(np.arange(n) < m, 0.0, c).astype(np.float32).astype(np.float64)
    s = line_scene(f, w, axis=2, lam=lam, data_term=1, iters=20000)
    u = _line_u(s)
    if c * lw > 1.0 / m + 1.0 / (n - m):
        want = np.where(np.arange(n) < m, 1.0 / (lw * m), f[-1] - 1.0 / (lw * (n - m)))
    else:
        want = np.full(n, f.mean())
    assert np.abs(u - want).max() < 1e-4


def _tvl1_dp_min(f, lw):
    """Exact minimum of the 1-D TV-L1 energy Σ|u_{i+1} − u_i| + lw·Σ|u_i − f_i| (SURVEY §8(c) '1-D exact
    minimiser'): a minimiser exists with every value in {f_j} (the energy is piecewise linear and its
    breakpoints in each u_i are the data values), so dynamic programming over those levels is exact."""
    levels = np.unique(f)
    V = lw * np.abs(levels - f[0])
    jump = np.abs(levels[:, None] - levels[None, :])
    for fi in f[1:]:
        V = lw * np.abs(levels - fi) + (V[None, :] + jump).min(axis=1)
    return float(V.min())


@pytest.mark.parametrize("seed,lam", [(1, 0.35), (2, 0.6), (3, 0.9)])
def test_tvl1_1d_energy_reaches_exact_dp_minimum(seed, lam):
    # random 1-D data (not a closed-form case): the CP iterate's energy must reach the exact minimum
    rng = np.random.default_rng(seed)
    n = 24
    f = np.round(rng.normal(0.0, 1.0, n), 2).astype(np.float32).astype(np.float64)
    lam = F32(lam)
    s = line_scene(f, 1.0, axis=seed % 3, lam=lam, iters=30000)
    u = _line_u(s)
    E = float(np.abs(np.diff(u)).sum() + lam * np.abs(u - f).sum())
    Emin = _tvl1_dp_min(f, lam)
    assert Emin <= E + 1e-9                      # the DP value is a true lower bound
    assert E - Emin <= 1e-4 * max(1.0, Emin)     # and the iterate attains it


@pytest.mark.parametrize("seed,lam,w", [(4, 0.8, 1.0), (5, 2.0, 3.0)])
def test_rof_1d_matches_exact_minimiser(seed, lam, w):
    # 1-D weighted ROF (paper Eq. 8 data term (λW/2)(u − f)²) solved exactly through its dual, a
    # box-constrained least-squares problem: u* = f − Dᵀp*/(λW), p* = argmin_{|p| ≤ 1} ‖Dᵀp/√(λW) − √(λW) f‖²
    from scipy.optimize import lsq_linear
    rng = np.random.default_rng(seed)
    n = 24
    f = rng.normal(0.0, 1.0, n).astype(np.float32).astype(np.float64)
    lam = F32(lam)
    lw = lam * w
    D = np.zeros((n - 1, n))
    D[np.arange(n - 1), np.arange(n - 1)] = -1.0
    D[np.arange(n - 1), np.arange(1, n)] = 1.0
    r = lsq_linear(D.T / np.sqrt(lw), np.sqrt(lw) * f, bounds=(-1.0, 1.0), tol=1e-14, lsmr_tol="auto", max_iter=10000)
    u_star = f - D.T @ r.x / lw
    s = line_scene(f, w, axis=seed % 3, lam=lam, data_term=1, iters=20000)
    u = _line_u(s)
    assert np.abs(u - u_star).max() < 1e-5


def test_l2_zero_and_warm_init_reach_same_minimiser():
    s = random_instance(8, seed=7, extent=1, data_term=1, lam=2.0, iters=3000)
    a, _, _ = oracle.regularise_scene(s)
    s.init = 1
    b, _, _ = oracle.regularise_scene(s)
    assert np.abs(a - b).max() < 1e-5


# --------------------------------------------------------------------------- convergence behaviour

def test_energy_checkpoints_and_gap(tiny_scene):
    s = tiny_scene
    nbr = oracle.neighbours(s.coords)
    f = s.f.numpy()
    E0, _ = oracle.energy(nbr, s.f, s.W, f.astype(np.float64), s.lam, s.eps, s.data_term)
    state = None
    Es, gaps, it = [E0], [], 0
    for target in (10, 20, 50, 100, 200):
        state = oracle.regularise_scene(s, iters=target - it, state=state, nbr=nbr)
        it = target
        P, D = oracle.energy(nbr, s.f, s.W, state[0], s.lam, s.eps, s.data_term, p=state[2])
        Es.append(P)
        gaps.append(P - D)
    # non-increasing at the checkpoints (rel. tol 1e-6, reading c-16), strictly lower at the end
    for a, b in zip(Es, Es[1:]):
        assert b <= a * (1 + 1e-6)
    assert Es[-1] < Es[0]
    assert all(g >= -1e-9 * abs(E0) for g in gaps)                     # weak duality
    assert gaps[-1] < gaps[0]


def test_l2_gap_shrinks(tiny_scene):
    s = tiny_scene
    nbr = oracle.neighbours(s.coords)
    state, it, gaps = None, 0, []
    for target in (1, 10, 50, 100, 200):
        state = oracle.regularise(s.coords, s.f, s.W, s.lam, 0.0, s.tau, s.sigma, target - it, data_term=1,
                                  state=state, nbr=nbr)
        it = target
        P, D = oracle.energy(nbr, s.f, s.W, state[0], s.lam, 0.0, 1, p=state[2])
        gaps.append(P - D)
    assert all(b < a for a, b in zip(gaps, gaps[1:]))
    assert gaps[-1] >= 0


def test_fp32_close_to_fp64(tiny_oracle):
    # reading c-18: fp32 drift after the config's 200 iterations stays below the 1e-5 parity budget
    assert np.abs(tiny_oracle["u32"] - tiny_oracle["u64"]).max() < 5e-6


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_openmp_timing_build_is_bitwise_the_plain_oracle(tiny_scene, prec):
    """liboracle_omp.so (bench.py cpu_baseline_omp) runs the same phase loops over all host cores; every
    phase reads a frozen snapshot, so the result must equal the plain build bit for bit."""
    s = tiny_scene
    a = oracle.regularise_scene(s, precision=prec, iters=25)
    b = oracle.regularise(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, 25, theta=s.theta,
                          data_term=s.data_term, init=s.init, precision=prec, omp=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_phase_split_composes_to_the_iteration():
    """oracle.phase (dual = Eq. 3 + Eq. 7, primal = Eq. 4 + Eq. 8 + Eq. 9) applied alternately equals
    oracle.regularise bit for bit, in both precisions; a primal phase alone on the initial state (p = 0)
    leaves u = f, and a dual phase alone from u = ū = f gives the projected σ-scaled gradient of f."""
    import oracle
    from synth import random_instance
    s = random_instance(60, seed=5, extent=3, w_density=0.8, lam=0.7, eps=0.02, iters=7)
    nbr = oracle.neighbours(s.coords)
    for prec in ("f32", "f64"):
        ref = oracle.regularise_scene(s, precision=prec, nbr=nbr)
        st = oracle.regularise_scene(s, precision=prec, iters=0, nbr=nbr)
        for _ in range(s.iters):
            oracle.phase(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, "dual", st, precision=prec, nbr=nbr)
            oracle.phase(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, "primal", st, precision=prec, nbr=nbr)
        for a, b in zip(st, ref):
            assert np.array_equal(a, b)
    st = oracle.regularise_scene(s, precision="f64", iters=0, nbr=nbr)
    oracle.phase(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, "primal", st, nbr=nbr)
    assert np.array_equal(st[0], s.f.numpy().astype(np.float64))
    st = oracle.regularise_scene(s, precision="f64", iters=0, nbr=nbr)
    oracle.phase(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, "dual", st, nbr=nbr)
    g = oracle.gradient(nbr, s.W, s.f.numpy().astype(np.float64))
    q = np.float64(np.float32(s.sigma)) * g * (1.0 / (1.0 + np.float64(np.float32(s.sigma)) * np.float64(np.float32(s.eps))))
    nrm = np.sqrt((q ** 2).sum(0))
    assert np.allclose(st[2], q / np.maximum(1.0, nrm)[None], rtol=1e-14, atol=1e-15)


def test_native_timing_build_is_bitwise_the_oracle():
    """bench.py's CPU baselines run the -O3 -march=native build; it must compute the same
    bits as the parity oracle (no contraction, no fast-math, independent per-voxel loops)."""
    import oracle
    from synth import random_instance
    s = random_instance(150, seed=8, extent=4, w_density=0.8, lam=0.6, eps=0.02, iters=15)
    nbr = oracle.neighbours(s.coords)
    for prec in ("f32", "f64"):
        kw = dict(theta=s.theta, data_term=s.data_term, init=s.init, precision=prec, nbr=nbr)
        a = oracle.regularise(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, s.iters, **kw)
        b = oracle.regularise(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, s.iters, native=True, **kw)
        c = oracle.regularise(s.coords, s.f, s.W, s.lam, s.eps, s.tau, s.sigma, s.iters, native=True, omp=True, **kw)
        for x, y, z in zip(a, b, c):
            assert np.array_equal(x, y) and np.array_equal(x, z)
