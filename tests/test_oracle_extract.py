"""Pins of the extraction oracle (oracle/extract_oracle.c, readings X-1 … X-7).

Each pin is fixed by geometry, not by the oracle's code:
  * planar fields u = n·p − c: linear interpolation is exact, so every vertex lies on the plane; the
    triangulated surface of an axis-aligned plane has exactly the area of the cell region's cross
    section; every normal points toward u > 0;
  * an analytic sphere SDF: a closed, consistently oriented 2-manifold (every edge shared by exactly two
    triangles, used once in each direction), Euler characteristic 2, vertices within interpolation
    error of the sphere, area and enclosed volume within 1 % of 4πr² and 4πr³/3;
  * Ω restriction: no geometry in cells with an unobserved or unallocated corner;
  * empty input → empty mesh.
"""
import math

import numpy as np
import pytest

import oracle
from synth import dense_box

V = 0.1


def _grid(coords):
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    return coords.astype(np.int64)[:, None, :] * 8 + loc[None]


def _centres(coords, v=V):
    return (_grid(coords).astype(np.float64) + 0.5) * v


def _normals(T):
    T = T.astype(np.float64)
    return np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])


def _edges(T):
    """Directed edges of all triangles as tuples of exact vertex bit patterns."""
    key = [tuple(map(tuple, t)) for t in T.view(np.uint32).reshape(-1, 3, 3)]
    return [(t[i], t[(i + 1) % 3]) for t in key for i in range(3)]


def test_empty():
    s = dense_box(1, 1, 1)
    c = s.coords.numpy()
    assert oracle.extract(c, np.ones((1, 512), np.float32), np.zeros((1, 512), np.float32), V).shape[0] == 0
    # a constant field has no zero crossing
    assert oracle.extract(c, np.ones((1, 512), np.float32), np.ones((1, 512), np.float32), V).shape[0] == 0


@pytest.mark.parametrize("axis,c0", [(2, 0.73), (0, 1.012), (1, 0.455)])
def test_axis_plane_exact(axis, c0):
    s = dense_box(3, 2, 2)
    c = s.coords.numpy()
    P = _centres(c)
    u = (P[..., axis] - c0).astype(np.float32)
    T = oracle.extract(c, u, np.ones_like(u), V)
    assert np.abs(T[..., axis] - c0).max() <= 1e-6
    n = _normals(T)
    area = 0.5 * np.linalg.norm(n, axis=1).sum()
    ext = [24, 16, 16]
    others = [ext[k] - 1 for k in range(3) if k != axis]
    assert abs(area - others[0] * others[1] * V * V) <= 1e-5 * area
    assert (n[:, axis] > 0).all()                      # toward u > 0 (free space)


@pytest.mark.parametrize("seed", range(4))
def test_tilted_plane(seed):
    rng = np.random.default_rng(seed)
    nrm = rng.normal(size=3)
    nrm /= np.linalg.norm(nrm)
    s = dense_box(2, 2, 2)
    c = s.coords.numpy()
    P = _centres(c)
    off = float(nrm @ np.array([0.8, 0.8, 0.8]))
    u = (P @ nrm - off).astype(np.float32)
    T = oracle.extract(c, u, np.ones_like(u), V)
    assert T.shape[0] > 100
    assert np.abs(T.astype(np.float64) @ nrm - off).max() <= 2e-6
    n = _normals(T)
    assert (n @ nrm > 0).all()
    # every edge interior to the region is shared by exactly two triangles in opposite directions
    E = _edges(T)
    cnt = {}
    for e in E:
        cnt[e] = cnt.get(e, 0) + 1
    assert max(cnt.values()) == 1                      # no directed edge repeated (consistent orientation)


def _sphere(radius_vox=10.5, blocks=3, centre_vox=12.3):
    s = dense_box(blocks, blocks, blocks)
    c = s.coords.numpy()
    P = _centres(c)
    ctr = centre_vox * V
    r = radius_vox * V
    u = (np.linalg.norm(P - ctr, axis=-1) - r).astype(np.float32)
    return c, u, ctr, r


def test_sphere_closed_manifold():
    c, u, ctr, r = _sphere()
    T = oracle.extract(c, u, np.ones_like(u), V)
    E = _edges(T)
    d = {}
    for e in E:
        d[e] = d.get(e, 0) + 1
    assert max(d.values()) == 1
    for (a, b) in d:
        assert (b, a) in d                             # closed: every edge used once in each direction
    verts = {v for t in T.view(np.uint32).reshape(-1, 3, 3) for v in map(tuple, t)}
    undirected = {tuple(sorted(e)) for e in d}
    assert len(verts) - len(undirected) + T.shape[0] == 2     # Euler characteristic of a sphere
    rad = np.linalg.norm(T.astype(np.float64).reshape(-1, 3) - ctr, axis=1)
    assert np.abs(rad - r).max() <= 0.1 * V
    n = _normals(T)
    area = 0.5 * np.linalg.norm(n, axis=1).sum()
    assert abs(area / (4 * math.pi * r * r) - 1) <= 0.01
    # enclosed volume by the divergence theorem; positive = outward orientation
    T64 = T.astype(np.float64) - ctr
    vol = np.einsum("ij,ij->i", T64[:, 0], np.cross(T64[:, 1], T64[:, 2])).sum() / 6.0
    assert abs(vol / (4.0 / 3.0 * math.pi * r ** 3) - 1) <= 0.01


def test_omega_restriction():
    c, u, ctr, r = _sphere()
    g = _grid(c)
    W = np.ones_like(u)
    W[g[..., 0] < 12] = 0.0                            # unobserved half-space
    T = oracle.extract(c, u, W, V)
    assert T.shape[0] > 0
    assert T[..., 0].min() >= (12 + 0.5) * V - 1e-6    # every vertex inside the observed cells
    full = oracle.extract(c, u, np.ones_like(u), V)
    assert T.shape[0] < full.shape[0]
    # w_min restricts further, unallocated blocks act like Ω̄
    W2 = np.where(g[..., 1] < 14, 1.0, 3.0).astype(np.float32)
    T2 = oracle.extract(c, u, W2, V, w_min=2.0)
    assert T2.shape[0] > 0 and T2[..., 1].min() >= (14 + 0.5) * V - 1e-6
    keep = ~((c[:, 0] == 0) & (c[:, 1] == 0) & (c[:, 2] == 0))
    T3 = oracle.extract(c[keep], u[keep], np.ones_like(u[keep]), V)
    assert T3.shape[0] < full.shape[0]
    assert not (np.all(T3 < 8.5 * V, axis=(1, 2))).any()    # nothing in cells touching the removed block
    E = _edges(T3)
    assert len(set(E)) == len(E)


def test_caller_block_order_only_permutes_blocks():
    c, u, ctr, r = _sphere(blocks=2, centre_vox=8.1, radius_vox=5.2)
    T = oracle.extract(c, u, np.ones_like(u), V)
    perm = np.random.default_rng(0).permutation(c.shape[0])
    T2 = oracle.extract(c[perm], u[perm], np.ones_like(u), V)
    key = lambda A: sorted(map(bytes, A.view(np.uint8).reshape(A.shape[0], -1)))
    assert key(T) == key(T2)


def test_degenerate_triangles_dropped():
    """X-6: corners with u exactly 0 collapse edge vertices onto the corner; such triangles are
    dropped, every emitted triangle has three distinct vertices, and the surface stays manifold."""
    s = dense_box(2, 2, 2)
    c = s.coords.numpy()
    # integer-valued fields on the voxel lattice: many corners exactly 0, every zero/sign combination
    u = np.random.default_rng(5).integers(-2, 3, size=(c.shape[0], 512)).astype(np.float32)
    assert (u == 0).sum() > 100
    T = oracle.extract(c, u, np.ones_like(u), V)
    assert T.shape[0] > 0
    b = T.view(np.uint32).reshape(-1, 3, 3)
    same = lambda i, j: (b[:, i] == b[:, j]).all(-1)
    assert not (same(0, 1) | same(1, 2) | same(0, 2)).any()
    # every emitted triangle has a genuine area (the integer field puts vertices at small rationals of
    # the voxel size, so a non-degenerate triangle has area >= v²/1000), every dropped one had none
    area = 0.5 * np.linalg.norm(_normals(T), axis=1)
    assert area.min() >= V * V / 1000
    # (with arbitrary zero patterns the zero set may touch itself, so no manifold claim here; a smooth
    # integer field with zeros keeps it)
    g = _grid(c)
    u2 = (g[..., 0] + g[..., 1] - g[..., 2] - 3).astype(np.float32)
    T2 = oracle.extract(c, u2, np.ones_like(u2), V)
    E = _edges(T2)
    assert len(set(E)) == len(E)
    assert (0.5 * np.linalg.norm(_normals(T2), axis=1)).min() >= V * V / 1000


def test_extract64_planar_field_vertices_on_plane():
    """Pin of the float64 extraction (oracle/extract64.py): on a planar field u = n·p − c the linear
    interpolation of X-4 is exact, so in float64 every vertex lies on the plane to ~1e-12, and every
    normal points toward u > 0 (X-5, decided there by a determinant, not a parity)."""
    from oracle.extract64 import extract_f64
    c = dense_box(2, 2, 2).coords.numpy()
    P = _centres(c)
    n = np.array([0.3, -0.5, 0.81])
    n /= np.linalg.norm(n)
    u = (P @ n - 0.77).astype(np.float32)
    T = extract_f64(c, u, np.ones_like(u), V)
    assert T.shape[0] > 100
    # the field values are fp32 roundings of n·p − c: vertices sit on the plane of the rounded values to
    # within the rounding (1e-7 of |u|), far below any formula error
    assert np.abs(T.reshape(-1, 3) @ n - 0.77).max() <= 1e-6
    N = np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])
    assert (N @ n > 0).all()


@pytest.mark.parametrize("seed", [1, 2])
def test_extract64_matches_c_oracle(seed):
    """The float64 numpy extraction and the fp32 C oracle, written separately (orientation by determinant
    vs permutation parity), give the same triangles in the same order, vertices within fp32 rounding."""
    from oracle.extract64 import extract_f64, match_up_to_rotation
    rng = np.random.default_rng(seed)
    c = dense_box(2, 2, 2).coords.numpy()
    u = rng.normal(size=(c.shape[0], 512)).astype(np.float32)
    u[rng.random(u.shape) < 0.05] = 0.0                  # exact zeros: the X-6 drops
    W = (rng.random(u.shape) < 0.97).astype(np.float32)  # unobserved voxels: X-1
    perm = rng.permutation(c.shape[0])
    T = oracle.extract(c[perm], u[perm], W[perm], V)
    R = extract_f64(c[perm], u[perm], W[perm], V)
    assert T.shape == R.shape and T.shape[0] > 1000
    assert match_up_to_rotation(T, R) <= 1e-6
