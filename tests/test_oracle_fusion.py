"""Pins of the fusion oracle (oracle/fusion_oracle.c, oracle/dense_fusion.py) — paper §III-A, Eq. 1.

What pins it (task rule ③), each independent of the oracle's own code:
  * worked examples of step 3 and Eq. 1 (tests/golden/fusion_examples.txt, SPEC S:132-143 hand
    evaluations of P:158-176);
  * closed forms: a fronto-parallel plane seen under random rigid poses: every voxel's f is
    clamp((D − z_c)/μ) with z_c evaluated in fp64, untouched outside the image and behind D + μ; the
    running average of several planes (Eq. 1 unrolled = arithmetic mean); idempotence; the
    weight cap (F-4); the sequential allocate-then-update order (F-8);
  * brute force: the block walk and the allocated block set against exact (fp64) segment/box
    intersection with a 1e-4 m erosion/dilation; the dense legacy grid O2-fusion bit for bit.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle.dense_fusion import fuse_dense

GOLD = os.path.join(os.path.dirname(__file__), "golden", "fusion_examples.txt")


def _golden(kind):
    out = []
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        k, cite, rest = line.split(None, 2)
        if k != kind:
            continue
        lhs, rhs = rest.split("->")
        out.append((cite, [float(v) for v in lhs.split()], [float(v) for v in rhs.split()]))
    return out


@pytest.mark.parametrize("cite,inp,exp", _golden("tsdf"))
def test_tsdf_update_worked_examples(cite, inp, exp):
    f, w, sdf, mu, wmax = inp
    f2, w2, up = oracle.tsdf_update(f, w, sdf, mu, wmax if math.isfinite(wmax) else 1e30)
    assert abs(f2 - exp[0]) <= 1e-6, cite
    assert w2 == exp[1] and up == bool(exp[2]), cite


def _pose(R, t):
    return np.concatenate([np.asarray(R, np.float64), np.asarray(t, np.float64).reshape(3, 1)], 1).reshape(12).astype(np.float32)


def _rand_rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    return np.array([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                     [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                     [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]])


@pytest.mark.parametrize("cite,inp,exp", _golden("sdf"))
def test_sdf_worked_examples_through_fusion(cite, inp, exp):
    # one camera (identity rotation) at t = (¼, ¼, −¼) looking down +z; voxel 0.5 m so that the voxel
    # centres (¼, ¼, (g+½)/2) sit on the optical axis at z_c = (g+½)/2 + ¼
    d, zc, mu = inp
    intr = np.array([10, 10, 4, 4], np.float32)
    pose = _pose(np.eye(3), [0.25, 0.25, -0.25])
    depth = np.full((1, 9, 9), d, np.float32)
    xyz, first, f, W = oracle.fuse(depth, intr, pose, 0.5, mu, 100.0, 1e30)
    gz = int(round(2 * (zc - 0.25) - 0.5))
    b = np.where((xyz[:, 0] == 0) & (xyz[:, 1] == 0) & (xyz[:, 2] == gz // 8))[0]
    assert b.size == 1, cite
    v = 64 * (gz % 8)
    assert W[b[0], v] == 1.0 and abs(f[b[0], v] - exp[0]) <= 1e-7, cite


# ------------------------------------------------------------------------------------ plane closed form

INTR = np.array([60.0, 60.0, 31.5, 23.5], np.float32)
HH, WW = 48, 64


def _voxel_geometry(xyz, pose, voxel):
    """fp64 camera-frame coordinates and image coordinates of every voxel centre of the blocks."""
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    g = xyz.astype(np.int64)[:, None, :] * 8 + loc[None]
    p = (g.astype(np.float64) + 0.5) * np.float64(np.float32(voxel))
    T = pose.astype(np.float64).reshape(3, 4)
    pc = (p - T[:, 3]) @ T[:, :3]
    zc = pc[..., 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        ix = INTR[0] * pc[..., 0] / zc + INTR[2]
        iy = INTR[1] * pc[..., 1] / zc + INTR[3]
    return zc, ix, iy


def _clear_of_pixel_edges(ix, iy, tol=1e-3):
    fx = (ix + 0.5) - np.floor(ix + 0.5)
    fy = (iy + 0.5) - np.floor(iy + 0.5)
    return (np.minimum(fx, 1 - fx) > tol) & (np.minimum(fy, 1 - fy) > tol)


@pytest.mark.parametrize("seed", range(6))
def test_plane_closed_form_random_pose(seed):
    """fronto-parallel plane at depth D = 5 m, μ = 1 m, 10 cm voxels, under a random rigid pose."""
    rng = np.random.default_rng(seed)
    R = _rand_rot(rng)
    t = rng.uniform(-3, 3, size=3)
    pose = _pose(R, t)
    D, mu, voxel = 5.0, 1.0, 0.1
    depth = np.full((1, HH, WW), D, np.float32)
    xyz, first, f, W = oracle.fuse(depth, INTR, pose, voxel, mu, 100.0, 1e30)
    assert xyz.shape[0] > 50 and (first == 0).all()
    zc, ix, iy = _voxel_geometry(xyz, pose, voxel)
    inside = (zc > 0) & (np.floor(ix + 0.5) >= 0) & (np.floor(ix + 0.5) < WW) & (np.floor(iy + 0.5) >= 0) & \
             (np.floor(iy + 0.5) < HH)
    expect_upd = inside & (zc <= D + mu)
    clear = _clear_of_pixel_edges(ix, iy) & (np.abs(zc - (D + mu)) > 1e-4)
    # untouched outside the image and behind the surface by more than μ (carve protection, Eq. 1)
    assert np.array_equal(W[clear] > 0, expect_upd[clear])
    assert set(np.unique(W)) <= {0.0, 1.0}
    # f = clamp((D − z_c)/μ): the zero crossing lies between the two voxel layers nearest the plane
    sel = clear & expect_upd
    exp_f = np.clip((D - zc[sel]) / mu, -1.0, 1.0)
    assert np.abs(f[sel] - exp_f).max() <= 2e-5
    assert (f[W == 0] == 0).all()
    assert sel.sum() > 1000


def _segment_boxes(a, b, lo, Bm, delta):
    """Blocks (of edge Bm, integer coords in the range lo + [0, 6)^3) met by segment a→b, with boxes
    grown by delta (delta < 0 erodes).  Exact slab test in fp64."""
    rngs = [np.arange(lo[k], lo[k] + 6) for k in range(3)]
    X, Y, Z = np.meshgrid(*rngs, indexing="ij")
    B = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    bl = B * Bm - delta
    bh = (B + 1) * Bm + delta
    d = b - a
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (bl - a) / d
        t2 = (bh - a) / d
    tlo = np.where(d == 0, np.where((a >= bl) & (a <= bh), -np.inf, np.inf), np.minimum(t1, t2))
    thi = np.where(d == 0, np.where((a >= bl) & (a <= bh), np.inf, -np.inf), np.maximum(t1, t2))
    t0 = np.maximum(tlo.max(1), 0.0)
    t1_ = np.minimum(thi.min(1), 1.0)
    return {tuple(x) for x in B[t0 <= t1_]}


@pytest.mark.parametrize("seed", range(3))
def test_allocated_blocks_match_exact_band_intersection(seed):
    """Reading F-5/F-7: allocated blocks = blocks met by each pixel ray between depths d − μ and d + μ."""
    rng = np.random.default_rng(100 + seed)
    pose = _pose(_rand_rot(rng), rng.uniform(-2, 2, size=3))
    D, mu, voxel = 5.0, 1.0, 0.1
    Bm = 8 * np.float64(np.float32(voxel))
    depth = np.full((1, HH, WW), D, np.float32)
    xyz, first = oracle.fuse_alloc(depth, INTR, pose, voxel, mu, 100.0)
    alloc = {tuple(x) for x in xyz}
    T = pose.astype(np.float64).reshape(3, 4)
    inner, outer = set(), set()
    for j in range(0, HH):
        for i in range(0, WW):
            dc = np.array([(i - INTR[2]) / INTR[0], (j - INTR[3]) / INTR[1], 1.0])
            a = T[:, :3] @ (dc * (D - mu)) + T[:, 3]
            b = T[:, :3] @ (dc * (D + mu)) + T[:, 3]
            lo = np.floor(np.minimum(a, b) / Bm).astype(np.int64) - 1
            inner |= _segment_boxes(a, b, lo, Bm, -1e-4)
            outer |= _segment_boxes(a, b, lo, Bm, 1e-4)
    assert inner <= alloc <= outer
    assert len(alloc) >= 0.99 * len(inner)


@pytest.mark.parametrize("seed", range(40))
def test_block_walk_exact(seed):
    rng = np.random.default_rng(seed)
    Bm = 0.4
    a = rng.uniform(-3, 3, size=3).astype(np.float32)
    b = (a + rng.uniform(-2, 2, size=3)).astype(np.float32)
    if seed % 5 == 0:
        b[seed % 3] = a[seed % 3]          # axis-parallel cases
    cells = oracle.block_walk(a, b, Bm)
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    Bm32 = np.float64(np.float32(Bm))
    assert tuple(cells[0]) == tuple(np.floor(a64 / Bm32).astype(int))
    assert tuple(cells[-1]) == tuple(np.floor(b64 / Bm32).astype(int))
    assert len(cells) == 1 + np.abs(cells[-1] - cells[0]).sum()
    assert (np.abs(np.diff(cells, axis=0)).sum(1) == 1).all()          # 6-connected
    lo = np.minimum(cells.min(0), np.floor(np.minimum(a64, b64) / Bm32)) - 1
    span = int(max(cells.max(0) - lo + 2))
    walk = {tuple(c) for c in cells}
    rngs = [np.arange(lo[k], lo[k] + max(span, 6)) for k in range(3)]
    X, Y, Z = np.meshgrid(*rngs, indexing="ij")
    B = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)

    def met(delta):
        bl, bh = B * Bm32 - delta, (B + 1) * Bm32 + delta
        d = b64 - a64
        with np.errstate(divide="ignore", invalid="ignore"):
            t1, t2 = (bl - a64) / d, (bh - a64) / d
        inside = (a64 >= bl) & (a64 <= bh)
        tlo = np.where(d == 0, np.where(inside, -np.inf, np.inf), np.minimum(t1, t2))
        thi = np.where(d == 0, np.where(inside, np.inf, -np.inf), np.maximum(t1, t2))
        return {tuple(x) for x in B[np.maximum(tlo.max(1), 0) <= np.minimum(thi.min(1), 1)]}

    assert met(-1e-5) <= walk <= met(1e-5)


# ------------------------------------------------------------------------------------ Eq. 1 sequences

def _plane_frames(depths, seed=7):
    rng = np.random.default_rng(seed)
    pose = _pose(_rand_rot(rng), rng.uniform(-1, 1, size=3))
    K = len(depths)
    D = np.stack([np.full((HH, WW), d, np.float32) for d in depths])
    return D, np.repeat(pose[None], K, 0)


def test_idempotent_repeated_frame():
    """integrating the same depth map twice leaves f unchanged and doubles w."""
    D1, P1 = _plane_frames([5.0])
    D2, P2 = _plane_frames([5.0, 5.0])
    x1, fr1, f1, W1 = oracle.fuse(D1, INTR, P1, 0.1, 1.0, 100.0, 1e30)
    x2, fr2, f2, W2 = oracle.fuse(D2, INTR, P2, 0.1, 1.0, 100.0, 1e30)
    assert np.array_equal(x1, x2)
    assert np.array_equal(f1, f2)          # (u + 1·u)/2 = u exactly
    assert np.array_equal(W2, 2 * W1)


def test_weight_cap():
    D, P = _plane_frames([5.0, 5.0, 5.0])
    _, _, f, W = oracle.fuse(D, INTR, P, 0.1, 1.0, 100.0, 2.0)
    D1, P1 = _plane_frames([5.0])
    _, _, f1, W1 = oracle.fuse(D1, INTR, P1, 0.1, 1.0, 100.0, 1e30)
    assert W.max() == 2.0 and np.array_equal(W > 0, W1 > 0)
    assert np.abs(f - f1).max() <= 2e-7


def test_running_average_closed_form():
    """Eq. 1 unrolled: f = mean of the clamped u_SDF/μ over the frames that updated the voxel."""
    depths = [4.8, 5.1, 5.3, 4.9]
    D, P = _plane_frames(depths)
    mu = 1.0
    xyz, first, f, W = oracle.fuse(D, INTR, P, 0.1, mu, 100.0, 1e30)
    zc, ix, iy = _voxel_geometry(xyz, P[0], 0.1)
    ok = (first[:, None] == 0) & _clear_of_pixel_edges(ix, iy) & (W > 0)
    for d in depths:
        ok &= np.abs(zc - (d + mu)) > 1e-4
    terms = np.stack([np.where(zc <= d + mu, np.clip((d - zc) / mu, -1, 1), np.nan) for d in depths])
    cnt = np.isfinite(terms).sum(0)
    mean = np.nansum(terms, 0) / np.maximum(cnt, 1)
    assert np.array_equal(W[ok], cnt[ok].astype(np.float32))
    assert np.abs(f[ok] - mean[ok]).max() <= 2e-5      # z_c carries fp32 rounding of |p| ~ 5 m
    assert ok.sum() > 1000


def test_sequential_allocate_then_update():
    """Reading F-8: a block allocated by frame 1 receives no update from frame 0, although frame 0 would
    have updated its voxels (they lie in front of frame 0's surface, u_SDF > 0)."""
    D, P = _plane_frames([8.0, 3.0])
    mu = 1.0
    xyz, first, f, W = oracle.fuse(D, INTR, P, 0.1, mu, 100.0, 1e30)
    assert set(np.unique(first)) == {0, 1}
    zc, ix, iy = _voxel_geometry(xyz, P[0], 0.1)
    late = (first[:, None] == 1) & (W > 0) & _clear_of_pixel_edges(ix, iy)
    assert late.sum() > 500
    assert (W[late] == 1.0).all()
    assert np.abs(f[late] - np.clip((3.0 - zc[late]) / mu, -1, 1)).max() <= 2e-5
    # frame 0's band (z_c in [7, 9]) lies more than μ behind frame 1's surface: frame 1 leaves it alone
    early = (first[:, None] == 0) & (W > 0) & _clear_of_pixel_edges(ix, iy) & (np.abs(zc - 9.0) > 1e-4)
    assert early.sum() > 500 and (W[early] == 1.0).all()
    assert np.abs(f[early] - np.clip((8.0 - zc[early]) / mu, -1, 1)).max() <= 2e-5


def test_invalid_depths_are_ignored():
    D = np.full((1, HH, WW), np.inf, np.float32)
    D[0, :10] = 0.0
    D[0, 10:20] = np.nan
    D[0, 20:30] = 150.0        # beyond max_range
    D[0, 30:] = -1.0
    _, P = _plane_frames([5.0])
    xyz, _, _, _ = oracle.fuse(D, INTR, P, 0.1, 1.0, 100.0, 1e30)
    assert xyz.shape[0] == 0


# ------------------------------------------------------------------------------------ O2 dense brute force

def _dense_vs_hvg(depth, intr, poses, voxel, mu, max_range, w_max):
    xyz, first, f, W = oracle.fuse(depth, intr, poses, voxel, mu, max_range, w_max)
    keep = first == 0
    assert keep.sum() > 0
    lo = xyz[keep].min(0) * 8
    hi = xyz[keep].max(0) * 8 + 7
    fd, Wd_ = fuse_dense(depth, intr, poses, voxel, mu, max_range, w_max, lo, hi)
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    g = xyz[keep].astype(np.int64)[:, None, :] * 8 + loc[None] - lo
    assert np.array_equal(W[keep], Wd_[g[..., 2], g[..., 1], g[..., 0]])
    assert np.array_equal(f[keep], fd[g[..., 2], g[..., 1], g[..., 0]])
    return xyz, first


def test_dense_equivalence_planes():
    D, P = _plane_frames([4.8, 5.1, 5.3, 4.9], seed=3)
    _dense_vs_hvg(D, INTR, P, 0.1, 1.0, 100.0, 3.0)


def test_dense_equivalence_fusion_tiny():
    from synth.depth import sphere_depth
    ds = sphere_depth(n_cams=4, H=60, Wd=80)
    _dense_vs_hvg(ds.depth.numpy(), ds.intr.numpy(), ds.poses.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)


def test_alloc_and_block_updates_compose_to_fuse():
    from synth.depth import sphere_depth
    ds = sphere_depth()
    args = (ds.depth, ds.intr, ds.poses, ds.voxel, ds.mu, ds.max_range)
    xyz, first, f, W = oracle.fuse(*args, ds.w_max)
    xa, fa = oracle.fuse_alloc(*args)
    assert np.array_equal(xyz, xa) and np.array_equal(first, fa)
    sel = np.arange(0, len(xa), 7)
    fs, Ws = oracle.fuse_update_blocks(*args, ds.w_max, xa[sel], fa[sel])
    assert np.array_equal(fs, f[sel]) and np.array_equal(Ws, W[sel])
    # canonical order: sorted by (x, y, z)
    rows = [tuple(r) for r in xyz.tolist()]
    assert rows == sorted(set(rows))
    assert torch.is_tensor(ds.depth)


def test_incremental_equals_batch():
    """Reading F-11: fusing frames 0..K−1 at once equals fusing 0..k−1 and then continuing with k..K−1 from
    the resulting blocks, bit for bit (each voxel's Eq. 1 recurrence only sees its own (f, w))."""
    from synth.depth import sphere_depth
    ds = sphere_depth()
    D, I, P = ds.depth.numpy(), ds.intr.numpy(), ds.poses.numpy()
    prm = (ds.voxel, ds.mu, ds.max_range, ds.w_max)
    xa, fa, f_all, W_all = oracle.fuse(D, I, P, *prm)
    for k in (1, 3, 7):
        x1, _, f1, W1 = oracle.fuse(D[:k], I, P[:k], *prm)
        x2, fr2, f2, W2 = oracle.fuse_incremental((x1, f1, W1), D[k:], I, P[k:], *prm)
        assert np.array_equal(x2, xa)
        assert np.array_equal(f2, f_all) and np.array_equal(W2, W_all)
        # blocks from the first call carry −1, the others their frame shifted by k
        old = {tuple(r) for r in x1}
        is_old = np.array([tuple(r) in old for r in x2])
        assert (fr2[is_old] == -1).all() and np.array_equal(fr2[~is_old] + k, fa[~is_old])
    with pytest.raises(ValueError):
        oracle.fuse_incremental((np.concatenate([x1, x1[:1]]), np.concatenate([f1, f1[:1]]),
                                 np.concatenate([W1, W1[:1]])), D, I, P, *prm)


def test_dense_f64_closed_form_fronto_parallel_plane():
    """Pin of the float64 dense fusion (the independent-precision reference of the GPU fusion test): a plane
    at depth d seen by an identity-pose camera gives, at every voxel centre in view with z − d <= mu,
    f = clamp((d − z)/mu, −1, 1) after one frame and the running mean of those values after several."""
    voxel, mu = 0.1, 0.3
    intr = np.array([60.0, 60.0, 31.5, 23.5], np.float32)
    pose = _pose(np.eye(3), [0.0, 0.0, 0.0])
    depths = [2.0, 2.2, 1.9]
    D = np.stack([np.full((48, 64), d, np.float32) for d in depths])
    lo, hi = np.array([-3, -3, 10]), np.array([3, 3, 30])
    f, W = fuse_dense(D, intr, np.repeat(pose[None], 3, 0), voxel, mu, 100.0, 1e30, lo, hi, precision="f64")
    z = (np.arange(lo[2], hi[2] + 1) + 0.5) * np.float64(np.float32(voxel))
    d64 = np.array(depths, np.float32).astype(np.float64)[:, None]   # the depth maps hold fp32 numbers
    s = np.clip((d64 - z[None]) / np.float64(np.float32(mu)), -1, 1)
    upd = (d64 - z[None]) >= -np.float64(np.float32(mu))
    # centre column (x = y = 0 voxel: centre (0.05, 0.05) projects inside the image)
    fz, wz = f[:, 3, 3], W[:, 3, 3]
    exp_w = upd.sum(0)
    exp_f = np.where(exp_w > 0, (s * upd).sum(0) / np.maximum(exp_w, 1), 0.0)
    assert np.array_equal(wz, exp_w.astype(np.float64))
    assert np.abs(fz - exp_f).max() <= 1e-12


def test_dense_f64_agrees_with_f32_on_random_poses():
    """The two precisions of the dense fusion agree to 1e-4 on all but 1e-4 of the voxels (random poses,
    noisy depth): a dropped term or wrong sign in either fails."""
    rng = np.random.default_rng(4)
    P = np.stack([_pose(_rand_rot(rng), rng.uniform(-1, 1, size=3)) for _ in range(3)])
    D = np.stack([np.full((HH, WW), d, np.float32) for d in (4.8, 5.1, 5.3)])
    D = D + rng.uniform(-0.3, 0.3, D.shape).astype(np.float32)
    xyz, first, f, W = oracle.fuse(D, INTR, P, 0.1, 1.0, 100.0, 3.0)
    keep = first == 0
    lo, hi = xyz[keep].min(0) * 8, xyz[keep].max(0) * 8 + 7
    a = fuse_dense(D, INTR, P, 0.1, 1.0, 100.0, 3.0, lo, hi)
    b = fuse_dense(D, INTR, P, 0.1, 1.0, 100.0, 3.0, lo, hi, precision="f64")
    ok = (a[1] == b[1]) & (np.abs(a[0] - b[0]) <= 1e-4)
    assert (b[1] > 0).sum() > 10000
    assert (~ok).mean() <= 1e-4
