"""GPU parity of the TSDF fusion (vol_fuse, paper §III-A Eq. 1) against the
fusion oracle (oracle/fusion_oracle.c).

Bar: the allocated block set, its (x, y, z) order and the allocating frame are integer results —
bit-exact; f and W are evaluated by both sides in the same written fp32 order (reading F-10, the
pixel choice and the block walk are floating-point decisions taken in the kernel's precision), so
they are compared bit for bit as well.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from synth.depth import sphere_depth, street_depth

pytestmark = pytest.mark.gpu

INTR = np.array([60.0, 60.0, 31.5, 23.5], np.float32)
HH, WW = 48, 64


@pytest.fixture(scope="module")
def fuse():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_03734_b200 import fuse as F
    return F


def _gpu(fuse, depth, intr, poses, voxel, mu, max_range, w_max, **kw):
    xyz, first, f, W = fuse(torch.as_tensor(np.asarray(depth, np.float32)).cuda(),
                            torch.as_tensor(np.asarray(poses, np.float32)).cuda(), intr, voxel, mu, max_range, w_max,
                            **kw)
    return xyz.cpu().numpy(), first.cpu().numpy(), f.cpu().numpy(), W.cpu().numpy()


def _same(a, b):
    xa, fa, f1, W1 = a
    xb, fb, f2, W2 = b
    assert xa.shape == xb.shape, (xa.shape, xb.shape)
    assert np.array_equal(xa, xb)
    assert np.array_equal(fa, fb)
    assert np.array_equal(W1, W2), f"{int((W1 != W2).sum())} weights differ"
    bad = int((f1 != f2).sum())
    assert bad == 0, f"{bad} f values differ (max {np.abs(f1 - f2).max()})"


def _rand_pose(seed, scale=3.0):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    R = np.array([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                  [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                  [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]])
    t = rng.uniform(-scale, scale, size=3)
    return np.concatenate([R, t[:, None]], 1).reshape(12).astype(np.float32)


def test_fusion_tiny_bit_exact(fuse):
    ds = sphere_depth()
    args = (ds.depth.numpy(), ds.intr.numpy(), ds.poses.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    _same(_gpu(fuse, *args), oracle.fuse(*args))


@pytest.mark.parametrize("seed", range(4))
def test_plane_random_pose_bit_exact(fuse, seed):
    depth = np.full((1, HH, WW), 5.0, np.float32)
    args = (depth, INTR, _rand_pose(seed)[None], 0.1, 1.0, 100.0, 1e30)
    _same(_gpu(fuse, *args), oracle.fuse(*args))


@pytest.mark.parametrize("depths,w_max", [([4.8, 5.1, 5.3, 4.9], 1e30), ([8.0, 3.0], 1e30), ([5.0] * 3, 2.0)])
def test_plane_sequences_bit_exact(fuse, depths, w_max):
    P = np.repeat(_rand_pose(7, 1.0)[None], len(depths), 0)
    D = np.stack([np.full((HH, WW), d, np.float32) for d in depths])
    args = (D, INTR, P, 0.1, 1.0, 100.0, w_max)
    _same(_gpu(fuse, *args), oracle.fuse(*args))


def test_noisy_frames_many_poses_bit_exact(fuse):
    """Random poses and noisy, partly invalid depth maps (every branch of steps 1-4 and of the walk)."""
    g = np.random.default_rng(5)
    K = 6
    P = np.stack([_rand_pose(50 + k, 0.5) for k in range(K)])
    D = g.uniform(1.0, 9.0, size=(K, HH, WW)).astype(np.float32)
    D[g.uniform(size=D.shape) < 0.05] = np.inf
    D[g.uniform(size=D.shape) < 0.05] = 0.0
    D[g.uniform(size=D.shape) < 0.02] = np.nan
    D[g.uniform(size=D.shape) < 0.05] = 20.0        # > max_range
    args = (D, INTR, P, 0.05, 0.3, 12.0, 20.0)
    _same(_gpu(fuse, *args), oracle.fuse(*args))


def test_cull_never_changes_results(fuse):
    ds = sphere_depth(n_cams=8)
    args = (ds.depth.numpy(), ds.intr.numpy(), ds.poses.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    a = _gpu(fuse, *args)
    os.environ["HVG_FUSE_NOCULL"] = "1"
    try:
        b = _gpu(fuse, *args)
    finally:
        del os.environ["HVG_FUSE_NOCULL"]
    _same(a, b)


def test_host_outputs_equal_device_outputs(fuse):
    from paper_1604_03734_b200 import _native as N
    import ctypes
    ds = sphere_depth(n_cams=3)
    dev = _gpu(fuse, ds.depth.numpy(), ds.intr.numpy(), ds.poses.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    n = dev[0].shape[0]
    cap = n + 10
    xyz = np.zeros((cap, 3), np.int32)
    first = np.zeros(cap, np.int32)
    f = np.zeros((cap, 512), np.float32)
    W = np.zeros((cap, 512), np.float32)
    D = np.ascontiguousarray(ds.depth.numpy())
    P = np.ascontiguousarray(ds.poses.numpy())
    it = ds.intr.numpy()
    cam = N.vol_camera(*(float(v) for v in it), ds.Wd, ds.H)
    prm = N.vol_fusion_params(ds.voxel, ds.mu, ds.max_range, ds.w_max)
    nb = ctypes.c_int64()
    N.check(N.lib().vol_fuse(D.ctypes.data, ds.K, ctypes.byref(cam), P.ctypes.data, ctypes.byref(prm), cap, None, 0,
                             None, xyz.ctypes.data, first.ctypes.data, f.ctypes.data, W.ctypes.data,
                             ctypes.byref(nb), None))
    assert nb.value == n
    _same(dev, (xyz[:n], first[:n], f[:n], W[:n]))


def test_stats_counters(fuse):
    """pixels_valid, blocks and voxel_updates are exact counts (the latter = number of Eq. 1 updates,
    i.e. the sum of W for an uncapped fusion); block_frames lies between the frames that update some
    voxel of a block and all frames since its allocation."""
    ds = sphere_depth()
    st = {}
    xyz, first, f, W = fuse(ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy(), ds.voxel, ds.mu, ds.max_range, 1e30,
                            stats=st)
    D = ds.depth.numpy()
    assert st["pixels_valid"] == int((np.isfinite(D) & (D > 0) & (D <= ds.max_range)).sum())
    assert st["blocks"] == xyz.shape[0]
    assert st["voxel_updates"] == int(W.sum().item())
    fr = first.cpu().numpy()
    assert st["block_frames"] <= int((ds.K - fr).sum())
    assert st["block_frames"] >= int(W.cpu().numpy().max(1).sum())


def test_capacity_errors_and_retry(fuse):
    from paper_1604_03734_b200._native import VolError, VOL_ENOMEM
    ds = sphere_depth(n_cams=2)
    args = (ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    with pytest.raises(VolError) as e:
        fuse(*args, max_blocks=5)
    assert e.value.status == VOL_ENOMEM
    xyz, first, f, W = fuse(*args)            # default: grows the capacity and retries
    xo, fo, _, _ = oracle.fuse(ds.depth, ds.intr, ds.poses, ds.voxel, ds.mu, ds.max_range, ds.w_max)
    assert np.array_equal(xyz.cpu().numpy(), xo)


def test_out_of_range_and_invalid(fuse):
    from paper_1604_03734_b200._native import VolError, VOL_EDATA, VOL_EINVAL
    P = _rand_pose(1)
    P[3] = 1.0e6                              # 1000 km away: block coordinates beyond 2^20
    D = np.full((1, HH, WW), 5.0, np.float32)
    with pytest.raises(ValueError):
        oracle.fuse(D, INTR, P[None], 0.05, 0.3, 100.0, 30.0)
    with pytest.raises(VolError) as e:
        _gpu(fuse, D, INTR, P[None], 0.05, 0.3, 100.0, 30.0)
    assert e.value.status == VOL_EDATA
    with pytest.raises(VolError) as e:
        _gpu(fuse, D, INTR, P[None], 0.05, -0.3, 100.0, 30.0)
    assert e.value.status == VOL_EINVAL
    empty = _gpu(fuse, np.full((1, HH, WW), np.inf, np.float32), INTR, P[None] * 0 + _rand_pose(2)[None], 0.05, 0.3,
                 100.0, 30.0)
    assert empty[0].shape[0] == 0


def test_fused_volume_regularises_like_oracle(fuse):
    """Pipeline: depth maps → vol_fuse → Volume → vol_regularise, against oracle.fuse → oracle.regularise."""
    from paper_1604_03734_b200 import Volume
    ds = sphere_depth()
    xyz, first, f, W = fuse(ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    vol = Volume(xyz, f, W)
    vol.regularise(1.0, 0.0, float(np.float32(1 / 12 ** 0.5)), float(np.float32(1 / 12 ** 0.5)), 30)
    u = vol.u().cpu().numpy()
    xo, _, fo, Wo = oracle.fuse(ds.depth, ds.intr, ds.poses, ds.voxel, ds.mu, ds.max_range, ds.w_max)
    u32, _, _ = oracle.regularise(xo, fo, Wo, 1.0, 0.0, float(np.float32(1 / 12 ** 0.5)),
                                  float(np.float32(1 / 12 ** 0.5)), 30, precision="f32")
    assert np.array_equal(u, u32)


def test_street_fusion_full_size(fuse):
    """fusion-street at full size (61 frames of 1240×376): block set and allocating frames bit-exact
    against the oracle's sequential allocation; f, W bit-exact on a 1-in-50 sample of the blocks."""
    ds = street_depth(device="cuda")
    xyz, first, f, W = fuse(ds.depth, ds.poses, ds.intr.cpu().numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    D, P, I = ds.depth.cpu().numpy(), ds.poses.cpu().numpy(), ds.intr.cpu().numpy()
    xo, fo = oracle.fuse_alloc(D, I, P, ds.voxel, ds.mu, ds.max_range)
    assert np.array_equal(xyz.cpu().numpy(), xo)
    assert np.array_equal(first.cpu().numpy(), fo)
    sel = np.arange(0, xo.shape[0], 50)
    fs, Ws = oracle.fuse_update_blocks(D, I, P, ds.voxel, ds.mu, ds.max_range, ds.w_max, xo[sel], fo[sel])
    assert np.array_equal(W.cpu().numpy()[sel], Ws)
    assert np.array_equal(f.cpu().numpy()[sel], fs)
    assert xo.shape[0] > 20000


def test_edge_cases_bit_exact(fuse):
    """Weight cap 1, an all-invalid frame inside the sequence, depths below μ (band clamped at the camera,
    z_c → 0), negative coordinates and a camera looking back along −z: GPU == oracle bit for bit."""
    g = np.random.default_rng(11)
    K = 5
    P = np.stack([_rand_pose(200 + k, 0.3) for k in range(K)])
    P[:, 3] -= 7.0                                   # negative x everywhere
    P[2, :3] = -P[2, :3]                             # an improper (reflected) rotation: still just numbers
    D = g.uniform(0.05, 4.0, size=(K, HH, WW)).astype(np.float32)
    D[1] = np.nan                                    # whole frame invalid
    D[3, :, :10] = 0.1                               # < μ: band starts at the camera
    args = (D, INTR, P, 0.05, 0.3, 6.0, 1.0)
    _same(_gpu(fuse, *args), oracle.fuse(*args))


@pytest.mark.parametrize("k", [1, 4])
def test_incremental_equals_batch_bit_exact(fuse, k):
    """vol_fuse_incremental (reading F-11): frames 0..k−1, then k..K−1 continued from those blocks, equals
    the one-call fusion of all frames and the oracle's incremental fusion, bit for bit."""
    ds = sphere_depth()
    D, P, I = ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy()
    prm = (ds.voxel, ds.mu, ds.max_range, ds.w_max)
    xa, fa, f_all, W_all = fuse(D, P, I, *prm)
    x1, _, f1, W1 = fuse(D[:k], P[:k], I, *prm)
    x2, fr2, f2, W2 = fuse(D[k:], P[k:], I, *prm, prev=(x1, f1, W1))
    assert torch.equal(x2, xa) and torch.equal(f2, f_all) and torch.equal(W2, W_all)
    xo, fro, fo, Wo = oracle.fuse_incremental((x1.cpu().numpy(), f1.cpu().numpy(), W1.cpu().numpy()),
                                              ds.depth[k:], I, ds.poses[k:], *prm)
    _same((x2.cpu().numpy(), fr2.cpu().numpy(), f2.cpu().numpy(), W2.cpu().numpy()), (xo, fro, fo, Wo))
    # host-resident previous blocks take the staging path
    x3, fr3, f3, W3 = fuse(D[k:], P[k:], I, *prm, prev=(x1.cpu(), f1.cpu(), W1.cpu()))
    assert torch.equal(f3, f2) and torch.equal(fr3, fr2)
    from paper_1604_03734_b200._native import VolError, VOL_EDATA
    with pytest.raises(VolError) as e:
        fuse(D[k:], P[k:], I, *prm, prev=(torch.cat([x1, x1[:1]]), torch.cat([f1, f1[:1]]), torch.cat([W1, W1[:1]])))
    assert e.value.status == VOL_EDATA


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_fusion_within_fp64_dense(fuse, seed):
    """Independent-precision check (the bit-exact tests above compare with an fp32 oracle whose rounding
    order follows reading F-12): the kernel's f and W against a float64 dense fusion with the paper's plain
    x/z projection (oracle/dense_fusion.py, precision "f64"), on the blocks allocated by the first frame,
    for 4 noisy depth maps from random poses.  Bar: W equal and |f − f64| <= 1e-4 on all but 1e-4 of the
    voxels (a voxel projecting within fp32 rounding of a pixel boundary may pick the neighbouring pixel in
    one precision; the axis-aligned sphere cameras put voxel centres exactly on pixel boundaries, so they
    are not used here)."""
    from oracle.dense_fusion import fuse_dense
    P = np.stack([_rand_pose(seed + 100 * k, 1.0) for k in range(4)])
    D = np.stack([np.full((HH, WW), d, np.float32) for d in (4.8, 5.1, 5.3, 4.9)])
    D = D + np.random.default_rng(seed).uniform(-0.3, 0.3, D.shape).astype(np.float32)
    args = (D, INTR, P, 0.1, 1.0, 100.0, 3.0)
    xyz, first, f, W = _gpu(fuse, *args)
    keep = first == 0
    assert keep.sum() > 0
    lo = xyz[keep].min(0) * 8
    hi = xyz[keep].max(0) * 8 + 7
    fd, Wd_ = fuse_dense(*args, lo, hi, precision="f64")
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    g = xyz[keep].astype(np.int64)[:, None, :] * 8 + loc[None] - lo
    f64 = fd[g[..., 2], g[..., 1], g[..., 0]]
    W64 = Wd_[g[..., 2], g[..., 1], g[..., 0]]
    ok = (W[keep] == W64) & (np.abs(f[keep].astype(np.float64) - f64) <= 1e-4)
    assert (W64 > 0).sum() > 10000
    assert (~ok).mean() <= 1e-4, f"{int((~ok).sum())} of {ok.size} voxels off the fp64 fusion"
