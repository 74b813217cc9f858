"""The whole device pipeline of the paper (Fig. 2): stereo pairs → depth maps (§IV) → TSDF fusion
(§III-A) → primal-dual regularisation (§III-C) → surface extraction, each stage through its C-ABI entry
point, against the chain of oracles stage by stage, bit for bit (every stage's arithmetic is the same
written fp32 order on both sides)."""
import numpy as np
import pytest
import torch

import oracle
from synth.stereo import street_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1604_03734_b200 as P
    return P


def _bits(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert int((a.view(np.uint32) != b.view(np.uint32)).sum()) == 0


def test_stereo_to_surface_bit_exact(lib):
    # quarter-resolution rig (310×94, fx = 180), 3 frames 1 m apart
    H, W, f = 94, 310, 180.0
    IL, IR, dt, poses, intr, B = street_pair(frames=(20, 21, 22), H=H, Wd=W, fpx=f, device="cuda", return_rig=True)
    kw = dict(n_disp=32, outer=4, inner=10)
    d = lib.stereo.stereo(IL, IR, **kw)
    z = lib.stereo.disparity_to_depth(d, f * B, d_min=0.5)
    voxel, mu, rmax, wmax = 0.1, 0.5, 25.0, 30.0
    xyz, first, fu, Wt = lib.fuse(z, poses, intr, voxel, mu, rmax, wmax)
    vol = lib.Volume(xyz, fu, Wt)
    tau = float(np.float32(1 / 12 ** 0.5))
    vol.regularise(0.8, 0.01, tau, tau, 50)
    T = vol.extract(voxel)
    # oracle chain
    zo = []
    for k in range(3):
        do, _, _ = oracle.stereo(IL[k].cpu().numpy(), IR[k].cpu().numpy(), D=32, outer=4, inner=10)
        _bits(d[k].cpu().numpy(), do)
        zk = np.where(do > np.float32(0.5), np.float32(f * B) / do, np.float32(0)).astype(np.float32)
        zo.append(zk)
    zo = np.stack(zo)
    _bits(z.cpu().numpy(), zo)
    xo, fo, ffo, Wo = oracle.fuse(zo, intr, poses.cpu().numpy(), voxel, mu, rmax, wmax)
    assert np.array_equal(xyz.cpu().numpy(), xo) and np.array_equal(first.cpu().numpy(), fo)
    _bits(fu.cpu().numpy(), ffo)
    _bits(Wt.cpu().numpy(), Wo)
    u32, _, _ = oracle.regularise(xo, ffo, Wo, 0.8, 0.01, tau, tau, 50, precision="f32")
    _bits(vol.u().cpu().numpy(), u32)
    To = oracle.extract(xo, u32, Wo, voxel)
    assert To.shape[0] > 1000
    _bits(T.cpu().numpy(), To)
