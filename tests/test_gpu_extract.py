"""GPU parity of the isosurface extraction (vol_extract) against the
extraction oracle (oracle/extract_oracle.c).  The triangle count is an integer result and the vertex
arithmetic is the same written fp32 order on both sides, so the triangle soups are compared bit for bit,
in the specified order (caller block, cell, tetrahedron, triangle)."""
import numpy as np
import pytest
import torch

import oracle
from synth import dense_box, tiny

pytestmark = pytest.mark.gpu

V = 0.1


@pytest.fixture(scope="module")
def Vol():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_03734_b200 import Volume
    return Volume


def _same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    bad = int((a.view(np.uint32) != b.view(np.uint32)).sum())
    assert bad == 0, f"{bad} vertex coordinates differ"


def _sphere(blocks=3, r_vox=10.5, c_vox=12.3):
    s = dense_box(blocks, blocks, blocks)
    c = s.coords.numpy()
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    P = (c[:, None, :].astype(np.float64) * 8 + loc[None] + 0.5) * V
    u = (np.linalg.norm(P - c_vox * V, axis=-1) - r_vox * V).astype(np.float32)
    return c, u


def test_sphere_field_f_bit_exact(Vol):
    c, u = _sphere()
    W = np.ones_like(u)
    vol = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
    T = vol.extract(V, field="f").cpu().numpy()
    _same(T, oracle.extract(c, u, W, V))
    # permuted caller order: same triangles, block-permuted order as specified
    perm = np.random.default_rng(1).permutation(c.shape[0])
    vol2 = Vol(torch.from_numpy(c[perm]).cuda(), torch.from_numpy(u[perm]).cuda(), torch.from_numpy(W).cuda())
    _same(vol2.extract(V, field="f").cpu().numpy(), oracle.extract(c[perm], u[perm], W, V))


def test_omega_wmin_and_missing_blocks(Vol):
    c, u = _sphere()
    i = np.arange(512)
    gx = c[:, None, 0] * 8 + (i % 8)[None]
    gy = c[:, None, 1] * 8 + ((i // 8) % 8)[None]
    W = np.where(gx < 12, 0.0, np.where(gy < 14, 1.0, 3.0)).astype(np.float32)
    keep = np.ones(c.shape[0], bool)
    keep[[0, 5, 13]] = False
    c2, u2, W2 = c[keep], u[keep], W[keep]
    vol = Vol(torch.from_numpy(c2).cuda(), torch.from_numpy(u2).cuda(), torch.from_numpy(W2).cuda())
    for w_min in (0.0, 2.0):
        _same(vol.extract(V, w_min=w_min, field="f").cpu().numpy(), oracle.extract(c2, u2, W2, V, w_min=w_min))


def test_regularised_tiny_bit_exact(Vol, tiny_scene):
    s = tiny_scene
    vol = Vol(s.coords.cuda(), s.f.cuda(), s.W.cuda())
    vol.regularise_scene(s, iters=60)
    T = vol.extract(s.meta["voxel"]).cpu().numpy()
    u32, _, _ = oracle.regularise_scene(s, precision="f32", iters=60)
    assert np.array_equal(vol.u().cpu().numpy(), u32)
    To = oracle.extract(s.coords, u32, s.W, s.meta["voxel"])
    assert To.shape[0] > 1000
    _same(T, To)
    # raw f gives a different (noisier) surface; both through the same API
    Tf = vol.extract(s.meta["voxel"], field="f").cpu().numpy()
    _same(Tf, oracle.extract(s.coords, s.f, s.W, s.meta["voxel"]))


def test_host_output_and_errors(Vol):
    import ctypes
    from paper_1604_03734_b200 import _native as N
    c, u = _sphere(blocks=2, r_vox=5.2, c_vox=8.1)
    W = np.ones_like(u)
    vol = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
    L = N.lib()
    n = ctypes.c_int64()
    N.check(L.vol_extract(vol._h, 1, V, 0.0, None, 0, ctypes.byref(n)))
    host = np.zeros((n.value, 3, 3), np.float32)
    m = ctypes.c_int64()
    N.check(L.vol_extract(vol._h, 1, V, 0.0, host.ctypes.data, n.value, ctypes.byref(m)))
    _same(host, oracle.extract(c, u, W, V))
    assert L.vol_extract(vol._h, 1, V, 0.0, host.ctypes.data, n.value - 1, ctypes.byref(m)) == N.VOL_ENOMEM
    _same(vol.extract(V, field="u").cpu().numpy(), host)          # u = f (warm state) before regularising
    assert L.vol_extract(vol._h, 2, V, 0.0, None, 0, ctypes.byref(m)) == N.VOL_EINVAL
    assert L.vol_extract(vol._h, 1, -1.0, 0.0, None, 0, ctypes.byref(m)) == N.VOL_EINVAL
    empty = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.zeros_like(torch.from_numpy(W)).cuda()
                + torch.from_numpy((np.arange(c.shape[0] * 512) % 7 == 0).reshape(-1, 512).astype(np.float32)).cuda())
    assert empty.extract(V, field="f").shape[0] == 0


def test_pipeline_fuse_regularise_extract(Vol):
    """depth maps → vol_fuse → vol_regularise → vol_extract against the oracle chain, bit for bit."""
    from paper_1604_03734_b200 import fuse
    from synth.depth import sphere_depth
    ds = sphere_depth()
    xyz, first, f, W = fuse(ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy(), ds.voxel, ds.mu, ds.max_range, ds.w_max)
    vol = Vol(xyz, f, W)
    tau = float(np.float32(1 / 12 ** 0.5))
    vol.regularise(1.0, 0.0, tau, tau, 40)
    T = vol.extract(ds.voxel).cpu().numpy()
    xo, _, fo, Wo = oracle.fuse(ds.depth, ds.intr, ds.poses, ds.voxel, ds.mu, ds.max_range, ds.w_max)
    u32, _, _ = oracle.regularise(xo, fo, Wo, 1.0, 0.0, tau, tau, 40, precision="f32")
    To = oracle.extract(xo, u32, Wo, ds.voxel)
    assert To.shape[0] > 100
    _same(T, To)


def test_street_full_size_f(Vol):
    """street (configs[1], 24.6 M voxels): extraction of the fused f, bit-exact against the oracle."""
    from synth import street
    s = street(device="cuda", chunk_blocks=4096)
    vol = Vol(s.coords, s.f, s.W)
    T = vol.extract(s.meta["voxel"], field="f").cpu().numpy()
    To = oracle.extract(s.coords.cpu().numpy(), s.f.cpu().numpy(), s.W.cpu().numpy(), s.meta["voxel"])
    assert To.shape[0] > 1_000_000
    _same(T, To)


def test_degenerate_and_tiny_t_bit_exact(Vol):
    """Exact zeros at corners (X-6 drops) and values that make t round to 0 or 1: GPU == oracle."""
    s = dense_box(2, 2, 2)
    c = s.coords.numpy()
    i = np.arange(512)
    loc = np.stack([i % 8, (i // 8) % 8, i // 64], 1)
    g = c[:, None, :].astype(np.int64) * 8 + loc[None]
    u = (g[..., 0] + g[..., 1] - g[..., 2] - 3).astype(np.float32)
    u[(g[..., 0] % 3) == 0] *= np.float32(1e-30)                 # tiny values next to O(1) ones
    W = np.ones_like(u)
    vol = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
    T = vol.extract(V, field="f").cpu().numpy()
    To = oracle.extract(c, u, W, V)
    assert To.shape[0] > 0
    _same(T, To)


def test_device_output_offsets_and_overflow(Vol):
    """The ordered single pass into a device buffer: every 4-byte offset of the output pointer (the copy-out
    stages whole float4s at the buffer's alignment), and a buffer that is too small: VOL_ENOMEM with the
    exact count, the first max_tris triangles written in order and nothing past the buffer."""
    import ctypes
    from paper_1604_03734_b200 import _native as N
    c, u = _sphere(blocks=3, r_vox=10.5, c_vox=12.3)
    W = np.ones_like(u)
    rng = np.random.default_rng(5)
    perm = rng.permutation(c.shape[0])
    c, u = c[perm], u[perm]
    vol = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
    ref = oracle.extract(c, u, W, V)
    n = ref.shape[0]
    assert n > 1000
    L = N.lib()
    m = ctypes.c_int64()
    for off in range(4):
        buf = torch.full((n * 9 + 64,), 7.0, device="cuda")
        st = L.vol_extract(vol._h, 1, V, 0.0, ctypes.c_void_p(buf.data_ptr() + 4 * off), n, ctypes.byref(m))
        assert st == N.VOL_OK and m.value == n
        h = buf.cpu().numpy()
        _same(h[off:off + 9 * n].reshape(n, 3, 3), ref)
        assert (h[:off] == 7.0).all() and (h[off + 9 * n:] == 7.0).all()
    for cap in (0, 1, 333, n - 1):
        buf = torch.full((n * 9 + 64,), 7.0, device="cuda")
        st = L.vol_extract(vol._h, 1, V, 0.0, ctypes.c_void_p(buf.data_ptr() + 4), cap, ctypes.byref(m))
        assert st == N.VOL_ENOMEM and m.value == n
        h = buf.cpu().numpy()
        _same(h[1:1 + 9 * cap].reshape(cap, 3, 3), ref[:cap])
        assert (h[:1] == 7.0).all() and (h[1 + 9 * cap:] == 7.0).all()


@pytest.mark.parametrize("case", ["sphere", "random"])
def test_within_fp64_extraction(Vol, case):
    """Independent-precision check: the kernel's triangles against the float64 numpy extraction
    (oracle/extract64.py — written separately from the C oracle, orientation by determinant): same
    triangles in the same order (topology is decided on exact signs and zeros), each equal up to a cyclic
    rotation of its vertices (which keeps the orientation), vertices within 1e-6 (fp32 rounding of
    coordinates below 3 m is ~2.4e-7)."""
    from oracle.extract64 import extract_f64, match_up_to_rotation
    if case == "sphere":
        c, u = _sphere()
        W = np.ones_like(u)
    else:
        rng = np.random.default_rng(9)
        c = dense_box(2, 2, 2).coords.numpy()
        u = rng.normal(size=(c.shape[0], 512)).astype(np.float32)
        u[rng.random(u.shape) < 0.05] = 0.0
        W = (rng.random(u.shape) < 0.97).astype(np.float32)
        perm = rng.permutation(c.shape[0])
        c, u, W = c[perm], u[perm], W[perm]
    vol = Vol(torch.from_numpy(c).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
    T = vol.extract(V, field="f").cpu().numpy()
    R = extract_f64(c, u, W, V)
    assert T.shape == R.shape and T.shape[0] > 1000
    assert match_up_to_rotation(T, R) <= 1e-6


def test_single_block_and_single_cell_row(Vol):
    """The ordered single pass at its smallest: one block (one CTA, no predecessor in the look-back), and two
    blocks far apart (no cell spans both), into a device buffer and through the count-only call."""
    import ctypes
    from paper_1604_03734_b200 import _native as N
    rng = np.random.default_rng(3)
    for coords in (np.array([[2, -1, 5]], np.int32), np.array([[0, 0, 0], [9, 9, 9]], np.int32)):
        u = rng.normal(size=(coords.shape[0], 512)).astype(np.float32)
        W = np.ones_like(u)
        vol = Vol(torch.from_numpy(coords).cuda(), torch.from_numpy(u).cuda(), torch.from_numpy(W).cuda())
        ref = oracle.extract(coords, u, W, V)
        assert ref.shape[0] > 0
        _same(vol.extract(V, field="f").cpu().numpy(), ref)
        out = torch.empty(ref.shape[0] + 3, 3, 3, device="cuda")
        _same(vol.extract(V, field="f", out=out).cpu().numpy(), ref)
        n = ctypes.c_int64()
        N.check(N.lib().vol_extract(vol._h, 1, V, 0.0, None, 0, ctypes.byref(n)))
        assert n.value == ref.shape[0]
