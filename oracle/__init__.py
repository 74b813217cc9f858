"""CPU oracle of the hashed-voxel-grid primal-dual TV regulariser (arXiv 1604.03734 §III-B/C).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_1604_03734_b200``) never imports it and shares no code with it.

Two independent oracles:
  * O1 — ``hvg_oracle.c`` (plain C, fp64 and fp32 in one written formula order), loaded via ctypes:
    its own hash table, CSR buckets and neighbour table, per-phase loops over every voxel.
  * O2 — ``oracle.dense`` (numpy): dense brute force on the bounding box of the blocks.

Parity status per function:
  hash / tables ......... pinned (hand-evaluated hash values, brute-force neighbour search)
  gradient / divergence . pinned (SPEC worked examples, adjointness, dense O2)
  dual / primal / relax . pinned (worked examples, closed forms of 1-D TV-L1 and ROF steps)
  regularise ............ pinned (closed forms, exact invariants, O1 == O2); general 3-D
                          isotropic TV-L1 at finite iterations has no closed form ("parity unpinned
                          beyond these", SURVEY §8(c) last pin row)
  energy ................ pinned (worked examples, brute force, weak duality)
  fusion (Eq. 1) ........ pinned (SPEC worked examples, fronto-parallel plane closed form under random
                          rigid poses, running-average closed form, block walk vs exact segment-box
                          intersection, dense numpy brute force O2-fusion) — ``fusion_oracle.c``
  stereo (§IV) .......... pinned (census worked example, strict-order invariance, shifted-pair WTA, tensor
                          closed forms and eigen-structure, K/Kᵀ adjointness, dual feasibility,
                          constant and slanted-plane disparities, λ → ∞ gives WTA) — ``stereo_oracle.c``;
                          ``oracle.stereo64``: a float64 numpy solve (textbook division forms), pinned by
                          operator adjointness, tensor closed forms and agreement with the C oracle
  fusion, float64 ....... ``oracle.dense_fusion`` precision "f64" (plain x/z projection), pinned by the
                          fronto-parallel closed form and agreement with the fp32 dense fusion
  extraction ............ pinned (planar fields: vertices on the plane, exact area, orientation; analytic
                          sphere: closed 2-manifold, Euler characteristic 2, area/volume; Ω
                          restriction) — ``extract_oracle.c``; ``oracle.extract64``: a float64 numpy
                          version with geometric (determinant) orientation, pinned to the C oracle and
                          to planar fields (vertices on the plane to 1e-12)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "hvg_oracle.c"), os.path.join(_HERE, "fusion_oracle.c"),
        os.path.join(_HERE, "extract_oracle.c"), os.path.join(_HERE, "stereo_oracle.c"),
        os.path.join(_HERE, "hvg_oracle_real.inc")]


def build(force: bool = False) -> str:
    """Compile the C oracle with -O2 -ffp-contract=off (reading c-18: no FMA contraction)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _SRC[0], _SRC[1], _SRC[2], _SRC[3], "-lm"])
        os.replace(tmp, _SO)
    return _SO


_SO_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build_omp(force: bool = False) -> str:
    """The same sources with -fopenmp (ORC_PAR loops over all host cores): a TIMING build for
    bench.py's cpu_baseline_omp only — identical arithmetic, checked bitwise against build() in
    tests/test_oracle_iteration.py."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO_OMP) or os.path.getmtime(_SO_OMP) < newest:
        tmp = _SO_OMP + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", "-Wall", "-o", tmp, _SRC[0], _SRC[1], _SRC[2], _SRC[3], "-lm"])
        os.replace(tmp, _SO_OMP)
    return _SO_OMP


def _cpu_tag() -> str:
    """A short digest of this host's CPU model and ISA flags (the -march=native build is host-specific)."""
    import hashlib
    info = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith(("model name", "flags")):
                info += line
                if line.startswith("flags"):
                    break
    except OSError:
        pass
    return hashlib.sha1(info.encode()).hexdigest()[:10]


def build_native(omp: bool = False, force: bool = False) -> str:
    """TIMING build for bench.py's CPU baselines ("O1 is built -O3 -march=native
    -ffp-contract=off"): the same sources, -O3 -march=native, optionally -fopenmp.  Built on the host that
    runs it (the file name carries a digest of the CPU model and flags, so a library built for another
    CPU is never loaded).  No contraction and no fast-math, and every loop is over independent voxels,
    so the arithmetic is the plain build's bit for bit (checked in tests/test_oracle_iteration.py)."""
    so = os.path.join(_HERE, f"liboracle_native{'_omp' if omp else ''}_{_cpu_tag()}.so")
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(so) or os.path.getmtime(so) < newest:
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall"] + (["-fopenmp"] if omp else []) +
                              ["-o", tmp, _SRC[0], _SRC[1], _SRC[2], _SRC[3], "-lm"])
        os.replace(tmp, so)
    return so


_lib = None
_lib_omp = None
_lib_native = {}


def lib(omp: bool = False, native: bool = False):
    global _lib, _lib_omp
    if native:
        if omp not in _lib_native:
            _lib_native[omp] = _declare(ctypes.CDLL(build_native(omp)))
        return _lib_native[omp]
    if omp:
        if _lib_omp is None:
            _lib_omp = _declare(ctypes.CDLL(build_omp()))
        return _lib_omp
    if _lib is None:
        _lib = _declare(ctypes.CDLL(build()))
    return _lib


def _declare(L):
    """ctypes signatures of every oracle entry point."""
    P = ctypes.c_void_p
    i64, u32, i32, dbl, flt, cint = ctypes.c_int64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_double, ctypes.c_float, ctypes.c_int
    L.orc_hash.restype = u32
    L.orc_hash.argtypes = [i32, i32, i32, u32]
    L.orc_table_size.restype = u32
    L.orc_table_size.argtypes = [i64]
    L.orc_build_table.restype = i64
    L.orc_build_table.argtypes = [P, i64, u32, P, P, P]
    L.orc_lookup.restype = i64
    L.orc_lookup.argtypes = [P, P, P, u32, i32, i32, i32]
    L.orc_neighbours.restype = None
    L.orc_neighbours.argtypes = [P, i64, u32, P, P, P]
    for sfx, real in (("f64", dbl), ("f32", flt)):
        g = getattr(L, f"orc_gradient_{sfx}")
        g.restype = None
        g.argtypes = [i64, P, P, P, P]
        d = getattr(L, f"orc_divergence_{sfx}")
        d.restype = None
        d.argtypes = [i64, P, P, P, P]
        r = getattr(L, f"orc_regularise_{sfx}")
        r.restype = cint
        r.argtypes = [i64, P, P, P, real, real, real, real, real, cint, cint, i64, P, P, P, cint]
        ph = getattr(L, f"orc_phase_{sfx}")
        ph.restype = cint
        ph.argtypes = [i64, P, P, P, real, real, real, real, real, cint, cint, P, P, P]
    L.orc_energy.restype = None
    L.orc_energy.argtypes = [i64, P, P, P, P, P, dbl, dbl, cint, P, P]
    # fusion (fusion_oracle.c)
    L.orc_tsdf_update.restype = cint
    L.orc_tsdf_update.argtypes = [P, P, flt, flt, flt]
    L.orc_project.restype = cint
    L.orc_project.argtypes = [P, P, i32, i32, flt, flt, flt, P, P, P]
    L.orc_block_walk.restype = i64
    L.orc_block_walk.argtypes = [P, P, flt, P, i64]
    L.orc_fuse.restype = i64
    L.orc_fuse.argtypes = [P, i32, i32, i32, P, P, flt, flt, flt, flt, i64, P, P, P, P]
    L.orc_fuse_incremental.restype = i64
    L.orc_fuse_incremental.argtypes = [P, P, P, i64, P, i32, i32, i32, P, P, flt, flt, flt, flt, i64, P, P, P, P]
    L.orc_fuse_alloc.restype = i64
    L.orc_fuse_alloc.argtypes = [P, i32, i32, i32, P, P, flt, flt, flt, i64, P, P]
    L.orc_extract.restype = i64
    L.orc_extract.argtypes = [P, i64, P, P, flt, flt, P, i64]
    L.orc_census.restype = None
    L.orc_census.argtypes = [P, cint, cint, cint, P]
    L.orc_cost.restype = None
    L.orc_cost.argtypes = [P, P, cint, cint, cint, cint, P]
    L.orc_tensor.restype = None
    L.orc_tensor.argtypes = [P, cint, cint, flt, flt, P]
    L.orc_tgv_K.restype = None
    L.orc_tgv_K.argtypes = [P, P, P, cint, cint, P, P]
    L.orc_tgv_KT.restype = None
    L.orc_tgv_KT.argtypes = [P, P, P, cint, cint, P, P, P]
    L.orc_data_step.restype = flt
    L.orc_data_step.argtypes = [flt, P, cint, flt, flt]
    L.orc_stereo_theta.restype = flt
    L.orc_stereo_theta.argtypes = [P, cint]
    L.orc_stereo.restype = cint
    L.orc_stereo.argtypes = [P, P, cint, cint, P, P, P, P]
    L.orc_fuse_update_blocks.restype = None
    L.orc_fuse_update_blocks.argtypes = [P, i32, i32, i32, P, P, flt, flt, flt, flt, P, P, i64, P, P]
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _np(x, dtype):
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=dtype)


def block_hash(x: int, y: int, z: int, T: int) -> int:
    return int(lib().orc_hash(x, y, z, T))


def table_size(n: int) -> int:
    return int(lib().orc_table_size(n))


def build_table(coords):
    """Returns (T, bucket_start[T+1] uint32, bucket_entry[n] int32, dup) with dup = None or (j, i)."""
    c = _np(coords, np.int32).reshape(-1, 3)
    n = c.shape[0]
    T = table_size(n)
    bs = np.zeros(T + 1, np.uint32)
    be = np.zeros(max(n, 1), np.int32)
    dj = np.zeros(1, np.int64)
    i = lib().orc_build_table(_ptr(c), n, T, _ptr(bs), _ptr(be), _ptr(dj))
    dup = None if i < 0 else (int(dj[0]), int(i))
    return T, bs, be[:n], dup


def lookup(coords, tables, x, y, z) -> int:
    c = _np(coords, np.int32).reshape(-1, 3)
    T, bs, be, _ = tables
    be = np.ascontiguousarray(be) if be.size else np.zeros(1, np.int32)
    return int(lib().orc_lookup(_ptr(c), _ptr(bs), _ptr(be), T, x, y, z))


def neighbours(coords, tables=None) -> np.ndarray:
    """nbr [n, 6] int32 in direction order (−x, +x, −y, +y, −z, +z), −1 = unallocated."""
    c = _np(coords, np.int32).reshape(-1, 3)
    n = c.shape[0]
    if tables is None:
        tables = build_table(c)
    T, bs, be, dup = tables
    if dup is not None:
        raise ValueError(f"duplicate block coordinates at caller indices {dup}")
    be = np.ascontiguousarray(be) if be.size else np.zeros(1, np.int32)
    nbr = np.zeros((n, 6), np.int32)
    lib().orc_neighbours(_ptr(c), n, T, _ptr(bs), _ptr(be), _ptr(nbr))
    return nbr


def _rt(precision):
    return (np.float64, "f64") if precision == "f64" else (np.float32, "f32")


def gradient(nbr, W, u, precision="f64") -> np.ndarray:
    """Eq. 3 masked forward gradient; returns [3, n, 512]."""
    dt, sfx = _rt(precision)
    nbr = _np(nbr, np.int32)
    n = nbr.shape[0]
    Wf = _np(W, np.float32)
    uu = _np(u, dt)
    g = np.zeros((3, n, 512), dt)
    getattr(lib(), f"orc_gradient_{sfx}")(n, _ptr(nbr), _ptr(Wf), _ptr(uu), _ptr(g))
    return g


def divergence(nbr, W, p, precision="f64") -> np.ndarray:
    """Eq. 4 masked backward divergence of p [3, n, 512]; returns [n, 512]."""
    dt, sfx = _rt(precision)
    nbr = _np(nbr, np.int32)
    n = nbr.shape[0]
    Wf = _np(W, np.float32)
    pp = _np(p, dt)
    d = np.zeros((n, 512), dt)
    getattr(lib(), f"orc_divergence_{sfx}")(n, _ptr(nbr), _ptr(Wf), _ptr(pp), _ptr(d))
    return d


def regularise(coords, f, W, lam, eps, tau, sigma, iters, theta=1.0, data_term=0, init=0, precision="f64",
               state=None, nbr=None, omp=False, native=False):
    """Run `iters` CP iterations; returns (u, ubar, p) with u, ubar [n, 512] and p [3, n, 512].

    `state` = (u, ubar, p) resumes from a previous call.  Parameters are rounded to fp32 first
    (the values the product path receives), then widened for the fp64 oracle.
    """
    dt, sfx = _rt(precision)
    if nbr is None:
        nbr = neighbours(coords)
    nbr = _np(nbr, np.int32)
    n = nbr.shape[0]
    ff = _np(f, np.float32).reshape(n, 512)
    Wf = _np(W, np.float32).reshape(n, 512)
    if state is None:
        u = np.zeros((n, 512), dt)
        ub = np.zeros((n, 512), dt)
        p = np.zeros((3, n, 512), dt)
        resume = 0
    else:
        u, ub, p = (np.array(a, dtype=dt, copy=True) for a in state)
        resume = 1
    r32 = lambda x: float(np.float32(x))
    getattr(lib(omp, native), f"orc_regularise_{sfx}")(n, _ptr(nbr), _ptr(ff), _ptr(Wf), r32(lam), r32(eps), r32(tau),
                                            r32(sigma), r32(theta), int(data_term), int(init), int(iters),
                                            _ptr(u), _ptr(ub), _ptr(p), resume)
    return u, ub, p


def phase(coords, f, W, lam, eps, tau, sigma, which, state, theta=1.0, data_term=0, precision="f64", nbr=None):
    """One phase of the iteration on `state` = (u, ubar, p), updated in place and returned:
    which = "dual" (Eq. 3 + Eq. 7 with Huber) or "primal" (Eq. 4 + Eq. 8 + Eq. 9 relaxation).
    `regularise` is dual then primal, `iters` times; tests use the split to replay other schedules."""
    dt, sfx = _rt(precision)
    if nbr is None:
        nbr = neighbours(coords)
    nbr = _np(nbr, np.int32)
    n = nbr.shape[0]
    ff = _np(f, np.float32).reshape(n, 512)
    Wf = _np(W, np.float32).reshape(n, 512)
    u, ub, p = state
    for a in (u, ub, p):
        assert a.dtype == dt and a.flags.c_contiguous
    r32 = lambda x: float(np.float32(x))
    rc = getattr(lib(), f"orc_phase_{sfx}")(n, _ptr(nbr), _ptr(ff), _ptr(Wf), r32(lam), r32(eps), r32(tau), r32(sigma),
                                            r32(theta), int(data_term), {"dual": 0, "primal": 1}[which],
                                            _ptr(u), _ptr(ub), _ptr(p))
    assert rc == 0
    return u, ub, p


def regularise_scene(scene, precision="f64", iters=None, state=None, nbr=None):
    it = scene.iters if iters is None else iters
    return regularise(scene.coords, scene.f, scene.W, scene.lam, scene.eps, scene.tau, scene.sigma, it,
                      theta=scene.theta, data_term=scene.data_term, init=scene.init, precision=precision,
                      state=state, nbr=nbr)


def energy(nbr, f, W, u, lam, eps, data_term=0, p=None):
    """(primal, dual) in fp64; dual is None when p is None."""
    nbr = _np(nbr, np.int32)
    n = nbr.shape[0]
    ff = _np(f, np.float32)
    Wf = _np(W, np.float32)
    uu = _np(u, np.float64)
    out = np.zeros(2, np.float64)
    pp = _np(p, np.float64) if p is not None else None
    r32 = lambda x: float(np.float32(x))
    lib().orc_energy(n, _ptr(nbr), _ptr(ff), _ptr(Wf), _ptr(uu), _ptr(pp) if pp is not None else None,
                     r32(lam), r32(eps), int(data_term), _ptr(out[0:1]), _ptr(out[1:2]))
    return float(out[0]), (float(out[1]) if p is not None else None)


# ---------------------------------------------------------------------------------------------------
# TSDF fusion (paper §III-A, Eq. 1; fusion_oracle.c).  All arithmetic is fp32 in the written order.
# ---------------------------------------------------------------------------------------------------

def tsdf_update(f, w, sdf, mu, w_max=1e30):
    """Eq. 1 for one voxel: returns (f, w, updated)."""
    ff = np.array([f], np.float32)
    ww = np.array([w], np.float32)
    up = lib().orc_tsdf_update(_ptr(ff), _ptr(ww), float(np.float32(sdf)), float(np.float32(mu)),
                               float(np.float32(w_max)))
    return float(ff[0]), float(ww[0]), bool(up)


def project(pose, intr, H, Wd, p):
    """Steps 1-2 of P:160-164: (i, j, z_c) of the nearest pixel of global point p, or None."""
    ps = _np(pose, np.float32).reshape(12)
    it = _np(intr, np.float32).reshape(4)
    i, j = np.zeros(1, np.int32), np.zeros(1, np.int32)
    z = np.zeros(1, np.float32)
    ok = lib().orc_project(_ptr(ps), _ptr(it), int(H), int(Wd), float(np.float32(p[0])), float(np.float32(p[1])),
                           float(np.float32(p[2])), _ptr(i), _ptr(j), _ptr(z))
    return (int(i[0]), int(j[0]), float(z[0])) if ok else None


def block_walk(a, b, Bm, max_cells=100000) -> np.ndarray:
    """Reading F-7 lattice walk of blocks from point a to point b (metres); [m, 3] int32."""
    aa = _np(a, np.float32).reshape(3)
    bb = _np(b, np.float32).reshape(3)
    cells = np.zeros((max_cells, 3), np.int32)
    m = lib().orc_block_walk(_ptr(aa), _ptr(bb), float(np.float32(Bm)), _ptr(cells), max_cells)
    assert m <= max_cells
    return cells[:m].copy()


def _fusion_inputs(depth, intr, poses):
    D = _np(depth, np.float32)
    if D.ndim == 2:
        D = D[None]
    K, H, Wd = D.shape
    return D, K, H, Wd, _np(intr, np.float32).reshape(4), _np(poses, np.float32).reshape(K, 12)


def fuse(depth, intr, poses, voxel, mu, max_range, w_max):
    """Sequential fusion of K depth maps (allocation then update, frame by frame).
    Returns (xyz [n,3] int32 sorted by (x,y,z), first [n] int32, f [n,512], W [n,512])."""
    D, K, H, Wd, it, ps = _fusion_inputs(depth, intr, poses)
    r = lambda x: float(np.float32(x))
    n = lib().orc_fuse(_ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range), r(w_max), 0,
                       None, None, None, None)
    if n < 0:
        raise ValueError("fusion oracle: block walk out of range")
    xyz = np.zeros((max(n, 1), 3), np.int32)
    first = np.zeros(max(n, 1), np.int32)
    f = np.zeros((max(n, 1), 512), np.float32)
    W = np.zeros((max(n, 1), 512), np.float32)
    n2 = lib().orc_fuse(_ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range), r(w_max), n,
                        _ptr(xyz), _ptr(first), _ptr(f), _ptr(W))
    assert n2 == n
    return xyz[:n], first[:n], f[:n], W[:n]


def fuse_incremental(prev, depth, intr, poses, voxel, mu, max_range, w_max):
    """Continue a fusion: prev = (xyz [m,3], f [m,512], W [m,512]) of earlier frames, then the new depth
    maps in sequence (reading F-11).  Returns (xyz, first, f, W) like :func:`fuse` (first = −1 for the
    previous blocks)."""
    px = _np(prev[0], np.int32).reshape(-1, 3)
    m = px.shape[0]
    pf = _np(prev[1], np.float32).reshape(m, 512)
    pw = _np(prev[2], np.float32).reshape(m, 512)
    D, K, H, Wd, it, ps = _fusion_inputs(depth, intr, poses)
    r = lambda x: float(np.float32(x))
    args = (_ptr(px), _ptr(pf), _ptr(pw), m, _ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range),
            r(w_max))
    n = lib().orc_fuse_incremental(*args, 0, None, None, None, None)
    if n == -2:
        raise ValueError("fusion oracle: repeated block in prev")
    if n < 0:
        raise ValueError("fusion oracle: block walk out of range")
    xyz = np.zeros((max(n, 1), 3), np.int32)
    first = np.zeros(max(n, 1), np.int32)
    f = np.zeros((max(n, 1), 512), np.float32)
    W = np.zeros((max(n, 1), 512), np.float32)
    lib().orc_fuse_incremental(*args, n, _ptr(xyz), _ptr(first), _ptr(f), _ptr(W))
    return xyz[:n], first[:n], f[:n], W[:n]


def fuse_alloc(depth, intr, poses, voxel, mu, max_range):
    """Allocation passes only: (xyz [n,3] sorted by (x,y,z), first [n])."""
    D, K, H, Wd, it, ps = _fusion_inputs(depth, intr, poses)
    r = lambda x: float(np.float32(x))
    n = lib().orc_fuse_alloc(_ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range), 0, None, None)
    if n < 0:
        raise ValueError("fusion oracle: block walk out of range")
    xyz = np.zeros((max(n, 1), 3), np.int32)
    first = np.zeros(max(n, 1), np.int32)
    lib().orc_fuse_alloc(_ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range), n, _ptr(xyz),
                         _ptr(first))
    return xyz[:n], first[:n]


def fuse_update_blocks(depth, intr, poses, voxel, mu, max_range, w_max, xyz, first):
    """Update passes for a subset of blocks (each from its allocating frame on): (f, W) [nb, 512]."""
    D, K, H, Wd, it, ps = _fusion_inputs(depth, intr, poses)
    c = _np(xyz, np.int32).reshape(-1, 3)
    fr = _np(first, np.int32).reshape(-1)
    nb = c.shape[0]
    f = np.zeros((max(nb, 1), 512), np.float32)
    W = np.zeros((max(nb, 1), 512), np.float32)
    r = lambda x: float(np.float32(x))
    lib().orc_fuse_update_blocks(_ptr(D), K, H, Wd, _ptr(it), _ptr(ps), r(voxel), r(mu), r(max_range), r(w_max),
                                 _ptr(c), _ptr(fr), nb, _ptr(f), _ptr(W))
    return f[:nb], W[:nb]


# ---------------------------------------------------------------------------------------------------
# Ω-restricted isosurface extraction (marching tetrahedra; extract_oracle.c)
# ---------------------------------------------------------------------------------------------------

def extract(coords, u, W, voxel, w_min=0.0) -> np.ndarray:
    """Triangle soup [m, 3, 3] float32 of the zero level set of u over the fully observed cells."""
    c = _np(coords, np.int32).reshape(-1, 3)
    n = c.shape[0]
    uu = _np(u, np.float32).reshape(n, 512)
    ww = _np(W, np.float32).reshape(n, 512)
    r = lambda x: float(np.float32(x))
    m = lib().orc_extract(_ptr(c), n, _ptr(uu), _ptr(ww), r(voxel), r(w_min), None, 0)
    out = np.zeros((max(m, 1), 3, 3), np.float32)
    m2 = lib().orc_extract(_ptr(c), n, _ptr(uu), _ptr(ww), r(voxel), r(w_min), _ptr(out), m)
    assert m2 == m
    return out[:m]


# ---------------------------------------------------------------------------------------------------
# Depth-map estimation (paper §IV: census data term + tensor TGV; stereo_oracle.c)
# ---------------------------------------------------------------------------------------------------

class orc_stereo_params(ctypes.Structure):
    _fields_ = [("win", ctypes.c_int), ("D", ctypes.c_int), ("outer", ctypes.c_int), ("inner", ctypes.c_int),
                ("lam", ctypes.c_float), ("alpha1", ctypes.c_float), ("alpha2", ctypes.c_float),
                ("beta", ctypes.c_float), ("gamma", ctypes.c_float), ("theta0", ctypes.c_float),
                ("theta_end", ctypes.c_float), ("tau", ctypes.c_float), ("sigma", ctypes.c_float)]


def stereo_params(D=64, win=5, outer=10, inner=10, lam=0.5, alpha1=1.0, alpha2=5.0, beta=1.0, gamma=4.0,
                  theta0=1.0, theta_end=0.01, tau=None, sigma=None):
    t = float(np.float32(1.0 / np.sqrt(12.0)))
    return orc_stereo_params(win, D, outer, inner, lam, alpha1, alpha2, beta, gamma, theta0, theta_end,
                             t if tau is None else tau, t if sigma is None else sigma)


def census(I, win=5) -> np.ndarray:
    A = _np(I, np.float32)
    H, W = A.shape
    out = np.zeros((H, W), np.uint32)
    lib().orc_census(_ptr(A), H, W, win, _ptr(out))
    return out


def cost_volume(sigL, sigR, D, win=5) -> np.ndarray:
    """[H, W, D] uint8 Hamming distances (win² − 1 where x + d leaves the image)."""
    L_ = _np(sigL, np.uint32)
    R_ = _np(sigR, np.uint32)
    H, W = L_.shape
    out = np.zeros((H, W, D), np.uint8)
    lib().orc_cost(_ptr(L_), _ptr(R_), H, W, D, win, _ptr(out))
    return out


def tensor(I, beta=1.0, gamma=4.0) -> np.ndarray:
    A = _np(I, np.float32)
    H, W = A.shape
    out = np.zeros((H, W, 3), np.float32)
    lib().orc_tensor(_ptr(A), H, W, float(np.float32(beta)), float(np.float32(gamma)), _ptr(out))
    return out


def tgv_K(T, d, w):
    T_ = _np(T, np.float32)
    d_ = _np(d, np.float32)
    w_ = _np(w, np.float32)
    H, W = d_.shape
    u = np.zeros((2, H, W), np.float32)
    v = np.zeros((4, H, W), np.float32)
    lib().orc_tgv_K(_ptr(T_), _ptr(d_), _ptr(w_), H, W, _ptr(u), _ptr(v))
    return u, v


def tgv_KT(T, p, q):
    T_ = _np(T, np.float32)
    p_ = _np(p, np.float32)
    q_ = _np(q, np.float32)
    H, W = p_.shape[1:]
    kd = np.zeros((H, W), np.float32)
    kw = np.zeros((2, H, W), np.float32)
    tp = np.zeros((2, H, W), np.float32)
    lib().orc_tgv_KT(_ptr(T_), _ptr(p_), _ptr(q_), H, W, _ptr(kd), _ptr(kw), _ptr(tp))
    return kd, kw


def data_step(d, rho, c, lam) -> float:
    r = _np(rho, np.float32)
    return float(lib().orc_data_step(float(np.float32(d)), _ptr(r), r.shape[0], float(np.float32(c)),
                                     float(np.float32(lam))))


def stereo(IL, IR, params=None, **kw):
    """Solve one rectified pair; returns (d [H, W], w [2, H, W], a [H, W]) float32."""
    P = params if params is not None else stereo_params(**kw)
    L_ = _np(IL, np.float32)
    R_ = _np(IR, np.float32)
    H, W = L_.shape
    d = np.zeros((H, W), np.float32)
    w = np.zeros((2, H, W), np.float32)
    a = np.zeros((H, W), np.float32)
    rc = lib().orc_stereo(_ptr(L_), _ptr(R_), H, W, ctypes.byref(P), _ptr(d), _ptr(w), _ptr(a))
    if rc != 0:
        raise ValueError("stereo oracle: bad parameters")
    return d, w, a
