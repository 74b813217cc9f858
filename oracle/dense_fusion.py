"""O2-fusion: numpy brute force of the TSDF update (paper §III-A, Eq. 1) on a dense "legacy voxel grid".

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  P:150: "If one considers each HVG voxel block to be
a legacy voxel grid, then the update equations are identical to those presented by [KinectFusion]" —
so this module fuses every voxel of a dense box (no hash, no blocks, no allocation) with steps 1-4 of
P:152-176, vectorised over voxels, one depth map after another.  On blocks that the sequential
hashed-grid oracle allocated in the first frame, the two must agree bit for bit (same fp32 formula
order: every array and constant is np.float32, NumPy 2 weak scalars do not upcast).
"""
from __future__ import annotations

import numpy as np

F = np.float32


def fuse_dense(depth, intr, poses, voxel, mu, max_range, w_max, lo, hi, precision="f32"):
    """Fuse K depth maps into the dense voxel box lo <= g <= hi (global voxel coords, inclusive).

    Returns (f, W) arrays of shape [nz, ny, nx] (index [gz−lo_z, gy−lo_y, gx−lo_x]).
    precision "f32": the written fp32 order of the hashed-grid oracle and the kernel (reading F-12: one
    reciprocal of z_c); "f64": every step in float64 with the paper's plain x/z, y/z — the
    independent-precision reference (inputs are the same fp32 numbers, widened).
    """
    if precision == "f64":
        return _fuse_dense_f64(depth, intr, poses, voxel, mu, max_range, w_max, lo, hi)
    D = np.asarray(depth, F)
    if D.ndim == 2:
        D = D[None]
    K, H, Wd = D.shape
    fx, fy, cx, cy = (F(v) for v in np.asarray(intr, F).reshape(4))
    P = np.asarray(poses, F).reshape(K, 12)
    v, mu, rmax, wmax = F(voxel), F(mu), F(max_range), F(w_max)
    gz, gy, gx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1), np.arange(lo[0], hi[0] + 1),
                             indexing="ij")
    # voxel centre (g + ½)·v (SURVEY §8(d) frame convention)
    px = (gx.astype(F) + F(0.5)) * v
    py = (gy.astype(F) + F(0.5)) * v
    pz = (gz.astype(F) + F(0.5)) * v
    f = np.zeros(px.shape, F)
    w = np.zeros(px.shape, F)
    for k in range(K):
        T = P[k]
        # step 1: p_c = R^T (p_g − t)
        d0, d1, d2 = px - T[3], py - T[7], pz - T[11]
        xc = (T[0] * d0 + T[4] * d1) + T[8] * d2
        yc = (T[1] * d0 + T[5] * d1) + T[9] * d2
        zc = (T[2] * d0 + T[6] * d1) + T[10] * d2
        front = zc > F(0)
        zs = np.where(front, zc, F(1))
        # step 2: nearest pixel
        with np.errstate(over="ignore", invalid="ignore"):
            rz = F(1) / zs                              # reading F-12: one reciprocal of z_c
            ix = fx * (xc * rz) + cx
            iy = fy * (yc * rz) + cy
            fi = np.floor(ix + F(0.5))
            fj = np.floor(iy + F(0.5))
        inside = front & (fi >= 0) & (fi < F(Wd)) & (fj >= 0) & (fj < F(H))
        ii = np.where(inside, fi, 0).astype(np.int64)
        jj = np.where(inside, fj, 0).astype(np.int64)
        d = D[k][jj, ii]
        valid = inside & np.isfinite(d) & (d > F(0)) & (d <= rmax)
        # step 3: u_SDF = d − z_c
        sdf = np.where(valid, d, F(0)) - zc
        # step 4, Eq. 1
        upd = valid & (sdf >= -mu)
        tsdf = np.minimum(np.maximum(sdf, -mu), mu) * (F(1) / mu)
        fn = (tsdf + w * f) / (w + F(1))
        wn = np.minimum(w + F(1), wmax)
        f = np.where(upd, fn, f).astype(F)
        w = np.where(upd, wn, w).astype(F)
    return f, w


def _fuse_dense_f64(depth, intr, poses, voxel, mu, max_range, w_max, lo, hi):
    """Steps 1-4 of P:152-176 in float64 (no reciprocal reading)."""
    G = np.float64
    D = np.asarray(depth, F).astype(G)
    if D.ndim == 2:
        D = D[None]
    K, H, Wd = D.shape
    fx, fy, cx, cy = (G(v) for v in np.asarray(intr, F).reshape(4))
    P = np.asarray(poses, F).reshape(K, 12).astype(G)
    v, mu, rmax, wmax = G(F(voxel)), G(F(mu)), G(F(max_range)), G(F(w_max))
    gz, gy, gx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1), np.arange(lo[0], hi[0] + 1),
                             indexing="ij")
    px, py, pz = (gx + 0.5) * v, (gy + 0.5) * v, (gz + 0.5) * v
    f = np.zeros(px.shape, G)
    w = np.zeros(px.shape, G)
    for k in range(K):
        T = P[k]
        d0, d1, d2 = px - T[3], py - T[7], pz - T[11]
        xc = T[0] * d0 + T[4] * d1 + T[8] * d2     # p_c = R^T (p_g − t)
        yc = T[1] * d0 + T[5] * d1 + T[9] * d2
        zc = T[2] * d0 + T[6] * d1 + T[10] * d2
        front = zc > 0
        zs = np.where(front, zc, 1.0)
        fi = np.floor(fx * xc / zs + cx + 0.5)     # nearest pixel
        fj = np.floor(fy * yc / zs + cy + 0.5)
        inside = front & (fi >= 0) & (fi < Wd) & (fj >= 0) & (fj < H)
        d = D[k][np.where(inside, fj, 0).astype(np.int64), np.where(inside, fi, 0).astype(np.int64)]
        valid = inside & np.isfinite(d) & (d > 0) & (d <= rmax)
        sdf = np.where(valid, d, 0.0) - zc
        upd = valid & (sdf >= -mu)
        tsdf = np.clip(sdf, -mu, mu) / mu
        f = np.where(upd, (tsdf + w * f) / (w + 1), f)
        w = np.where(upd, np.minimum(w + 1, wmax), w)
    return f, w
