"""O2: dense numpy brute force of the Ω-masked Chambolle-Pock iteration (TEST INFRASTRUCTURE ONLY).

A direct transcription of P:240-263 (Eqs. 3, 4) and P:290-321 (steps 1-4) on a dense grid that
covers the bounding box of the allocated blocks, with every unallocated voxel in Ω̄.  It
shares no code with O1 (hvg_oracle.c) or with the CUDA path: no hash table, no blocks, no
neighbour table — plain array shifts.  Readings as in SURVEY §8(c) (sign c-2, relaxation c-3,
edge-based divergence c-8, Huber c-12).  Every constant and array stays in the chosen dtype
(NumPy 2 / NEP 50: Python scalars do not upcast np.float32), and sums are written in x, y, z order,
so the fp32 result is bitwise comparable to O1's fp32 build.
"""
from __future__ import annotations

import numpy as np


def to_dense(coords, *fields, fill=0.0):
    """Scatter [n,512] block fields into dense [X,Y,Z] arrays over the block bounding box.

    Returns (origin_block, alloc_mask, dense_fields...)."""
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    lo = c.min(0)
    ext = (c.max(0) - lo + 1) * 8
    alloc = np.zeros(tuple(ext), dtype=bool)
    outs = [np.full(tuple(ext), fill, dtype=np.asarray(fld).dtype) for fld in fields]
    loc = np.arange(512)
    lx, ly, lz = loc % 8, (loc // 8) % 8, loc // 64
    for i, b in enumerate(c):
        o = (b - lo) * 8
        X, Y, Z = o[0] + lx, o[1] + ly, o[2] + lz
        alloc[X, Y, Z] = True
        for out, fld in zip(outs, fields):
            out[X, Y, Z] = np.asarray(fld)[i]
    return lo, alloc, outs


def from_dense(coords, lo, dense):
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    loc = np.arange(512)
    lx, ly, lz = loc % 8, (loc // 8) % 8, loc // 64
    out = np.zeros((c.shape[0], 512), dtype=dense.dtype)
    for i, b in enumerate(c):
        o = (b - lo) * 8
        out[i] = dense[o[0] + lx, o[1] + ly, o[2] + lz]
    return out


def _fwd(a, axis):
    """a(v + ê_axis), 0 beyond the grid."""
    out = np.zeros_like(a)
    sl_dst = [slice(None)] * 3
    sl_src = [slice(None)] * 3
    sl_dst[axis] = slice(0, -1)
    sl_src[axis] = slice(1, None)
    out[tuple(sl_dst)] = a[tuple(sl_src)]
    return out


def _bwd(a, axis):
    """a(v − ê_axis), 0 before the grid."""
    out = np.zeros_like(a)
    sl_dst = [slice(None)] * 3
    sl_src = [slice(None)] * 3
    sl_dst[axis] = slice(1, None)
    sl_src[axis] = slice(0, -1)
    out[tuple(sl_dst)] = a[tuple(sl_src)]
    return out


def edges(omega):
    """Valid forward edges e_a(v) = v ∈ Ω ∧ v + ê_a ∈ Ω (Eq. 3 cases 2-4)."""
    return [omega & _fwd(omega, a) for a in range(3)]


def gradient(u, omega):
    e = edges(omega)
    z = u.dtype.type(0)
    return [np.where(e[a], _fwd(u, a) - u, z) for a in range(3)]


def divergence(p, omega):
    e = edges(omega)
    z = p[0].dtype.type(0)
    term = []
    for a in range(3):
        own = np.where(e[a], p[a], z)
        prv = _bwd(own, a)  # [e_a(v−ê_a)]·p_a(v−ê_a)
        term.append(own - prv)
    d = (term[0] + term[1]) + term[2]
    return np.where(omega, d, z)


def regularise(coords, f, W, lam, eps, tau, sigma, iters, theta=1.0, data_term=0, init=0, dtype=np.float64):
    """Dense CP run; returns u as [n, 512] in the caller's block order."""
    T = np.dtype(dtype).type
    r32 = lambda x: T(np.float32(x))
    lam, eps, tau, sigma, theta = (r32(x) for x in (lam, eps, tau, sigma, theta))
    lo, alloc, (fd, Wd) = to_dense(coords, np.asarray(f, np.float32), np.asarray(W, np.float32))
    omega = alloc & (Wd > 0)
    f_ = fd.astype(dtype)
    W_ = Wd.astype(dtype)
    one = T(1)
    u = np.where(omega & (init == 1), T(0), f_).astype(dtype)
    ub = u.copy()
    p = [np.zeros_like(u) for _ in range(3)]
    kappa = one / (one + sigma * eps)          # Huber damping 1/(1+σε), applied as a product (c-18)
    tl = tau * lam
    t = tl * W_
    for _ in range(iters):
        g = gradient(ub, omega)
        q = [(p[a] + sigma * g[a]) * kappa for a in range(3)]
        nrm = np.sqrt((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2])
        r = one / np.where(nrm > one, nrm, one)  # p = q · (1 / max(1, ‖q‖₂))
        p = [np.where(omega, q[a] * r, T(0)) for a in range(3)]
        d = divergence(p, omega)
        ut = u + tau * d
        if data_term == 0:
            r = ut - f_
            un = np.where(r > t, ut - t, np.where(r < -t, ut + t, f_))
        else:
            un = (ut + t * f_) / (one + t)
        un = np.where(omega, un, u)
        ub = np.where(omega, un + theta * (un - u), ub)
        u = un
    return from_dense(coords, lo, u)
