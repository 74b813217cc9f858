"""O2-extraction: float64 numpy marching tetrahedra (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The independent-precision reference of the isosurface extraction (readings X-1 … X-7):
the same cells, tetrahedra and triangle order as ``extract_oracle.c``, but written separately and in
float64, with the orientation of X-5 decided geometrically — (a, b, c, d) is positively oriented iff
det(P_b − P_a, P_c − P_a, P_d − P_a) > 0 — instead of by permutation parity.  Vertices: X-4's
p = P_lo + t·(P_hi − P_lo), t = u_lo/(u_lo − u_hi), in float64 from the fp32 field values.

Used by ``tests/test_gpu_extract.py`` (the kernel's fp32 vertices within 1e-6 of these, triangles equal
up to a cyclic rotation of their vertices, which keeps the orientation) and pinned against the C oracle
in ``tests/test_oracle_extract.py``.
"""
from __future__ import annotations

import numpy as np

# X-2: the 6 Freudenthal tetrahedra 000 → e_a → e_a + e_b → 111 for the axis permutations (a, b, c) in
# lexicographic order, listed as the axis order; the corner codes (i + 2j + 4k) follow from it.
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def _tet_corners(perm):
    """Corner codes in X-2's listing: 000 → e_a → e_a + e_b → 111, the last two swapped for an odd
    permutation (so that every listing is positively oriented)."""
    a, b, _ = perm
    c1 = 1 << a
    c2 = c1 | (1 << b)
    odd = sum(perm[i] > perm[j] for i in range(3) for j in range(i + 1, 3)) % 2 == 1
    return [0, c1, 7, c2] if odd else [0, c1, c2, 7]


def _offset(code):
    return np.array([code & 1, (code >> 1) & 1, code >> 2], np.int64)


def extract_f64(coords, u, W, voxel, w_min=0.0):
    """Triangle soup [m, 3, 3] float64 in X-7 order (caller block, cell, tetrahedron, triangle)."""
    c = np.asarray(coords, np.int64).reshape(-1, 3)
    n = c.shape[0]
    uu = np.asarray(u, np.float32).reshape(n, 512)
    ww = np.asarray(W, np.float32).reshape(n, 512)
    v = np.float64(np.float32(voxel))
    wmin = np.float32(w_min)
    # value and usability of every allocated voxel, by global voxel coordinate (X-1)
    val, use = {}, {}
    loc = np.arange(512)
    L = np.stack([loc % 8, (loc // 8) % 8, loc // 64], 1)
    for i in range(n):
        g = c[i] * 8 + L
        for j in range(512):
            key = (int(g[j, 0]), int(g[j, 1]), int(g[j, 2]))
            val[key] = float(uu[i, j])
            use[key] = bool(ww[i, j] > 0 and ww[i, j] >= wmin)
    tets = [_tet_corners(p) for p in _PERMS]
    out = []

    def edge(ga, ua, gb, ub):
        # X-4: ends ordered lexicographically by global voxel coordinate
        (gl, ul), (gh, uh) = sorted([(ga, ua), (gb, ub)], key=lambda e: e[0])
        t = ul / (ul - uh)
        Pl = (np.array(gl, np.float64) + 0.5) * v
        Ph = (np.array(gh, np.float64) + 0.5) * v
        return Pl + t * (Ph - Pl)

    for i in range(n):
        for j in range(512):
            o = c[i] * 8 + L[j]
            cg = [tuple(int(x) for x in o + _offset(k)) for k in range(8)]
            if not all(use.get(g, False) for g in cg):
                continue
            cv = [val[g] for g in cg]
            if all(x < 0 for x in cv) or not any(x < 0 for x in cv):
                continue
            for corners in tets:
                G = [cg[k] for k in corners]
                U = [np.float64(cv[k]) for k in corners]
                P = [np.array(g, np.float64) for g in G]
                ins = [q for q in range(4) if U[q] < 0]          # X-3
                if len(ins) in (0, 4):
                    continue

                def positive(a, b, cc, d):
                    return np.linalg.det(np.stack([P[b] - P[a], P[cc] - P[a], P[d] - P[a]])) > 0

                if len(ins) == 2:
                    a, b = ins
                    cc, d = [q for q in range(4) if q not in ins]
                    if not positive(a, b, cc, d):
                        cc, d = d, cc
                    E = lambda x, y: edge(G[x], U[x], G[y], U[y])
                    if U[d] != 0:                                 # X-6
                        out.append([E(a, cc), E(a, d), E(b, d)])
                    if U[cc] != 0:
                        out.append([E(a, cc), E(b, d), E(b, cc)])
                else:
                    a = ins[0] if len(ins) == 1 else [q for q in range(4) if q not in ins][0]
                    b, cc, d = [q for q in range(4) if q != a]
                    if not positive(a, b, cc, d):
                        cc, d = d, cc
                    E = lambda x, y: edge(G[x], U[x], G[y], U[y])
                    if len(ins) == 1:
                        out.append([E(a, b), E(a, cc), E(a, d)])
                    elif U[a] != 0:                               # X-6
                        out.append([E(a, b), E(a, d), E(a, cc)])
    return np.array(out, np.float64).reshape(-1, 3, 3)


def match_up_to_rotation(T, R):
    """Max over triangles of the smallest (over the 3 cyclic rotations of T's vertices) max-abs vertex
    deviation from R; T and R [m, 3, 3] in the same triangle order."""
    T = np.asarray(T, np.float64)
    R = np.asarray(R, np.float64)
    assert T.shape == R.shape, (T.shape, R.shape)
    if T.shape[0] == 0:
        return 0.0
    dev = np.stack([np.abs(np.roll(T, r, axis=1) - R).max(axis=(1, 2)) for r in range(3)], 1).min(1)
    return float(dev.max())
