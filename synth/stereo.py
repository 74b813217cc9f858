"""Seeded synthetic rectified stereo pairs for the depth-map estimation row.

Input plumbing only (no census, tensor or TGV arithmetic).  Convention (reading S-1):
the right image is the reference; a scene point at depth z seen at column x in the right image is at
column x + d in the left image with d = f·B/z ≥ 0, so I_L(x + d, y) = I_R(x, y).

  plane_pair   a textured plane (2-D value noise in right-image coordinates) with disparity
               d(x, y) = a·x + b·y + c; the left image is rendered through the exact inverse map;
  street_pair  the config-2 street canyon rendered by exact ray casting from a stereo rig (baseline
               0.54 m, fx = fy = 720, 1240×376, both cameras looking down the road at 1.5 m) with a
               solid 3-D value-noise texture on every surface; ground-truth disparity of the right view.
               A synthetic stand-in for KITTI stereo pairs; no KITTI data is used.
Intensities are in [0, 1].
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import rng
from .depth import _street_hit, look_at, pixel_rays, _pose12
from .scenes import CAM_Z, CONFIG_IDS, STREET_H, Segment, _make_boxes

S_TEX2, S_TEX3 = 15, 16


def _lattice(key, ix, iy, iz=None):
    c = (ix.to(torch.int64) & 0xFFFFF) | ((iy.to(torch.int64) & 0xFFFFF) << 20)
    if iz is not None:
        c = c | ((iz.to(torch.int64) & 0xFFFFF) << 40)
    return rng.uniform(key, c)


def value_noise2(x, y, seed=0, cells=(2.0, 5.0, 13.0, 31.0)):
    """Sum of bilinear value-noise octaves at the given cell sizes (pixels), in [0, 1]."""
    out = torch.zeros_like(x)
    wsum = 0.0
    for o, cs in enumerate(cells):
        key = rng.stream_key(seed, 100 + o, S_TEX2)
        u, v = x / cs, y / cs
        i0, j0 = torch.floor(u), torch.floor(v)
        fu, fv = u - i0, v - j0
        fu = fu * fu * (3 - 2 * fu)
        fv = fv * fv * (3 - 2 * fv)
        a = _lattice(key, i0, j0)
        b = _lattice(key, i0 + 1, j0)
        c = _lattice(key, i0, j0 + 1)
        d = _lattice(key, i0 + 1, j0 + 1)
        val = (a * (1 - fu) + b * fu) * (1 - fv) + (c * (1 - fu) + d * fu) * fv
        wgt = 1.0 / (1 + o)
        out = out + wgt * val
        wsum += wgt
    return out / wsum


def value_noise3(P, seed=0, cells=(0.03, 0.08, 0.2, 0.5, 1.2), footprint=None):
    """Solid 3-D value noise (trilinear octaves, cell sizes in metres) at points P [..., 3], in [0, 1].

    `footprint` (metres per pixel at each point) band-limits the texture like a mip-map: an octave fades
    out as its cell shrinks below two pixels, so point-sampled views of the same surface stay
    correlated (a real camera integrates over the pixel)."""
    out = torch.zeros(P.shape[:-1], dtype=P.dtype, device=P.device)
    wsum = torch.zeros_like(out) if footprint is not None else 0.0
    for o, cs in enumerate(cells):
        key = rng.stream_key(seed, 200 + o, S_TEX3)
        U = P / cs
        I0 = torch.floor(U)
        F = U - I0
        F = F * F * (3 - 2 * F)
        acc = torch.zeros_like(out)
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    wv = (F[..., 0] if dx else 1 - F[..., 0]) * (F[..., 1] if dy else 1 - F[..., 1]) * \
                         (F[..., 2] if dz else 1 - F[..., 2])
                    acc = acc + wv * _lattice(key, I0[..., 0] + dx, I0[..., 1] + dy, I0[..., 2] + dz)
        wgt = 1.0 / (1 + o)
        if footprint is not None:
            wgt = wgt * torch.clamp(cs / (2.0 * footprint) - 1.0, 0.0, 1.0)
        out = out + wgt * acc
        wsum = wsum + wgt
    if footprint is not None:
        return torch.where(wsum > 0, out / torch.clamp(wsum, min=1e-12), torch.full_like(out, 0.5))
    return out / wsum


def plane_pair(H=48, W=96, a=0.0, b=0.0, c=7.0, seed=0, device="cpu"):
    """(I_L, I_R, d_true) float32 [H, W] of a textured plane with disparity a·x + b·y + c (right view)."""
    y = torch.arange(H, dtype=torch.float64, device=device)[:, None].expand(H, W)
    x = torch.arange(W, dtype=torch.float64, device=device)[None, :].expand(H, W)
    IR = value_noise2(x, y, seed)
    # left pixel x' shows the right-image point x with x + a·x + b·y + c = x'
    xr = (x - b * y - c) / (1.0 + a)
    IL = value_noise2(xr, y, seed)
    d = a * x + b * y + c
    return IL.float().contiguous(), IR.float().contiguous(), d.float().contiguous()


def street_pair(seed: int = 0, frames=(0,), H: int = 376, Wd: int = 1240, fpx: float = 720.0,
                baseline: float = 0.54, length: float = 60.0, device="cpu", return_rig: bool = False):
    """(I_L, I_R, d_true) float32 [F, H, W] of the street canyon from a forward stereo rig at 1 m steps;
    with return_rig also the right (reference) cameras' poses T_gc [F, 12] float32, the intrinsics
    (fx, fy, cx, cy) and the baseline."""
    cfg = CONFIG_IDS["street"]
    seg = Segment(0.0, 0.0, 1.0, 0.0, length)
    boxes = _make_boxes(seed, cfg, [seg], 20.0 / 60.0, device)[0].to(torch.float64)
    intr = np.array([fpx, fpx, (Wd - 1) / 2.0, (H - 1) / 2.0])
    L, R, D, poses = [], [], [], []
    for k in frames:
        cam = np.array([float(k), 0.0, CAM_Z])
        Rm = look_at(cam, cam + np.array([1.0, 0.0, 0.0]))
        right_cam = cam + baseline * Rm[:, 0]         # +B along the camera x axis
        imgs = []
        for c in (cam, right_cam):
            P = torch.tensor(_pose12(Rm, c), dtype=torch.float64, device=device)
            o, dirs = pixel_rays(P, intr, H, Wd)
            t = _street_hit(o, dirs, boxes, STREET_H)
            hit = torch.isfinite(t)
            pts = o + dirs * torch.where(hit, t, torch.zeros_like(t))[..., None]
            tex = value_noise3(pts, seed, footprint=torch.where(hit, t, torch.ones_like(t)) / fpx)
            imgs.append((torch.where(hit, tex, torch.full_like(tex, 0.85)), t))   # sky: flat bright
        poses.append(_pose12(Rm, right_cam).astype(np.float32))
        L.append(imgs[0][0])
        R.append(imgs[1][0])
        z = imgs[1][1]
        D.append(torch.where(torch.isfinite(z), fpx * baseline / z, torch.zeros_like(z)))
    st = lambda xs: torch.stack(xs).to(torch.float32).contiguous()
    if return_rig:
        return st(L), st(R), st(D), torch.tensor(np.stack(poses), device=device), intr.astype(np.float32), baseline
    return st(L), st(R), st(D)
