"""Seeded synthetic depth maps and camera poses for the TSDF fusion row.

Input plumbing only: this module renders depth maps of the analytic synthetic scenes by ray casting
(exact ray/plane, ray/box and ray/sphere intersections) and adds stereo-like noise.  It contains none
of the fusion arithmetic (projection, TSDF update, block allocation); the oracle and the GPU path
both receive its outputs as inputs.

Camera model (DESIGN.md "Fusion readings" F-1, F-6): pinhole, intrinsics (fx, fy, cx, cy) in pixels,
pixel (i, j) = column i, row j, its viewing ray in the camera frame is ((i − cx)/fx, (j − cy)/fy, 1),
so the ray parameter is the camera depth z_c.  Pose T_gc = [R | t] maps camera to global
(p_g = R p_c + t), row-major 3×4, float32 (the paper's T_gc).  Camera axes: x right, y down,
z forward.

Depth-map conventions: metres, +inf where the ray meets nothing (sky), 0 for dropped-out pixels; the
fusion treats non-finite, <= 0 and > max_range as invalid.

Scenes:
  fusion-tiny    the tiny sphere (r = 0.4 m at the origin, config 1 geometry) seen by 8 cameras on a
                 ring of radius 1.2 m looking at the centre, 160×120 px, v = 0.02 m, μ = 0.1 m;
  fusion-street  the config-2 street canyon (same boxes as synth.street) seen by a forward camera every
                 1 m along the road at 1.5 m height (61 frames), 1240×376 px, fx = fy = 720, small
                 random yaw/pitch jitter, v = 0.05 m, μ = 0.3 m, range cap 25 m, weight cap 30.
                 Synthetic stand-in for the paper's KITTI stereo depth maps; no KITTI
                 data or calibration is used.
Noise: d ← d + N(0, k·d²) (stereo depth error grows with d², k = 0.002 /m), then i.i.d. dropout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import rng
from .scenes import CAM_Z, HALF_WIDTH, STREET_H, CONFIG_IDS, Segment, _make_boxes

S_POSE, S_DEPTH_NOISE, S_DEPTH_NOISE2, S_DROPOUT = 11, 12, 13, 14


@dataclass
class DepthSet:
    name: str
    depth: torch.Tensor        # float32 [K, H, W] metres
    poses: torch.Tensor        # float32 [K, 12] row-major T_gc (camera-to-global)
    intr: torch.Tensor         # float32 [4] (fx, fy, cx, cy)
    voxel: float
    mu: float
    max_range: float
    w_max: float
    meta: dict = field(default_factory=dict)

    @property
    def K(self) -> int:
        return int(self.depth.shape[0])

    @property
    def H(self) -> int:
        return int(self.depth.shape[1])

    @property
    def Wd(self) -> int:
        return int(self.depth.shape[2])

    def params(self) -> dict:
        return dict(voxel=self.voxel, mu=self.mu, max_range=self.max_range, w_max=self.w_max)

    def to(self, device) -> "DepthSet":
        return DepthSet(self.name, self.depth.to(device), self.poses.to(device), self.intr.to(device), self.voxel,
                        self.mu, self.max_range, self.w_max, dict(self.meta))


def look_at(cam, target) -> np.ndarray:
    """Camera-to-global rotation [right, down, forward] (columns) of a camera at `cam` looking at `target`."""
    fwd = np.asarray(target, np.float64) - np.asarray(cam, np.float64)
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], 1)


def _pose12(R, t) -> np.ndarray:
    return np.concatenate([np.asarray(R, np.float64), np.asarray(t, np.float64).reshape(3, 1)], 1).reshape(12)


def pixel_rays(pose64: torch.Tensor, intr, H: int, Wd: int):
    """Global ray origins [3] and directions [H, W, 3] (camera-depth parameterised), float64."""
    fx, fy, cx, cy = (float(v) for v in intr)
    dev = pose64.device
    j = torch.arange(H, dtype=torch.float64, device=dev)[:, None].expand(H, Wd)
    i = torch.arange(Wd, dtype=torch.float64, device=dev)[None, :].expand(H, Wd)
    dc = torch.stack([(i - cx) / fx, (j - cy) / fy, torch.ones_like(i)], -1)
    T = pose64.view(3, 4)
    R, t = T[:, :3], T[:, 3]
    return t, dc @ R.T


def _noise_and_dropout(depth, seed, cfg, frame, k_noise, p_drop):
    K, H, Wd = 1, depth.shape[0], depth.shape[1]
    del K
    ctr = (torch.arange(H * Wd, device=depth.device, dtype=torch.int64) + (int(frame) << 32)).view(H, Wd)
    n = rng.normal(rng.stream_key(seed, cfg, S_DEPTH_NOISE), rng.stream_key(seed, cfg, S_DEPTH_NOISE2), ctr)
    d = depth + k_noise * depth * depth * n
    drop = rng.uniform(rng.stream_key(seed, cfg, S_DROPOUT), ctr) < p_drop
    d = torch.where(drop & torch.isfinite(depth), torch.zeros_like(d), d)
    return d


# ----------------------------------------------------------------------------------------------- tiny

def sphere_depth(seed: int = 0, n_cams: int = 8, H: int = 120, Wd: int = 160, radius: float = 0.4,
                 ring: float = 1.2, k_noise: float = 0.002, p_drop: float = 0.02, device="cpu") -> DepthSet:
    """fusion-tiny: the config-1 sphere seen from a ring of cameras (analytic ray/sphere depth)."""
    cfg = CONFIG_IDS["tiny"]
    f = 150.0
    intr = np.array([f, f, (Wd - 1) / 2.0, (H - 1) / 2.0], np.float32)
    poses, depths = [], []
    for k in range(n_cams):
        a = 2.0 * math.pi * k / n_cams
        cam = np.array([ring * math.cos(a), ring * math.sin(a), 0.3 * math.sin(2.0 * a)])
        R = look_at(cam, [0.0, 0.0, 0.0])
        P = _pose12(R, cam).astype(np.float32)
        poses.append(P)
        o, dirs = pixel_rays(torch.tensor(P, dtype=torch.float64, device=device), intr, H, Wd)
        # |o + t d|^2 = r^2  ->  a t^2 + 2 b t + c = 0, nearest positive root
        aa = (dirs * dirs).sum(-1)
        bb = (dirs * o).sum(-1)
        cc = float((o * o).sum()) - radius * radius
        disc = bb * bb - aa * cc
        t = (-bb - torch.sqrt(torch.clamp(disc, min=0.0))) / aa
        t = torch.where((disc > 0) & (t > 0), t, torch.full_like(t, float("inf")))
        depths.append(_noise_and_dropout(t, seed, cfg, k, k_noise, p_drop))
    return DepthSet("fusion-tiny", torch.stack(depths).to(torch.float32).contiguous(),
                    torch.tensor(np.stack(poses)).to(device), torch.tensor(intr).to(device), voxel=0.02, mu=0.1,
                    max_range=5.0, w_max=100.0, meta=dict(seed=seed, radius=radius, ring=ring))


# ----------------------------------------------------------------------------------------------- street

def _street_hit(o, dirs, boxes, H_wall):
    """Camera depth of the first hit with the street canyon (ground z = 0, façades y = ±4 up to H, boxes)."""
    inf = torch.full(dirs.shape[:-1], float("inf"), dtype=dirs.dtype, device=dirs.device)
    t = inf.clone()
    dz = dirs[..., 2]
    tg = (0.0 - o[2]) / torch.where(dz < 0, dz, -torch.ones_like(dz))
    t = torch.where(dz < 0, torch.minimum(t, tg), t)
    dy = dirs[..., 1]
    for side in (1.0, -1.0):
        towards = (side * dy) > 0
        tw = (side * HALF_WIDTH - o[1]) / torch.where(towards, dy, torch.ones_like(dy))
        zw = o[2] + tw * dz
        ok = towards & (zw <= H_wall) & (zw >= 0.0)
        t = torch.where(ok, torch.minimum(t, tw), t)
    if boxes.shape[0]:
        lo = boxes[:, 0:3]
        hi = boxes[:, 3:6]
        D = dirs[..., None, :]
        D = torch.where(D.abs() < 1e-12, torch.full_like(D, 1e-12), D)
        t1 = (lo - o) / D
        t2 = (hi - o) / D
        tin = torch.minimum(t1, t2).max(-1).values
        tout = torch.maximum(t1, t2).min(-1).values
        hit = (tin <= tout) & (tin > 0)
        tb = torch.where(hit, tin, torch.full_like(tin, float("inf"))).min(-1).values
        t = torch.minimum(t, tb)
    return t


def street_depth(seed: int = 0, length: float = 60.0, step: float = 1.0, H: int = 376, Wd: int = 1240,
                 fpx: float = 720.0, k_noise: float = 0.002, p_drop: float = 0.03, H_wall: float = STREET_H,
                 device="cpu", frames=None) -> DepthSet:
    """fusion-street: forward camera along the config-2 street canyon (same boxes as synth.street)."""
    cfg = CONFIG_IDS["street"]
    seg = Segment(0.0, 0.0, 1.0, 0.0, length)
    boxes = _make_boxes(seed, cfg, [seg], 20.0 / 60.0, device)[0].to(torch.float64)
    intr = np.array([fpx, fpx, (Wd - 1) / 2.0, (H - 1) / 2.0], np.float32)
    n = int(math.floor(length / step + 1e-9)) + 1
    ks = range(n) if frames is None else frames
    key = rng.stream_key(seed, cfg, S_POSE)
    poses, depths = [], []
    for k in ks:
        u = rng.uniform(key, torch.tensor([2 * k, 2 * k + 1], dtype=torch.int64)).numpy()
        yaw = math.radians(4.0 * (u[0] - 0.5))       # ±2°
        pitch = math.radians(2.0 * (u[1] - 0.5))     # ±1°
        cam = np.array([k * step, 0.0, CAM_Z])
        fwd = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
        R = look_at(cam, cam + fwd)
        P = _pose12(R, cam).astype(np.float32)
        poses.append(P)
        o, dirs = pixel_rays(torch.tensor(P, dtype=torch.float64, device=device), intr, H, Wd)
        t = _street_hit(o, dirs, boxes, H_wall)
        depths.append(_noise_and_dropout(t, seed, cfg, k, k_noise, p_drop).to(torch.float32))
    return DepthSet("fusion-street", torch.stack(depths).contiguous(), torch.tensor(np.stack(poses)).to(device),
                    torch.tensor(intr).to(device), voxel=0.05, mu=0.3, max_range=25.0, w_max=30.0,
                    meta=dict(seed=seed, length=length, step=step, H_wall=H_wall))


# ----------------------------------------------------------------------------------------------- planes (pins)

def plane_depth(pose12, intr, H: int, Wd: int, D: float) -> torch.Tensor:
    """Depth map of a plane perpendicular to the optical axis at camera depth D (constant D)."""
    del pose12, intr
    return torch.full((H, Wd), float(D), dtype=torch.float32)


def by_name(name: str, seed: int = 0, device="cpu", **kw) -> DepthSet:
    if name == "fusion-tiny":
        return sphere_depth(seed, device=device, **kw)
    if name == "fusion-street":
        return street_depth(seed, device=device, **kw)
    raise KeyError(name)
