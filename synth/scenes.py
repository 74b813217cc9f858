"""Seeded synthetic scenes for the hashed-voxel-grid TV regulariser (BASELINE.json configs).

A scene is a set of allocated 8³ voxel blocks (integer block coordinates, caller order) with a fused
TSDF f and a fusion weight W per voxel, plus the solver parameters of its config.  Voxel index inside
a block is x + 8y + 64z (x fastest); the global voxel coordinate is 8·B + (x, y, z) and the
voxel centre is (8·B + i + 0.5)·v metres.

Configs (names used by tests and bench.py):
  tiny          config 1: noisy sphere, v=0.02 m, μ=0.1 m, r=0.4 m, TV-L1 λ=1, 200 it
  tiny-stress   config 1 geometry with W ~ U{1,2,3}, λ=0.5 (SURVEY.md §8(c) parity-stress input)
  street        config 2: 60 m street canyon, v=0.05 m, μ=0.3 m, Huber-TV ε=0.01, λ=0.8, 300 it
  street-outlier config 3: street + 5 % impulse outliers + ≥30 % W=0 in 1 m³ clumps, TV-L1 λ=0.5, 500 it
  city          config 4: 1 km staircase route of canyons, v=0.1 m, μ=0.5 m, Huber-TV, 200 it
  city-weak     config 5 (weak): route prefix of 125·G m

The generator is input plumbing only: it contains none of the regulariser's arithmetic.  It runs on
any torch device (CPU for the small configs in the CPU test-suite, the GPU for street/city in bench).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import rng

TAU_DEFAULT = float(np.float32(1.0 / math.sqrt(12.0)))  # τ = σ = 1/√12 (config 1)

CONFIG_IDS = {"tiny": 1, "tiny-stress": 11, "street": 2, "street-outlier": 3, "city": 4, "city-weak": 5, "test": 99}


@dataclass
class Scene:
    name: str
    coords: torch.Tensor          # int32 [n, 3] block coordinates, caller order
    f: torch.Tensor               # float32 [n, 512]
    W: torch.Tensor               # float32 [n, 512]
    lam: float = 1.0
    eps: float = 0.0
    tau: float = TAU_DEFAULT
    sigma: float = TAU_DEFAULT
    theta: float = 1.0
    iters: int = 200
    data_term: int = 0            # 0 = weighted L1 (north_star), 1 = weighted L2 (paper Eq. 8)
    init: int = 0                 # 0 = warm u = ū = f, 1 = zero (paper step 1)
    meta: dict = field(default_factory=dict)

    @property
    def n_blocks(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_alloc(self) -> int:
        return 512 * self.n_blocks

    def n_omega(self) -> int:
        return int((self.W > 0).sum())

    def params(self) -> dict:
        return dict(lam=self.lam, eps=self.eps, tau=self.tau, sigma=self.sigma, theta=self.theta,
                    iters=self.iters, data_term=self.data_term, init=self.init)

    def to(self, device) -> "Scene":
        return Scene(self.name, self.coords.to(device), self.f.to(device), self.W.to(device), self.lam,
                     self.eps, self.tau, self.sigma, self.theta, self.iters, self.data_term, self.init,
                     dict(self.meta))

    def numpy(self):
        return self.coords.cpu().numpy(), self.f.cpu().numpy(), self.W.cpu().numpy()


# ----------------------------------------------------------------------------------------------
# lattice helpers
# ----------------------------------------------------------------------------------------------

def _local_xyz(device) -> torch.Tensor:
    i = torch.arange(512, device=device)
    return torch.stack([i % 8, (i // 8) % 8, i // 64], dim=1)  # [512, 3]


def global_voxel_coords(coords: torch.Tensor) -> torch.Tensor:
    """[n, 512, 3] int64 global voxel coordinates 8·B + (x, y, z)."""
    return coords.to(torch.int64)[:, None, :] * 8 + _local_xyz(coords.device)[None]


def voxel_centres(coords: torch.Tensor, v: float) -> torch.Tensor:
    """[n, 512, 3] float64 voxel centres in metres."""
    return (global_voxel_coords(coords).to(torch.float64) + 0.5) * v


def _block_grid(lo, hi, device) -> torch.Tensor:
    """All integer block coords with lo <= b <= hi (inclusive), x fastest, as int32 [m, 3]."""
    xs = torch.arange(lo[0], hi[0] + 1, device=device)
    ys = torch.arange(lo[1], hi[1] + 1, device=device)
    zs = torch.arange(lo[2], hi[2] + 1, device=device)
    z, y, x = torch.meshgrid(zs, ys, xs, indexing="ij")
    return torch.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], 1).to(torch.int32)


def _uniform(seed, cfg, stream, counter):
    return rng.uniform(rng.stream_key(seed, cfg, stream), counter)


def _normal(seed, cfg, counter):
    return rng.normal(rng.stream_key(seed, cfg, rng.S_NOISE), rng.stream_key(seed, cfg, rng.S_NOISE2), counter)


# ----------------------------------------------------------------------------------------------
# config 1: tiny sphere
# ----------------------------------------------------------------------------------------------

def tiny(seed: int = 0, stress: bool = False, device="cpu") -> Scene:
    """Config 1 (BASELINE.json configs[0]); `stress` gives SURVEY.md §8(c) 'tiny-stress'."""
    v, mu, r = 0.02, 0.1, 0.4
    cfg = CONFIG_IDS["tiny-stress" if stress else "tiny"]
    bmax = int(math.ceil((r + mu) / (8 * v))) + 1
    cand = _block_grid((-bmax,) * 3, (bmax,) * 3, device)
    c = voxel_centres(cand, v)
    dist = torch.linalg.norm(c, dim=2) - r
    keep = (dist.abs() <= mu).any(dim=1)
    coords = cand[keep].contiguous()
    dist = dist[keep]
    gv = global_voxel_coords(coords)
    ctr = rng.pack_coords(gv[..., 0], gv[..., 1], gv[..., 2])
    seed_cfg = CONFIG_IDS["tiny"]  # noise shared with the stress variant (same geometry, same noise)
    f = (dist / mu).clamp(-1.0, 1.0) + 0.1 * _normal(seed, seed_cfg, ctr)
    whi = 3 if stress else 10
    W = rng.uniform_int(rng.stream_key(seed, cfg, rng.S_W), ctr, 1, whi).to(torch.float64)
    W0 = _uniform(seed, seed_cfg, rng.S_W0, ctr) < 0.1
    W = torch.where(W0, torch.zeros_like(W), W)
    return Scene("tiny-stress" if stress else "tiny", coords, f.to(torch.float32).contiguous(),
                 W.to(torch.float32).contiguous(), lam=0.5 if stress else 1.0, eps=0.0, iters=200,
                 meta=dict(voxel=v, mu=mu, radius=r, seed=seed))


# ----------------------------------------------------------------------------------------------
# street / city geometry (configs 2-5)
# ----------------------------------------------------------------------------------------------

@dataclass
class Segment:
    """One straight canyon of the route: start point (x0, y0), unit heading d ∈ {±x, ±y}, length L."""
    x0: float
    y0: float
    dx: float
    dy: float
    L: float
    caps: bool = False   # end walls at s = −4 and s = L + 4 (city); the street is open-ended

    def local(self, X, Y):
        s = (X - self.x0) * self.dx + (Y - self.y0) * self.dy
        lat = -(X - self.x0) * self.dy + (Y - self.y0) * self.dx  # left normal (−dy, dx)
        return s, lat


HALF_WIDTH = 4.0   # façades at lateral ±4 m (8 m apart)
CAM_Z = 1.5


def _canyon_sd(seg: Segment, X, Y, Z, H):
    """Signed distance to the free space of one canyon (positive in free space), SURVEY §8(d)."""
    s, lat = seg.local(X, Y)
    inner = HALF_WIDTH - lat.abs()
    if seg.caps:
        inner = torch.minimum(inner, torch.minimum(s + HALF_WIDTH, seg.L + HALF_WIDTH - s))
    return torch.minimum(Z, torch.maximum(inner, Z - H))


_BOX_SD_DIRECT = 1 << 28   # points x boxes evaluated in one tensor; above it, sub-chunks with box culling


def _box_sd(X, Y, Z, boxes, cut=None):
    """min over axis-aligned boxes of the exterior signed distance (positive outside). boxes [k, 6].

    `cut`: callers only use min(sd, ·) clamped at or below `cut` (f = clamp(sd/μ), |sd| ≤ μ tests), so for
    large problems (city-heavy: thousands of boxes) points are processed in spatially compact sub-chunks
    and boxes farther than `cut` from a sub-chunk's bounding box are skipped: where the true minimum is
    < cut its box is kept, elsewhere both values are >= cut — identical results downstream.  Street and
    city stay below _BOX_SD_DIRECT and take the direct path."""
    if boxes.shape[0] == 0:
        return torch.full_like(X, float("inf"))
    if cut is not None and X.numel() * boxes.shape[0] > _BOX_SD_DIRECT:
        out = torch.empty_like(X)
        step = 16384
        for i in range(0, X.numel(), step):
            x, y, z = X[i:i + step], Y[i:i + step], Z[i:i + step]
            pmin = torch.stack([x.min(), y.min(), z.min()])
            pmax = torch.stack([x.max(), y.max(), z.max()])
            gap = torch.clamp(torch.maximum(boxes[:, 0:3] - pmax, pmin - boxes[:, 3:6]), min=0.0)
            near = torch.linalg.norm(gap, dim=1) <= cut
            out[i:i + step] = _box_sd(x, y, z, boxes[near]) if bool(near.any()) else float("inf")
        return out
    lo = boxes[:, 0:3]
    hi = boxes[:, 3:6]
    P = torch.stack([X, Y, Z], -1)[..., None, :]              # [..., 1, 3]
    c = (lo + hi) * 0.5
    h = (hi - lo) * 0.5
    q = (P - c).abs() - h                                       # [..., k, 3]
    outside = torch.linalg.norm(q.clamp(min=0.0), dim=-1)
    inside = q.max(dim=-1).values.clamp(max=0.0)
    return (outside + inside).min(dim=-1).values


def _near_segments(segs, X, Y, cut):
    """Capped segments whose footprint rectangle (s ∈ [−4, L+4], |lat| ≤ 4) lies at Chebyshev distance
    < cut from the points' xy bounding box; (kept, any_dropped).  A dropped segment has inner ≤ −cut at
    every point, so its canyon sd there is exactly Z − H when Z − H > −cut and ≤ −cut otherwise."""
    xmin, xmax, ymin, ymax = float(X.min()), float(X.max()), float(Y.min()), float(Y.max())
    kept = []
    for seg in segs:
        if not seg.caps:
            kept.append(seg)
            continue
        xs = [seg.x0 + a * seg.dx - b * seg.dy for a in (-HALF_WIDTH, seg.L + HALF_WIDTH) for b in (-HALF_WIDTH, HALF_WIDTH)]
        ys = [seg.y0 + a * seg.dy + b * seg.dx for a in (-HALF_WIDTH, seg.L + HALF_WIDTH) for b in (-HALF_WIDTH, HALF_WIDTH)]
        gx = max(min(xs) - xmax, xmin - max(xs), 0.0)
        gy = max(min(ys) - ymax, ymin - max(ys), 0.0)
        if max(gx, gy) < cut:
            kept.append(seg)
    return kept, len(kept) < len(segs)


def _scene_sd(X, Y, Z, segs, boxes, H, cut=None):
    """Union of the canyons' free space (max of their sd) minus the boxes (min).  With `cut` and many
    segments (city-heavy) only the segments near the points are evaluated; the dropped ones contribute
    exactly Z − H where that exceeds −cut (see _near_segments), so every value > −cut is unchanged and
    every value ≤ −cut stays ≤ −cut — identical after the clamp and the |sd| ≤ cut tests downstream."""
    if cut is not None and len(segs) > 8:
        kept, dropped = _near_segments(segs, X, Y, cut)
        sd = Z - H if dropped else None
        for seg in kept:
            c = _canyon_sd(seg, X, Y, Z, H)
            sd = c if sd is None else torch.maximum(sd, c)
        return torch.minimum(sd, _box_sd(X, Y, Z, boxes, cut))
    sd = _canyon_sd(segs[0], X, Y, Z, H)
    for seg in segs[1:]:
        sd = torch.maximum(sd, _canyon_sd(seg, X, Y, Z, H))
    return torch.minimum(sd, _box_sd(X, Y, Z, boxes, cut))


def _ray_first_hit(seg: Segment, cam, P, boxes, H):
    """Parameter t ∈ (0, 1] of the first solid hit on the segment cam→P (1e9 if none) in one canyon frame.

    Occluders: ground z = 0, the two façades (lateral ±4, z ≤ H), the end caps if any, and the boxes.
    cam: [3] float64 (camera inside the canyon), P: [N, 3].
    """
    inf = torch.full(P.shape[:1], 1e9, dtype=P.dtype, device=P.device)
    D = P - cam
    t = inf.clone()
    # ground
    hit = P[:, 2] < 0.0
    tg = (0.0 - cam[2]) / torch.where(hit, D[:, 2], -torch.ones_like(D[:, 2]))
    t = torch.where(hit, torch.minimum(t, tg), t)
    # façades: camera has lat 0; the wall plane lat = ±4 is crossed iff |lat(P)| > 4
    sP, latP = seg.local(P[:, 0], P[:, 1])
    sC, latC = seg.local(cam[0:1], cam[1:2])
    dl = latP - latC
    for side in (1.0, -1.0):
        cross = (side * latP) > HALF_WIDTH
        tw = (side * HALF_WIDTH - latC) / torch.where(cross, dl, torch.ones_like(dl))
        zw = cam[2] + tw * D[:, 2]
        ok = cross & (zw <= H)
        t = torch.where(ok, torch.minimum(t, tw), t)
    if seg.caps:
        ds = sP - sC
        for wall in (-HALF_WIDTH, seg.L + HALF_WIDTH):
            cross = (sP < wall) if wall < 0 else (sP > wall)
            tw = (wall - sC) / torch.where(cross, ds, torch.ones_like(ds))
            zw = cam[2] + tw * D[:, 2]
            ok = cross & (zw <= H)
            t = torch.where(ok, torch.minimum(t, tw), t)
    if boxes.shape[0]:
        lo = boxes[None, :, 0:3]
        hi = boxes[None, :, 3:6]
        Dd = D[:, None, :]
        Dd = torch.where(Dd.abs() < 1e-12, torch.full_like(Dd, 1e-12), Dd)
        t1 = (lo - cam) / Dd
        t2 = (hi - cam) / Dd
        tin = torch.minimum(t1, t2).max(dim=-1).values
        tout = torch.maximum(t1, t2).min(dim=-1).values
        hitb = (tin <= tout) & (tout > 0.0) & (tin < 1.0)
        tb = torch.where(hitb, tin.clamp(min=0.0), torch.full_like(tin, 1e9)).min(dim=-1).values
        t = torch.minimum(t, tb)
    return t


def _observations(P, segs, seg_samples, boxes_of_seg, H, mu, R):
    """W = number of camera samples that observe P in the TSDF sense (first hit ≥ dist − μ), capped at 30.

    A sample observes a voxel centre iff it is within range R and the first solid along the ray is at
    distance ≥ dist − μ (paper Eq. 1: w is incremented iff u_SDF ≥ −μ).
    """
    cnt = torch.zeros(P.shape[0], dtype=torch.int32, device=P.device)
    pmin, pmax = P.min(0).values, P.max(0).values
    for seg, cams, boxes in zip(segs, seg_samples, boxes_of_seg):
        for cam in cams:
            D = P - cam
            dist = torch.linalg.norm(D, dim=1)
            inr = dist <= R
            if not bool(inr.any()):
                continue
            # a box can only cut a segment cam→P if it meets the bounding box of cam and the points:
            # the others never register a hit in the slab test, so skipping them is exact
            if boxes.shape[0] > 4:
                lo, hi = torch.minimum(pmin, cam), torch.maximum(pmax, cam)
                meet = ((boxes[:, 3:6] >= lo) & (boxes[:, 0:3] <= hi)).all(dim=1)
                bx = boxes[meet]
            else:
                bx = boxes
            t = _ray_first_hit(seg, cam, P, bx, H)
            obs = inr & (t * dist >= dist - mu)
            cnt += obs.to(torch.int32)
    return cnt.clamp(max=30)


def _make_boxes(seed, cfg, segs, per_metre, device):
    """Random axis-aligned boxes (cars, kerbs) of size U[1,5] m on the ground of each segment.

    Lateral size is clipped to 3 m so the box fits in 1 ≤ |lat| ≤ 4 (keeps the camera corridor clear).
    Counter = global box index; stream S_BOX.
    """
    key = rng.stream_key(seed, cfg, rng.S_BOX)
    out = []
    gi = 0
    for seg in segs:
        k = max(1, int(round(per_metre * seg.L)))
        idx = torch.arange(gi * 8, (gi + k) * 8, device=device, dtype=torch.int64).view(k, 8)
        gi += k
        u = rng.uniform(key, idx)
        sx = 1.0 + 4.0 * u[:, 0]
        sl = torch.clamp(1.0 + 4.0 * u[:, 1], max=3.0)
        sz = 1.0 + 4.0 * u[:, 2]
        sc = seg.L * u[:, 3]
        side = torch.where(u[:, 4] < 0.5, -1.0, 1.0)
        l0 = 1.0 + (HALF_WIDTH - 1.0 - sl) * u[:, 5]
        lat_lo = torch.where(side > 0, l0, -(l0 + sl))
        lat_hi = lat_lo + sl
        s_lo, s_hi = sc - sx / 2, sc + sx / 2
        # local (s, lat) -> world; headings are axis aligned
        corners = []
        for s_, l_ in ((s_lo, lat_lo), (s_hi, lat_hi)):
            X = seg.x0 + s_ * seg.dx - l_ * seg.dy
            Y = seg.y0 + s_ * seg.dy + l_ * seg.dx
            corners.append((X, Y))
        X0, X1 = torch.minimum(corners[0][0], corners[1][0]), torch.maximum(corners[0][0], corners[1][0])
        Y0, Y1 = torch.minimum(corners[0][1], corners[1][1]), torch.maximum(corners[0][1], corners[1][1])
        out.append(torch.stack([X0, Y0, torch.zeros_like(sz), X1, Y1, sz], 1))
    return out


def _route_candidates(segs, boxes_per_seg, v, mu, H, device, near_pred=None, compact=False):
    """Candidate blocks of a route scene: every block whose centre lies within μ + half a block diagonal
    of a surface (a superset of the allocated blocks), slab by slab in x; int32 [m, 3]."""
    allboxes = torch.cat(boxes_per_seg, 0) if boxes_per_seg else torch.zeros(0, 6, dtype=torch.float64, device=device)
    B = 8 * v
    # candidate block range = route bounding box ± (4 m + 1 block), z in [−μ−B, H+μ+B]
    xs, ys = [], []
    for seg in segs:
        for s in (0.0, seg.L):
            xs.append(seg.x0 + s * seg.dx)
            ys.append(seg.y0 + s * seg.dy)
    pad = HALF_WIDTH + mu + B
    lo = (math.floor((min(xs) - pad) / B), math.floor((min(ys) - pad) / B), math.floor((-mu - B) / B))
    hi = (math.floor((max(xs) + pad) / B), math.floor((max(ys) + pad) / B), math.floor((H + mu + B) / B))
    half_diag = math.sqrt(3.0) * B / 2
    cand_all = []
    # enumerate candidate blocks slab by slab in x to bound memory
    for bx0 in range(lo[0], hi[0] + 1, 64):
        grid = _block_grid((bx0, lo[1], lo[2]), (min(bx0 + 63, hi[0]), hi[1], hi[2]), device)
        c = (grid.to(torch.float64) + 0.5) * B
        sd = _scene_sd(c[:, 0], c[:, 1], c[:, 2], segs, allboxes, H, cut=mu + half_diag)
        m = sd.abs() <= mu + half_diag
        if near_pred is not None:
            m &= near_pred(c)
        cand_all.append(grid[m])
    cand = torch.cat(cand_all, 0)
    if compact:
        # spatially compact chunks (16³-block super cells in x, y, z order) so each chunk's observation
        # work involves only the nearby segments and cameras (city-heavy: 13 parallel lanes); the
        # per-voxel values do not depend on the chunking, only the output block order does
        sc = (cand.to(torch.int64) >> 4) + (1 << 20)
        key = (sc[:, 0] << 42) | (sc[:, 1] << 21) | sc[:, 2]
        cand = cand[torch.argsort(key, stable=True)]
    return cand


def _route_alloc(cand, segs, boxes_per_seg, v, mu, H, device, chunk_blocks, R=25.0, cam_step=1.0):
    """sd and W (observation count) of every voxel of the candidate blocks, chunk by chunk; keeps the
    blocks with some voxel at |sd| ≤ μ and W > 0.  Every value depends only on the voxel and the scene,
    so any subset of candidates gives the same per-block result (per-shard generation)."""
    allboxes = torch.cat(boxes_per_seg, 0) if boxes_per_seg else torch.zeros(0, 6, dtype=torch.float64, device=device)
    # camera samples per segment
    seg_samples = []
    for seg in segs:
        n_s = int(math.floor(seg.L / cam_step + 1e-9)) + 1
        s = torch.arange(n_s, dtype=torch.float64, device=device) * cam_step
        cams = torch.stack([seg.x0 + s * seg.dx, seg.y0 + s * seg.dy, torch.full_like(s, CAM_Z)], 1)
        seg_samples.append(cams)
    keep_coords, keep_sd, keep_W = [], [], []
    for i in range(0, cand.shape[0], chunk_blocks):
        cb = cand[i:i + chunk_blocks]
        P = voxel_centres(cb, v).reshape(-1, 3)
        sd = _scene_sd(P[:, 0], P[:, 1], P[:, 2], segs, allboxes, H, cut=mu)
        # restrict observation work to segments whose samples can reach the chunk
        segs_i, cams_i, boxes_i = [], [], []
        pmin, pmax = P.min(0).values, P.max(0).values
        for seg, cams, bxs in zip(segs, seg_samples, boxes_per_seg):
            dmin = torch.clamp(torch.maximum(pmin[None, :2] - cams[:, :2], cams[:, :2] - pmax[None, :2]), min=0)
            near = torch.linalg.norm(dmin, dim=1) <= R
            if bool(near.any()):
                segs_i.append(seg)
                cams_i.append(cams[near])
                boxes_i.append(bxs)
        W = _observations(P, segs_i, cams_i, boxes_i, H, mu, R) if segs_i else torch.zeros(P.shape[0], dtype=torch.int32, device=device)
        sd = sd.view(-1, 512)
        W = W.view(-1, 512)
        alloc = ((sd.abs() <= mu) & (W > 0)).any(dim=1)
        keep_coords.append(cb[alloc])
        keep_sd.append(sd[alloc])
        keep_W.append(W[alloc])
    if not keep_coords:
        return (torch.zeros(0, 3, dtype=torch.int32, device=device), torch.zeros(0, 512, dtype=torch.float64, device=device),
                torch.zeros(0, 512, dtype=torch.float64, device=device))
    coords = torch.cat(keep_coords, 0).contiguous()
    sd = torch.cat(keep_sd, 0)
    W = torch.cat(keep_W, 0).to(torch.float64)
    return coords, sd, W


def _route_scene(name, segs, boxes_per_seg, v, mu, H, seed, cfg, device, chunk_blocks, R=25.0,
                 cam_step=1.0, near_pred=None, compact=False):
    """Shared body of street and city: candidate blocks → sd, W per voxel → allocation → f."""
    cand = _route_candidates(segs, boxes_per_seg, v, mu, H, device, near_pred, compact)
    return _route_alloc(cand, segs, boxes_per_seg, v, mu, H, device, chunk_blocks, R, cam_step)


def route_polyline(segs, z=CAM_Z):
    """Vertices [m, 3] (metres) of the camera path through the segments (the route of SURVEY §8(e))."""
    pts = [(segs[0].x0, segs[0].y0, z)]
    for s in segs:
        pts.append((s.x0 + s.L * s.dx, s.y0 + s.L * s.dy, z))
    return np.asarray(pts, np.float64)


def _street_noise(coords, sd, W, v, mu, seed, cfg, path_dist, want_ctr=True, chunk=65536):
    """f = clamp(sd/μ, −1, 1) + N(0, 0.02·d²), d = distance to the camera path; f = 0 where unobserved.
    Element-wise, evaluated in chunks of blocks (bounded temporaries for city-heavy); returns (f fp64,
    the voxel counters or None)."""
    n = coords.shape[0]
    f = torch.empty(n, 512, dtype=torch.float64, device=coords.device)
    ctr_all = torch.empty(n, 512, dtype=torch.int64, device=coords.device) if want_ctr else None
    for i in range(0, n, chunk):
        c = coords[i:i + chunk]
        gv = global_voxel_coords(c)
        ctr = rng.pack_coords(gv[..., 0], gv[..., 1], gv[..., 2])
        P = voxel_centres(c, v)
        d = path_dist(P)
        fi = (sd[i:i + chunk] / mu).clamp(-1.0, 1.0) + 0.02 * d * d * _normal(seed, cfg, ctr)
        f[i:i + chunk] = torch.where(W[i:i + chunk] > 0, fi, torch.zeros_like(fi))
        if want_ctr:
            ctr_all[i:i + chunk] = ctr
    return f, ctr_all


STREET_H = 25.0   # façade height (SURVEY §8(d) "calibrate so N_alloc ≈ 3e7 ± 30 %, then freeze")


def street(seed: int = 0, outlier: bool = False, length: float = 60.0, H: float = STREET_H,
           device="cpu", chunk_blocks: int = 2048) -> Scene:
    """Config 2 (street) or config 3 (street-outlier); `length` < 60 gives a reduced test variant."""
    v, mu = 0.05, 0.3
    cfg = CONFIG_IDS["street"]
    seg = Segment(0.0, 0.0, 1.0, 0.0, length)
    boxes = _make_boxes(seed, cfg, [seg], 20.0 / 60.0, device)
    coords, sd, W = _route_scene("street", [seg], boxes, v, mu, H, seed, cfg, device, chunk_blocks,
                                 near_pred=lambda c: (c[:, 0] >= 0) & (c[:, 0] <= length))
    path_dist = lambda P: torch.sqrt(P[..., 1] ** 2 + (P[..., 2] - CAM_Z) ** 2)
    f, ctr = _street_noise(coords, sd, W, v, mu, seed, cfg, path_dist)
    meta = dict(voxel=v, mu=mu, H=H, length=length, seed=seed, n_boxes=int(boxes[0].shape[0]),
                route=route_polyline([seg]))
    if not outlier:
        return Scene("street", coords, f.float().contiguous(), W.float().contiguous(), lam=0.8, eps=0.01,
                     iters=300, meta=meta)
    f, W = _outliers_and_clumps(coords, f, W, ctr, seed, CONFIG_IDS["street-outlier"])
    return Scene("street-outlier", coords, f.float().contiguous(), W.float().contiguous(), lam=0.5,
                 eps=0.0, iters=500, meta=meta)


def _outliers_and_clumps(coords, f, W, ctr, seed, cfg, frac=0.30, clump=20):
    """Config 3: f ← U[−1,1] on Ω voxels with prob 0.05; then W = 0 in axis-aligned clump³-voxel cubes
    (min corners uniform over the allocated bounding box, stream S_CLUMP, counter = clump index)
    until the clumps cover at least `frac` of the allocated voxels."""
    key_o = rng.stream_key(seed, cfg, rng.S_OUTLIER)
    key_v = rng.stream_key(seed, cfg, rng.S_OUTLIER_VAL)
    hit = (rng.uniform(key_o, ctr) < 0.05) & (W > 0)
    f = torch.where(hit, 2.0 * rng.uniform(key_v, ctr) - 1.0, f)
    gv = global_voxel_coords(coords).view(-1, 3)
    gmin = gv.min(0).values
    gmax = gv.max(0).values
    ext = (gmax - gmin + 1)
    # dense occupancy grid of allocated voxels over the bounding box
    dev = coords.device
    idx = ((gv - gmin) * torch.tensor([1, ext[0], ext[0] * ext[1]], device=dev)).sum(1)
    dense_alloc = torch.zeros(int(ext.prod()), dtype=torch.bool, device=dev)
    dense_alloc[idx] = True
    dense_alloc = dense_alloc.view(int(ext[2]), int(ext[1]), int(ext[0]))
    zero = torch.zeros_like(dense_alloc)
    # only voxels inside clumps count towards the fraction: the street's geometry alone already leaves
    # ~1/3 of the allocated voxels unobserved, which would otherwise satisfy the 30 % before any clump
    total = gv.shape[0]
    count = 0
    key_c = rng.stream_key(seed, cfg, rng.S_CLUMP)
    k = 0
    batch = 256
    while count < frac * total:
        ids = torch.arange(k * 4, (k + batch) * 4, device=dev, dtype=torch.int64).view(batch, 4)
        u = rng.uniform(key_c, ids)
        corner = (u[:, :3] * ext.to(torch.float64)).floor().to(torch.int64).cpu()
        for j in range(batch):
            x0, y0, z0 = (int(c) for c in corner[j])
            sub_a = dense_alloc[z0:z0 + clump, y0:y0 + clump, x0:x0 + clump]
            sub_z = zero[z0:z0 + clump, y0:y0 + clump, x0:x0 + clump]
            new = sub_a & ~sub_z
            count += int(new.sum())
            sub_z |= sub_a
            k += 1
            if count >= frac * total:
                break
    Wz = zero.view(-1)[idx].view_as(W)
    W = torch.where(Wz, torch.zeros_like(W), W)
    return f, W


@dataclass
class RoutePlan:
    """The cheap, global part of a route scene (city configs 4/5): geometry, solver-independent constants
    and the candidate blocks.  Every rank of a sharded run computes the same plan; the expensive per-voxel
    values are generated only for the blocks a rank owns (:func:`route_blocks`)."""
    name: str
    seed: int
    cfg: int
    segs: list          # all canyons (lanes × route segments)
    route_segs: list    # the route itself (first lane)
    boxes: list
    v: float
    mu: float
    H: float
    length: float
    cand: torch.Tensor  # int32 [m, 3] candidate blocks (superset of the allocated blocks)

    @property
    def block_edge(self) -> float:
        return 8.0 * self.v

    @property
    def route(self) -> np.ndarray:
        return route_polyline(self.route_segs)

    def path_dist(self, P):
        best = None
        for s in self.segs:
            sP, lat = s.local(P[..., 0], P[..., 1])
            ds = torch.clamp(torch.maximum(-sP, sP - s.L), min=0.0)
            d = torch.sqrt(ds ** 2 + lat ** 2 + (P[..., 2] - CAM_Z) ** 2)
            best = d if best is None else torch.minimum(best, d)
        return best

    def meta(self) -> dict:
        return dict(voxel=self.v, mu=self.mu, H=self.H, length=self.length, seed=self.seed, route=self.route,
                    segments=[(s.x0, s.y0, s.dx, s.dy, s.L) for s in self.segs])


def city_plan(seed: int = 0, length: float = 1000.0, H: float = 20.0, device="cpu", lanes: int = 1) -> RoutePlan:
    """Geometry and candidate blocks of config 4 (city): staircase polyline from the origin heading +x,
    segments U[100,200] m, 90° turns alternating left/right, truncated to `length` metres; each segment a
    config-2 canyon (20 boxes per 60 m), v = 0.1 m, μ = 0.5 m.  `lanes` > 1 is the city-heavy density
    knob (parallel canyons offset by 40 m)."""
    v, mu = 0.1, 0.5
    cfg = CONFIG_IDS["city"]
    key = rng.stream_key(seed, cfg, rng.S_ROUTE)
    segs, x, y, heading, total, i = [], 0.0, 0.0, 0, 0.0, 0
    while total < length - 1e-9:
        L = 100.0 + 100.0 * float(rng.uniform(key, torch.tensor([i]))[0])
        L = min(L, length - total)
        dx, dy = (1.0, 0.0) if heading == 0 else (0.0, 1.0)
        segs.append(Segment(x, y, dx, dy, L, caps=True))
        x += L * dx
        y += L * dy
        total += L
        heading ^= 1
        i += 1
    lanes_segs = [Segment(s.x0 + 40.0 * k, s.y0 - 40.0 * k, s.dx, s.dy, s.L, True)
                  for k in range(lanes) for s in segs]
    all_segs = lanes_segs if lanes > 1 else segs
    boxes = _make_boxes(seed, cfg, all_segs, 20.0 / 60.0, device)
    cand = _route_candidates(all_segs, boxes, v, mu, H, device, compact=lanes > 1)
    return RoutePlan("city" if lanes == 1 else "city-heavy", seed, cfg, all_segs, segs, boxes, v, mu, H, length, cand)


def route_blocks(plan: RoutePlan, cand: torch.Tensor, chunk_blocks: int = 1024):
    """The allocated blocks among the candidate blocks `cand` of `plan`, with their f and W
    (float32 [m, 512]), in the order of `cand`.  Per-block values do not depend on which other blocks
    are generated, so shards generated separately and concatenated equal the whole scene."""
    coords, sd, W = _route_alloc(cand, plan.segs, plan.boxes, plan.v, plan.mu, plan.H, cand.device, chunk_blocks)
    f, _ = _street_noise(coords, sd, W, plan.v, plan.mu, plan.seed, plan.cfg, plan.path_dist, want_ctr=False)
    return coords, f.float().contiguous(), W.float().contiguous()


def city(seed: int = 0, length: float = 1000.0, H: float = 20.0, device="cpu", chunk_blocks: int = 1024,
         lanes: int = 1) -> Scene:
    """Config 4 (city) on one device: :func:`city_plan` + :func:`route_blocks` over every candidate."""
    plan = city_plan(seed, length, H, device, lanes)
    coords, f, W = route_blocks(plan, plan.cand, chunk_blocks)
    return Scene(plan.name, coords, f, W, lam=0.8, eps=0.01, iters=200, meta=plan.meta())


# ----------------------------------------------------------------------------------------------
# small structured / random instances for tests
# ----------------------------------------------------------------------------------------------

def random_instance(n_blocks: int, seed: int = 0, extent: int = 4, w_density: float = 0.7, w_max: int = 4,
                    f_scale: float = 1.0, device="cpu", lam: float = 0.5, eps: float = 0.0,
                    data_term: int = 0, iters: int = 20) -> Scene:
    """n_blocks distinct random block coords in [−extent, extent)³ (dense enough to share faces),
    f ~ f_scale·N(0,1), W ~ U{1..w_max} with probability w_density else 0."""
    cfg = CONFIG_IDS["test"]
    side = 2 * extent
    total = side ** 3
    assert n_blocks <= total
    key = rng.stream_key(seed, cfg, rng.S_TEST)
    pri = rng.uniform(key, torch.arange(total, dtype=torch.int64) + (1 << 40))
    pick = torch.argsort(pri)[:n_blocks]
    coords = torch.stack([pick % side, (pick // side) % side, pick // (side * side)], 1) - extent
    coords = coords.to(torch.int32).to(device)
    gv = global_voxel_coords(coords)
    ctr = rng.pack_coords(gv[..., 0], gv[..., 1], gv[..., 2]) ^ (seed << 63 >> 63)
    f = f_scale * rng.normal(rng.stream_key(seed, cfg, rng.S_NOISE), rng.stream_key(seed, cfg, rng.S_NOISE2), ctr)
    W = rng.uniform_int(rng.stream_key(seed, cfg, rng.S_W), ctr, 1, w_max).to(torch.float64)
    on = rng.uniform(rng.stream_key(seed, cfg, rng.S_W0), ctr) < w_density
    W = torch.where(on, W, torch.zeros_like(W))
    return Scene(f"random{n_blocks}s{seed}", coords.contiguous(), f.float().contiguous(), W.float().contiguous(),
                 lam=lam, eps=eps, data_term=data_term, iters=iters, meta=dict(seed=seed))


def dense_box(a: int, b: int, c: int, seed: int = 0, origin=(0, 0, 0), w_density: float = 1.0, **kw) -> Scene:
    """Every block of an a×b×c block box allocated (dense-equivalence pin)."""
    coords = _block_grid(origin, (origin[0] + a - 1, origin[1] + b - 1, origin[2] + c - 1), "cpu")
    cfg = CONFIG_IDS["test"]
    gv = global_voxel_coords(coords)
    ctr = rng.pack_coords(gv[..., 0], gv[..., 1], gv[..., 2])
    f = rng.normal(rng.stream_key(seed, cfg, rng.S_NOISE), rng.stream_key(seed, cfg, rng.S_NOISE2), ctr)
    w_max = kw.pop("w_max", 4)
    W = rng.uniform_int(rng.stream_key(seed, cfg, rng.S_W), ctr, 1, w_max).to(torch.float64)
    on = rng.uniform(rng.stream_key(seed, cfg, rng.S_W0), ctr) < w_density
    W = torch.where(on, W, torch.zeros_like(W))
    defaults = dict(lam=0.5, eps=0.0, iters=20)
    defaults.update(kw)
    return Scene(f"dense{a}x{b}x{c}", coords.contiguous(), f.float().contiguous(), W.float().contiguous(),
                 **defaults, meta=dict(seed=seed))


def line_scene(values, W_line, axis: int = 0, n_blocks_along: int = 3, lam: float = 0.1, eps: float = 0.0,
               data_term: int = 0, iters: int = 20000, offset=(0, 0, 0)) -> Scene:
    """1-D embedding (SURVEY §8(c) closed-form pin): Ω = one straight line of voxels along `axis` crossing
    several blocks, W = 0 everywhere else, so the Ω-masked operators reduce exactly to 1-D."""
    values = np.asarray(values, dtype=np.float32)
    n = values.shape[0]
    assert n <= 8 * n_blocks_along
    coords = []
    for k in range(n_blocks_along):
        b = [offset[0], offset[1], offset[2]]
        b[axis] += k
        coords.append(b)
    coords_t = torch.tensor(coords, dtype=torch.int32)
    f = torch.zeros(n_blocks_along, 512)
    W = torch.zeros(n_blocks_along, 512)
    # line at local (3, 5, 2) in the other two axes
    other = {0: (1, 2), 1: (0, 2), 2: (0, 1)}[axis]
    pos = [3, 5, 2]
    for i in range(n):
        loc = list(pos)
        loc[axis] = i % 8
        vi = loc[0] + 8 * loc[1] + 64 * loc[2]
        f[i // 8, vi] = float(values[i])
        W[i // 8, vi] = float(W_line)
    del other
    return Scene("line", coords_t, f.contiguous(), W.contiguous(), lam=lam, eps=eps, iters=iters,
                 data_term=data_term, meta=dict(axis=axis, n=n, pos=pos))


def line_indices(scene: Scene):
    """(block, voxel) index pairs of the 1-D line of :func:`line_scene`, in line order."""
    axis, n, pos = scene.meta["axis"], scene.meta["n"], scene.meta["pos"]
    out = []
    for i in range(n):
        loc = list(pos)
        loc[axis] = i % 8
        out.append((i // 8, loc[0] + 8 * loc[1] + 64 * loc[2]))
    return out


def by_name(name: str, seed: int = 0, device="cpu", **kw) -> Scene:
    if name == "tiny":
        return tiny(seed, False, device)
    if name == "tiny-stress":
        return tiny(seed, True, device)
    if name == "street":
        return street(seed, False, device=device, **kw)
    if name == "street-outlier":
        return street(seed, True, device=device, **kw)
    if name == "city":
        return city(seed, device=device, **kw)
    if name == "city-heavy":
        return city(seed, device=device, lanes=kw.pop("lanes", 13), **kw)
    if name.startswith("city-weak"):
        g = int(name.split(":")[1]) if ":" in name else 1
        return city(seed, length=125.0 * g, device=device, **kw)
    raise KeyError(name)
