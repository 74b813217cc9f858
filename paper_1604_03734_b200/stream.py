"""Online reconstruction: depth maps arrive in batches, the volume grows and is "continuously regularized"
("The Dense Fusion module merges the depth maps ... into a compressed data structure that is
continuously regularized.  New incoming data can be added at any time").

`Reconstruction.integrate(depth, poses)` continues the fusion on the device (vol_fuse_incremental,
reading F-11), builds the grown volume and carries the regulariser's state (u, ū, p) of the blocks that
already existed over to it (new blocks start from the warm state u = ū = f, p = 0); `regularise(iters)`
then continues the Chambolle–Pock iterations from that state (vol_regularise with resume).  Every step
runs in libvol.so's kernels; the row matching between the old and the grown block list is plumbing
(both lists are sorted by (x, y, z), and the old blocks are a subset of the new ones).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .volume import Volume, fuse


def _keys(xyz: torch.Tensor) -> torch.Tensor:
    o = 1 << 20
    x = xyz.to(torch.int64) + o
    return (x[:, 0] << 42) | (x[:, 1] << 21) | x[:, 2]


class Reconstruction:
    """Fusion + regularisation + extraction of a growing hashed voxel-block volume on one GPU."""

    def __init__(self, intr, voxel: float, mu: float, max_range: float, w_max: float, lam: float, eps: float,
                 tau: float | None = None, sigma: float | None = None, theta: float = 1.0, data_term: int = 0):
        t = float(np.float32(1.0 / math.sqrt(12.0)))
        self.intr = [float(v) for v in (intr.tolist() if hasattr(intr, "tolist") else intr)]
        self.fusion = dict(voxel=voxel, mu=mu, max_range=max_range, w_max=w_max)
        self.solver = dict(lam=lam, eps=eps, tau=t if tau is None else tau, sigma=t if sigma is None else sigma)
        self.theta, self.data_term = theta, data_term
        self.xyz = self.f = self.W = None
        self.vol = None
        self._fresh = True      # the volume holds the warm initial state (no iteration run on it yet)
        self.frames = 0

    @property
    def n_blocks(self) -> int:
        return 0 if self.xyz is None else int(self.xyz.shape[0])

    def integrate(self, depth, poses):
        """Fuse a batch of depth maps [K, H, W] with poses [K, 12] into the (growing) volume."""
        F = self.fusion
        prev = None if self.xyz is None else (self.xyz, self.f, self.W)
        xyz, first, f, W = fuse(depth, poses, self.intr, F["voxel"], F["mu"], F["max_range"], F["w_max"], prev=prev)
        vol = Volume(xyz, f, W)
        if self.vol is not None and not self._fresh:
            u, ub, p = self.vol.state(device=xyz.device)
            rows = torch.searchsorted(_keys(xyz), _keys(self.xyz))     # old rows inside the grown list
            U, UB = f.clone(), f.clone()
            P = torch.zeros(3, xyz.shape[0], 512, device=xyz.device)
            U[rows], UB[rows], P[:, rows] = u, ub, p
            vol.load_state(U, UB, P)
            self._fresh = False
        if self.vol is not None:
            self.vol.close()
        self.vol = vol
        self.xyz, self.f, self.W = xyz, f, W
        self.frames += int(depth.shape[0]) if hasattr(depth, "shape") and len(depth.shape) == 3 else 1
        return self

    def regularise(self, iters: int):
        """Continue the Chambolle–Pock iterations on the current volume (asynchronous)."""
        S = self.solver
        self.vol.regularise(S["lam"], S["eps"], S["tau"], S["sigma"], int(iters), theta=self.theta,
                            data_term=self.data_term, resume=not self._fresh)
        self._fresh = False
        return self

    def u(self):
        return self.vol.u()

    def extract(self, w_min: float = 0.0, field: str = "u"):
        return self.vol.extract(self.fusion["voxel"], w_min=w_min, field=field)
