"""Per-block statistics of a scene at the start of a call (development): how many blocks have no voxel whose
primal step can change (every voxel Ω̄ or frozen by the opts.freeze bound of store.cu::k_freeze_mask)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from synth import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "street"
s = scenes.by_name(name, device="cuda", chunk_blocks=4096)
f, W = s.f, s.W
tau, lam = np.float32(s.tau), np.float32(s.lam)
t = (torch.tensor(tau * lam, device="cuda") * W)
bound = float(tau) * (4.7320508 * 1.0000019) + f.abs() * 2.3841858e-7
frozen = (W > 0) & (t >= bound) & (s.data_term == 0)
static = frozen | (W == 0)
blk_static = static.all(dim=1)
omega = (W > 0)
print(f"{name}: blocks {s.n_blocks}, voxels Ω {float(omega.float().mean()):.3f}, frozen {float(frozen.float().mean()):.3f} "
      f"of all ({float(frozen.float().sum() / omega.float().sum()):.3f} of Ω); blocks with no updatable voxel "
      f"{float(blk_static.float().mean()):.3f}; warps (128-voxel quarters) with none "
      f"{float(static.view(-1, 4, 128).all(dim=2).float().mean()):.3f}")
