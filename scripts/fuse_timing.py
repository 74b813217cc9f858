"""Development timing of vol_fuse on the fusion-street depth maps (device inputs, CUDA events)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1604_03734_b200 import fuse  # noqa: E402
from synth.depth import street_depth  # noqa: E402

t0 = time.time()
ds = street_depth(device="cuda")
torch.cuda.synchronize()
print(f"render {time.time() - t0:.1f} s, depth {tuple(ds.depth.shape)}")
intr = ds.intr.cpu().numpy()
st = {}
out = fuse(ds.depth, ds.poses, intr, ds.voxel, ds.mu, ds.max_range, ds.w_max, stats=st)
print("stats", st)
n = out[0].shape[0]
print("blocks", n, "observed voxels", int((out[3] > 0).sum()), "max W", float(out[3].max()))
for cap in (n, None):
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fuse(ds.depth, ds.poses, intr, ds.voxel, ds.mu, ds.max_range, ds.w_max, max_blocks=n + 16)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print("vol_fuse ms", [round(t, 3) for t in ts])
    break
st2 = {}
fuse(ds.depth, ds.poses, intr, ds.voxel, ds.mu, ds.max_range, ds.w_max, stats=st2)
print("warm stats", {k: round(v, 4) for k, v in st2.items() if k.startswith("ms_")})
