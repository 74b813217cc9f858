"""Development timing of vol_extract on the street volume (u after 300 iterations).
HVG_LIBVOL selects the library (A/B); --save writes a hash of the triangle soup for a bitwise comparison."""
import argparse
import hashlib
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_03734_b200 import Volume  # noqa: E402
from synth import street  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tag", default="")
args = ap.parse_args()
s = street(device="cuda", chunk_blocks=4096)
vol = Volume(s.coords, s.f, s.W)
vol.regularise_scene(s)
v = s.meta["voxel"]
T = vol.extract(v)
h = hashlib.sha1(T.cpu().numpy().tobytes()).hexdigest()[:12]
out = torch.empty(T.shape[0] + 16, 3, 3, device="cuda")
ts = []
for _ in range(args.reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    T2 = vol.extract(v, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
h2 = hashlib.sha1(T2.cpu().numpy().tobytes()).hexdigest()[:12]
ts.sort()
print(args.tag, "triangles", T.shape[0], "hash", h, h2, "vol_extract ms median", round(ts[len(ts) // 2], 3),
      "min", round(ts[0], 3))
