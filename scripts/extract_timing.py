"""Development timing of vol_extract on the street volume (u after 300 iterations)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_03734_b200 import Volume  # noqa: E402
from synth import street  # noqa: E402

s = street(device="cuda", chunk_blocks=4096)
vol = Volume(s.coords, s.f, s.W)
vol.regularise_scene(s)
v = s.meta["voxel"]
T = vol.extract(v)
print("triangles", T.shape[0], "blocks", s.n_blocks)
out = torch.empty(T.shape[0] + 16, 3, 3, device="cuda")
ts = []
for _ in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    vol.extract(v, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("vol_extract ms", [round(t, 3) for t in ts])
