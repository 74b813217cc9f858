"""Development timing of vol_energy on the street volume (after 300 iterations); HVG_LIBVOL for A/B."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_03734_b200 import Volume  # noqa: E402
from synth import street  # noqa: E402

s = street(device="cuda", chunk_blocks=4096)
vol = Volume(s.coords, s.f, s.W)
vol.regularise_scene(s)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    E = vol.energy(s.lam, s.eps, s.data_term)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(sys.argv[1:] or "", "energy", E, "ms median", round(ts[5], 4), "min", round(ts[0], 4))
