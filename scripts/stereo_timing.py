"""Development timing of vol_stereo on a batch of street stereo pairs (1240x376, D=128, 10 x 20)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_03734_b200 import stereo  # noqa: E402
from synth.stereo import street_pair  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8
IL, IR, dt = street_pair(frames=tuple(range(20, 20 + F)), device="cuda")
d = stereo.stereo(IL, IR, n_disp=128)
ts = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    stereo.stereo(IL, IR, n_disp=128)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
valid = (dt > 1) & (dt < 120)
print(f"F={F} vol_stereo ms {[round(t, 2) for t in ts]}  median |d - d_true| {float((d - dt).abs()[valid].median()):.3f}")
