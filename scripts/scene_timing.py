"""Development: generation time of the city / city-heavy synthetic scenes on the GPU at route prefixes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from synth import scenes  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 13
for L in [float(x) for x in (sys.argv[2:] or ["60", "125"])]:
    torch.cuda.synchronize()
    t = time.time()
    s = scenes.city(0, length=L, device="cuda", chunk_blocks=4096, lanes=lanes)
    torch.cuda.synchronize()
    print(f"lanes={lanes} length={L} blocks={s.n_blocks} voxels={s.n_alloc} {time.time() - t:.1f} s "
          f"peak_mem={torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
