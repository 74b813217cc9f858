"""How often two consecutive store rows (Morton order of the blocks) are face neighbours — the share of CTA
pairs of a 2-CTA cluster that could exchange a face through distributed shared memory.
    python scripts/pair_stats.py [config ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import scenes  # noqa: E402


def spread(v):
    x = v & 0x1FFFFF
    out = np.zeros_like(x)
    for b in range(21):
        out |= ((x >> b) & 1) << (3 * b)
    return out


for cfg in sys.argv[1:] or ["street"]:
    s = scenes.by_name(cfg, device="cuda" if torch.cuda.is_available() else "cpu", chunk_blocks=4096)
    c = s.coords.cpu().numpy().astype(np.int64)
    d = c - c.min(0)
    key = spread(d[:, 0]) | (spread(d[:, 1]) << 1) | (spread(d[:, 2]) << 2)
    cs = c[np.argsort(key, kind="stable")]
    n = len(cs)
    for off in (0, 1):
        a = cs[off::2]
        b = cs[off + 1::2]
        m = min(len(a), len(b))
        diff = b[:m] - a[:m]
        fr = {ax: float(np.mean(np.all(diff == v, axis=1))) for ax, v in (("x", (1, 0, 0)), ("y", (0, 1, 0)), ("z", (0, 0, 1)))}
        print(cfg, "blocks", n, "pair offset", off, "pairs that are +x/+y/+z neighbours:", fr, flush=True)
