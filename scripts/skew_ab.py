"""A/B of k_skew forms on the street volume (one process per form: HVG_SKEW_LEGACY is read once).

    python scripts/skew_ab.py [--iters 300] [--reps 5] [--config street] [--save u.npy]

Prints ms per iteration (CUDA events around vol_regularise, median of reps, freeze on and off) and
optionally saves u for a bitwise comparison between forms."""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--config", default="street")
    ap.add_argument("--save", default=None)
    a = ap.parse_args()
    cache = f"/tmp/scene_{a.config}.pt"
    if os.path.exists(cache):
        d = torch.load(cache)
    else:
        from synth import scenes
        if a.config.startswith("street-len:"):   # a shorter street (L2-residency experiments)
            s = scenes.street(0, length=float(a.config.split(":")[1]), device="cuda", chunk_blocks=4096)
        else:
            s = scenes.by_name(a.config, device="cuda", chunk_blocks=4096)
        d = dict(coords=s.coords.cpu(), f=s.f.cpu(), W=s.W.cpu(), p=s.params())
        torch.save(d, cache)
    from paper_1604_03734_b200 import Volume
    p = d["p"]
    c, f, W = d["coords"].cuda(), d["f"].cuda(), d["W"].cuda()
    vol = Volume(c, f, W)
    st = torch.cuda.current_stream()
    out = {}
    for frz in (True, False):
        ts = []
        for r in range(a.reps + 1):
            vol.regularise(p["lam"], p["eps"], p["tau"], p["sigma"], 0, theta=p["theta"], data_term=p["data_term"])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            vol.regularise(p["lam"], p["eps"], p["tau"], p["sigma"], a.iters, theta=p["theta"],
                           data_term=p["data_term"], resume=True, freeze=frz)
            e1.record(st)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1) / a.iters)
        out[frz] = statistics.median(ts)
    u = vol.u().cpu().numpy()
    if a.save:
        np.save(a.save, u)
    form = "legacy" if os.environ.get("HVG_SKEW_LEGACY") else "tma"
    print(f"{form}: {a.config} n_blocks={c.shape[0]} ms/iter freeze={out[True]:.4f} nofreeze={out[False]:.4f} "
          f"u_hash={hash(u.tobytes()) & 0xffffffff:08x}", flush=True)


if __name__ == "__main__":
    main()
