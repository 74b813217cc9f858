"""SURVEY §8(d) CPU baseline table (run once on the GPU box's host): the oracle's -O3
-march=native timing build over whole volumes for the configs' full iteration counts — fp64 and fp32 on one
thread, fp64 on all host threads; the city for 5 iterations, extrapolated (stated as such)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
from synth import scenes  # noqa: E402

rows = []
threads = len(os.sched_getaffinity(0))
for name, extrap in (("tiny", None), ("street", None), ("street-outlier", None), ("city", 5)):
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    if name == "city":
        plan = bench.route_plan("city", 0, dev)
        c, f, W = bench.shard_generate(plan, 1, 0)
        s = scenes.Scene("city", c.cpu(), f.cpu(), W.cpu(), lam=0.8, eps=0.01, iters=200, meta=plan.meta())
    else:
        s = scenes.by_name(name, device=dev, **({"chunk_blocks": 4096} if name != "tiny" else {})).to("cpu")
    nbr = oracle.neighbours(s.coords)
    for prec, omp in (("f64", False), ("f32", False), ("f64", True)):
        it = extrap or s.iters
        t = bench.time_oracle(s, it, omp=omp, precision=prec, nbr=nbr)
        r = {"config": name, "n_alloc": s.n_alloc, "iters": s.iters, "timed_iters": it, "precision": prec,
             "threads": threads if omp else 1, "seconds": t * (s.iters / it),
             "voxel_updates_per_s": s.n_alloc * it / t, "extrapolated": bool(extrap)}
        rows.append(r)
        print(json.dumps(r), flush=True)
print(json.dumps({"cpu_model": bench.platform_cpu(), "nproc": os.cpu_count(), "threads": threads,
                  "build": "gcc -O3 -march=native -ffp-contract=off (oracle.build_native)"}), flush=True)
