import os, sys, time
sys.path.insert(0, '.')
import torch
from paper_1604_03734_b200 import Volume
from paper_1604_03734_b200 import _native as N
from synth import scenes
s = scenes.street(0, device="cuda", chunk_blocks=4096)
W8 = s.W.to(torch.uint8)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v = Volume(s.coords, s.f, W8)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    v.regularise(s.lam, s.eps, s.tau, s.sigma, 0)
    t3 = time.perf_counter()
    v.regularise(s.lam, s.eps, s.tau, s.sigma, 300, resume=True)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    v.close()
    t6 = time.perf_counter()
    print(f"rep {rep}: Volume() {1e3*(t1-t0):.3f} ms, init call {1e3*(t3-t2):.3f}, iters call (host) {1e3*(t4-t3):.3f}, iters+sync {1e3*(t5-t3):.3f}, close {1e3*(t6-t5):.3f}", file=sys.stderr, flush=True)
