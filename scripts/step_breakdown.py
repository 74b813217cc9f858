"""Wall-clock breakdown of one bench step (create / init / iterations / energy / read-back) on street."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1604_03734_b200 import Volume  # noqa: E402
from synth import scenes  # noqa: E402


def main():
    sharded = "--sharded" in sys.argv
    kw = {}
    if sharded:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29541", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    s = scenes.street(0, device="cuda", chunk_blocks=4096)
    if sharded:
        kw = dict(part=torch.zeros(s.n_blocks, dtype=torch.int32), group=dist.group.WORLD)
    out = torch.empty(s.n_blocks, 512, device="cuda")
    for rep in range(4):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        v = Volume(s.coords, s.f, s.W, **kw)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        v.regularise(s.lam, s.eps, s.tau, s.sigma, 0)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        v.regularise(s.lam, s.eps, s.tau, s.sigma, 300, resume=True)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        v.energy(s.lam, s.eps)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        v.read_u(out)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        v.close()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        names = ["create", "init", "iters", "energy", "read_u", "close"]
        print(rep, " ".join(f"{n}={1e3 * (b - a):.3f}ms" for n, a, b in zip(names, t, t[1:])), flush=True)


if __name__ == "__main__":
    main()
