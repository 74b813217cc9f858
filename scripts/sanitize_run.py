"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): the fused and two-kernel
paths, state I/O, energy and a 2-shard loopback group, on the tiny sphere and a random instance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1604_03734_b200 import Volume, connect_group, group_energy, regularise_group  # noqa: E402
from synth import random_instance, tiny  # noqa: E402


def main():
    s = tiny()
    v = Volume(s.coords.cuda(), s.f.cuda(), s.W.cuda())
    v.regularise(s.lam, 0.01, s.tau, s.sigma, 4)
    v.regularise(s.lam, 0.0, s.tau, s.sigma, 3, kernel=1, data_term=1)
    u, ub, p = v.state()
    v.load_state(u, ub, p)
    print("energy", v.energy(s.lam, 0.0, 0))
    r = random_instance(120, seed=3, extent=4)
    c = r.coords
    part = (c[:, 0] >= 0).to(torch.int32)
    vols = []
    for k in range(2):
        mine = (part == k).nonzero().squeeze(1)
        vols.append(Volume(c, r.f[mine], r.W[mine], part=part, loopback=(k, 2)))
    connect_group(vols)
    regularise_group(vols, 0.5, 0.01, r.tau, r.sigma, 3)
    print("group energy", group_energy(vols, 0.5, 0.01))
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
