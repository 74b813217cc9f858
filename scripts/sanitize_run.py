"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): the fused and two-kernel
paths, state I/O, energy and a 2-shard loopback group, on the tiny sphere and a random instance; then
the widened rows on small inputs: vol_fuse, vol_extract, vol_stereo (two-kernel and fused iteration)."""
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
    # the direct-store transport on 3 loopback shards (peer stores, signal / wait kernels)
    part3 = ((c[:, 0] + 4) * 3 // 8).clamp(0, 2).to(torch.int32)
    vp = []
    for k in range(3):
        mine = (part3 == k).nonzero().squeeze(1)
        vp.append(Volume(c, r.f[mine], r.W[mine], part=part3, loopback=(k, 3)))
    connect_group(vp, transport="peer")
    regularise_group(vp, 0.5, 0.01, r.tau, r.sigma, 6)
    print("peer transport", [x.transport for x in vp])
    # widened rows: fusion, extraction, stereo
    from paper_1604_03734_b200 import fuse, stereo
    from synth.depth import sphere_depth
    from synth.stereo import plane_pair
    ds = sphere_depth(n_cams=3, H=40, Wd=56)
    xyz, first, f, W = fuse(ds.depth.cuda(), ds.poses.cuda(), ds.intr.numpy(), ds.voxel, ds.mu, ds.max_range,
                            ds.w_max, stats={})
    fv = Volume(xyz, f, W)
    fv.regularise(1.0, 0.0, s.tau, s.sigma, 3)
    print("triangles", fv.extract(ds.voxel).shape[0], fv.extract(ds.voxel, field="f", w_min=2.0).shape[0])
    IL, IR, _ = plane_pair(24, 72, 0.03, 0.01, 5.0)
    d = stereo.stereo(IL, IR, n_disp=16, outer=2, inner=3)
    os.environ["HVG_STEREO_FUSED"] = "1"
    d2 = stereo.stereo(IL, IR, n_disp=16, outer=2, inner=3)
    del os.environ["HVG_STEREO_FUSED"]
    print("stereo equal", bool(torch.equal(d, d2)), float(stereo.disparity_to_depth(d, 388.8, 0.5).mean()))
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
