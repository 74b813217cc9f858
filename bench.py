#!/usr/bin/env python3
"""Benchmark of the hashed-voxel-grid primal-dual TV regulariser on B200 (BASELINE.json metric:
voxel-updates/s and achieved HBM GB/s at 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config street] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: route-axis sharding over NCCL)

A step is one pass of the whole hot path (SURVEY §8(a) rows a-1 … a-8) over the config's synthetic
volume: vol_create (device hash/CSR/neighbour build from block coordinates + f + W), vol_regularise
(init + `iters` fused Chambolle–Pock iterations), vol_energy, vol_read_u.  `value` is
N_alloc·iters·N_gpu / step time with inputs resident in HBM; `e2e` is the same through the same C ABI
from pinned host buffers (host→device copies of coords/f/W and the device→host read of u inside the
timed region).  At N = 1 the workload is config 2 (street, 300 Huber-TV iterations); at N > 1 each
GPU owns one 60 m street segment of a 60·N m street (weak scaling).

--impl reference times the CPU oracle (oracle/, plain C, fp64, one thread) on a bounded sample of
the same workload: each step runs one oracle iteration over the whole volume.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALG_BYTES_PER_VOXEL = 48  # 28 B read (f, W, u, ū, p×3) + 20 B written (u, ū, p×3)
FUSE_OPS_PER_EVAL = 36    # fp32 operations of steps 1-4 + Eq. 1 for one voxel and one frame


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None,
                    help="street (default at N = 1), city (1 km route, strong scaling; default at N > 1), "
                         "city-weak (125 m of route per GPU), city-heavy, street-outlier, tiny")
    ap.add_argument("--iters", type=int, default=None, help="override the config's iteration count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", type=int, default=0, help="0 product (skewed on one GPU), 1 two-kernel baseline, 2 skewed, 3 one-pass fused")
    ap.add_argument("--freeze", type=int, default=1, help="opts.freeze (bit-identical skip of identity updates)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the NCCL sharded runtime even at one rank (tests the N > 1 code path on one GPU)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer"],
                    help="halo transport at N > 1: NCCL send/recv (default) or direct stores into the peers' "
                         "ghost rows over NVLink (CUDA IPC; vol_connect_peer_ipc)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fusion", action="store_true",
                    help="skip the widened rows (SURVEY §8(f) NEXT-2/3/4: fusion, extraction, stereo legs)")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


# ------------------------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()   # wait for the sampler's first line so the whole timed region is covered
        while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0 and self.proc.poll() is None:
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, fl in rows for k, v in enumerate(fl) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_inputs():
    """Per-kernel figures of the committed ncu captures (profiles/ncu_inputs.json, scripts/ncu_inputs.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_inputs.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def issue_peak():
    """Warp-instruction issue peak: 148 SMs x 4 schedulers x 1 warp instruction per clock x the max SM clock."""
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mhz = float(json.load(fh).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return 148 * 4 * mhz * 1e6, f"148 SMs x 4 schedulers x 1 warp-instruction/clk x {mhz:.0f} MHz"


def l2_peak():
    """L2 read bandwidth measured on this pool's B200 (profiles/l2_peak.json, scripts/probes/l2_bw.cu: a 64 MB
    L2-resident buffer streamed by every SM); fallback: the ~6300 B/clk LTS cap of B300_MICROARCH.md."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_peak.json")) as fh:
            d = json.load(fh)
        return float(d["l2_read_gbs"]), "measured L2 read bandwidth (profiles/l2_peak.json)"
    except Exception:
        return 6300.0 * 1965e6 / 1e9, "fallback: 6300 B/clk LTS cap (B300_MICROARCH.md) x 1965 MHz"


def make_scene(cfg: str, world: int, seed: int, device):
    from synth import scenes
    if cfg == "street":
        length = 60.0 * world
        s = scenes.street(seed, length=length, device=device, chunk_blocks=4096)
        if world > 1:
            s.name = f"street-{int(length)}m"
        return s
    if cfg.startswith("city"):
        return scenes.by_name(cfg, seed=seed, device=device, chunk_blocks=4096)
    return scenes.by_name(cfg, seed=seed, device=device)


def partition(scene, world):
    """Owner rank per block: the product's route-axis partition (libvol vol_partition_route) —
    blocks ordered by the arc length of the nearest point of the scene's camera path, cut into contiguous
    ranges of equal block count."""
    import torch

    from paper_1604_03734_b200 import partition_route
    return torch.from_numpy(partition_route(scene.coords.cpu(), scene.meta["route"], 8 * scene.meta["voxel"], world))


# ---------------------------------------------------------------- per-shard generation (configs 4/5)

def route_plan(cfg: str, seed: int, device):
    """Geometry + candidate blocks of a city config (cheap; every rank builds the same plan)."""
    from synth import scenes
    if cfg == "city":
        return scenes.city_plan(seed, length=1000.0, device=device)
    if cfg == "city-heavy":
        return scenes.city_plan(seed, length=1000.0, device=device, lanes=13)
    if cfg.startswith("city-weak"):
        g = int(cfg.split(":")[1])
        return scenes.city_plan(seed, length=125.0 * g, device=device)
    raise KeyError(cfg)


def shard_generate(plan, world: int, rank: int, chunk_blocks: int = 4096):
    """SURVEY §1 L0 `gen(config, seed, shard)`: the allocated blocks (coords, f, W) among this rank's
    candidate blocks — the `world` equal-count arc-length ranges of the candidates (vol_partition_route).
    The per-voxel values come from the counter-based generator, so they do not depend on the sharding."""
    import torch

    from paper_1604_03734_b200 import partition_route
    from synth import scenes
    cpart = torch.from_numpy(partition_route(plan.cand.cpu(), plan.route, plan.block_edge, world)).to(plan.cand.device)
    return scenes.route_blocks(plan, plan.cand[cpart == rank], chunk_blocks)


def shard_assemble(plan, world: int, rank: int, coords_all, coords_r, f_r, W_r, chunk_blocks: int = 4096):
    """Global block list = the ranks' generated blocks in rank order; owner map = the exact equal-count route
    partition of the allocated blocks (the one every sharded test uses); blocks whose owner differs from
    the rank that generated them (a few near each cut) are regenerated by their new owner.  Returns
    coords [n, 3] (all ranks identical), part [n] and this rank's f, W in global order."""
    import numpy as np
    import torch

    from paper_1604_03734_b200 import partition_route
    from synth import scenes
    dev = coords_r.device
    coords = torch.cat([c.to(dev) for c in coords_all], 0).contiguous()
    origin = torch.cat([torch.full((c.shape[0],), q, dtype=torch.int32) for q, c in enumerate(coords_all)])
    part = partition_route(coords.cpu(), plan.route, plan.block_edge, world)
    mine = torch.from_numpy(part == rank)
    have = origin == rank
    f = torch.empty(int(mine.sum()), 512, dtype=torch.float32, device=dev)
    W = torch.empty_like(f)
    pos = torch.cumsum(mine.to(torch.int64), 0) - 1                       # row among my blocks
    own_idx = torch.cumsum(have.to(torch.int64), 0) - 1                   # row in my generated piece
    keep = mine & have
    f[pos[keep].to(dev)] = f_r[own_idx[keep].to(dev)]
    W[pos[keep].to(dev)] = W_r[own_idx[keep].to(dev)]
    need = mine & ~have
    n_moved = int(need.sum())
    if n_moved:
        c2, f2, W2 = scenes.route_blocks(plan, coords[need.to(dev)], chunk_blocks)
        assert torch.equal(c2, coords[need.to(dev)]), "a moved block is no longer allocated"
        f[pos[need].to(dev)] = f2
        W[pos[need].to(dev)] = W2
    return {"coords": coords, "part": np.ascontiguousarray(part), "f": f, "W": W, "moved": n_moved}


def gather_coords(coords_r, world, dev):
    """all_gather of every rank's generated block coordinates (variable counts, padded)."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([coords_r.shape[0]], device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    m = int(max(int(x) for x in ns))
    pad = torch.zeros(m, 3, dtype=torch.int32, device=dev)
    pad[:coords_r.shape[0]] = coords_r
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return [b[:int(k)] for b, k in zip(bufs, ns)]


def alu_peak():
    """Issue-limited ALU peak in lane-operations/s: 148 SMs × 4 SMSPs × 32 lanes × 1 instruction per clock
    × the max SM clock (MEASURED_PEAKS.json sm_max_mhz, else 1965 MHz) — DESIGN.md §11."""
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mhz = float(json.load(fh).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return 148 * 4 * 32 * mhz * 1e6, f"148 SMs x 4 SMSPs x 32 lanes x 1 inst/clk x {mhz:.0f} MHz"


def fusion_leg(args, dev):
    """TSDF fusion of the fusion-street depth maps (61 frames, 1240x376) through vol_fuse, inputs in HBM."""
    import torch

    from paper_1604_03734_b200 import fuse
    from synth.depth import street_depth
    ds = street_depth(seed=args.seed, device=dev)
    intr = ds.intr.cpu().numpy()
    st = {}
    out = fuse(ds.depth, ds.poses, intr, ds.voxel, ds.mu, ds.max_range, ds.w_max, stats=st)
    n = int(out[0].shape[0])
    del out
    call = lambda **kw: fuse(ds.depth, ds.poses, intr, ds.voxel, ds.mu, ds.max_range, ds.w_max, max_blocks=n + 16, **kw)
    for _ in range(3):
        call()
    stream = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    a.record(stream)
    for _ in range(args.steps):
        call()
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / args.steps
    kst = []
    for _ in range(5):
        d = {}
        call(stats=d)
        kst.append(d)
    t_int = statistics.median(d["ms_integrate"] for d in kst)
    t_alloc = statistics.median(d["ms_alloc"] for d in kst)
    evals = st["block_frames"] * 512
    peak, peak_src = alu_peak()
    ach = FUSE_OPS_PER_EVAL * evals / (t_int / 1e3)
    res = {"workload": "fusion-street", "frames": ds.K, "image": [ds.H, ds.Wd], "voxel": ds.voxel, "mu": ds.mu,
           "w_max": ds.w_max, "ms_per_call": ms, "frames_per_s": ds.K / (ms / 1e3),
           "voxel_updates_per_s": st["voxel_updates"] / (ms / 1e3), "blocks": n,
           "stats": {k: st[k] for k in ("pixels_valid", "blocks", "block_frames", "voxel_updates")},
           "kernel_ms": {"k_fuse_alloc": t_alloc, "k_fuse_integrate": t_int},
           "step": "vol_fuse (alloc + compact + radix sort + integrate), depth maps and poses resident in HBM",
           "roofline": {"bound": "alu", "kernel": "k_fuse_integrate", "achieved": ach / 1e12, "peak": peak / 1e12,
                        "unit": "Tops/s", "frac": ach / peak, "peak_source": peak_src,
                        "basis": "algorithmic: 36 fp32 operations per evaluated voxel-frame (DESIGN.md §11) / "
                                 "issue-limited lane-op peak",
                        "alg_ops_per_launch": FUSE_OPS_PER_EVAL * evals, "avg_launch_ms": t_int,
                        "traffic": None}}
    ni = ncu_inputs().get("k_fuse_integrate/fusion-street")
    if ni:
        ip, ip_src = issue_peak()
        iss = ni["warp_instructions"] / (t_int / 1e3)
        res["roofline"].update({"issue": {"achieved": iss / 1e12, "peak": ip / 1e12, "unit": "T warp-instructions/s",
                                          "frac": iss / ip, "peak_source": ip_src,
                                          "warp_instructions_per_launch": ni["warp_instructions"],
                                          "source": ni["source"]},
                                "traffic": ni["dram_bytes"]})
    if not args.no_cpu_baseline:
        import oracle
        k = 4
        D, P = ds.depth[:k].cpu().numpy(), ds.poses[:k].cpu().numpy()
        t0 = time.perf_counter()
        oracle.fuse(D, intr, P, ds.voxel, ds.mu, ds.max_range, ds.w_max)
        dt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": k / dt, "unit": "frames/s", "cores": 1, "kind": "oracle",
                               "sample": f"first {k} of the {ds.K} fusion-street frames, sequential fp32 oracle, "
                                         f"{dt:.1f} s on one host core"}
    return res


def extraction_leg(args, dev, scene, iters, stream):
    """vol_extract of the regularised street u into a device buffer (one ordered pass: count, decoupled
    look-back, emit), inputs in HBM."""
    import torch

    from paper_1604_03734_b200 import Volume
    vol = Volume(scene.coords, scene.f, scene.W, stream=stream)
    vol.regularise(scene.lam, scene.eps, scene.tau, scene.sigma, iters, theta=scene.theta, data_term=scene.data_term,
                   init=scene.init)
    v = scene.meta["voxel"]
    T = vol.extract(v)
    cap = int(T.shape[0]) + 1024
    out = torch.empty(cap, 3, 3, dtype=torch.float32, device=dev)
    for _ in range(3):
        vol.extract(v, out=out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    a.record(stream)
    for _ in range(args.steps):
        T = vol.extract(v, out=out)
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / args.steps
    ntri = int(T.shape[0])
    nvox = scene.n_alloc
    alg = 8 * nvox + 36 * ntri          # read u and W once, write the triangles
    peak, peak_src = load_peaks()
    res = {"workload": scene.name + " (regularised u, " + str(iters) + " iterations)", "field": "u", "w_min": 0.0,
           "triangles": ntri, "cells": nvox, "ms_per_call": ms, "cells_per_s": nvox / (ms / 1e3),
           "triangles_per_s": ntri / (ms / 1e3),
           "step": "vol_extract: inverse permutation + one ordered count/look-back/emit kernel, output in HBM",
           "hbm": {"achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                   "frac": alg / (ms / 1e3) / 1e9 / peak, "alg_bytes_per_call": alg,
                   "note": "algorithmic bytes (read u and W once, write 36 B per triangle); not the bound"}}
    ne = ncu_inputs().get("k_extract/street")
    ip, ip_src = issue_peak()
    if ne and scene.name == "street":
        inst = ne["warp_instructions"]
        iss = inst / (ms / 1e3)
        res["roofline"] = {"bound": "issue", "kernel": "k_extract (single ordered pass)", "achieved": iss / 1e12,
                           "peak": ip / 1e12, "unit": "T warp-instructions/s", "frac": iss / ip, "peak_source": ip_src,
                           "basis": "physical: ncu warp instructions of the pass / CUDA-event call time",
                           "warp_instructions_per_call": inst,
                           "thread_instructions_per_triangle": 32 * inst / max(ntri, 1),
                           "traffic": ne["dram_bytes"], "sources": [ne["source"]]}
    else:
        res["roofline"] = {"bound": "issue", "kernel": "k_extract (single ordered pass)", "achieved": None,
                           "peak": ip / 1e12, "unit": "T warp-instructions/s", "frac": None, "peak_source": ip_src,
                           "traffic": None, "basis": "no ncu capture of this workload"}
    vol.close()
    return res


STEREO_BYTES_PER_PIXEL_ITER = 112   # 16 fields read + 12 written (fp32) per pixel-iteration


def stereo_leg(args, dev):
    """Depth-map estimation (§IV) of 8 street stereo pairs (1240x376, 128 disparities, 10 x 20 iterations)."""
    import torch

    from paper_1604_03734_b200 import stereo
    from synth.stereo import street_pair
    F = 8
    IL, IR, dt = street_pair(seed=args.seed, frames=tuple(range(20, 20 + F)), device=dev)
    kw = dict(n_disp=128, outer=10, inner=20)
    stream = torch.cuda.current_stream(dev)

    def timed(n, **k):
        for _ in range(2):
            stereo.stereo(IL, IR, **k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(stream)
        for _ in range(n):
            out = stereo.stereo(IL, IR, **k)
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b) / n, out

    ms, d = timed(args.steps, **kw)
    ms_half, _ = timed(max(2, args.steps // 2), **dict(kw, inner=10))
    it_ms = (ms - ms_half) / (10 * kw["outer"])            # one k_tgv_iter launch over the batch
    valid = (dt > 1) & (dt < 120)
    err = float((d - dt).abs()[valid].median())
    npx = F * IL.shape[1] * IL.shape[2]
    peak, peak_src = load_peaks()
    ach = STEREO_BYTES_PER_PIXEL_ITER * npx / (it_ms / 1e3) / 1e9
    res = {"workload": f"stereo-street ({F} pairs 1240x376, D=128, 10 x 20 iterations)", "frames": F,
           "ms_per_call": ms, "frames_per_s": F / (ms / 1e3),
           "pixel_iterations_per_s": npx * kw["outer"] * kw["inner"] / (ms / 1e3),
           "median_abs_disparity_error_px": err,
           "step": "vol_stereo: census x2, tensor, WTA init, 200 TGV iterations (k_dual4 + k_primal4 on L2-sized "
                   "chunks of 2 frames), 10 data steps, one CUDA graph",
           "hbm_alg": {"achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_source": peak_src,
                       "alg_bytes_per_iteration": STEREO_BYTES_PER_PIXEL_ITER * npx,
                       "note": "112 algorithmic B per pixel-iteration; the chunked state is L2-resident, so this is "
                               "not a DRAM figure (see roofline)"}}
    nd, npr = (ncu_inputs().get(k) for k in ("k_dual4/stereo-street", "k_primal4/stereo-street"))
    lp, lp_src = l2_peak()
    if nd and npr:
        px_launch = 2 * 1240 * 376   # one chunk of 2 frames per launch
        l2b = (nd["lts_tex_bytes"] + npr["lts_tex_bytes"]) / px_launch
        drb = (nd["dram_bytes"] + npr["dram_bytes"]) / px_launch
        l2a = l2b * npx / (it_ms / 1e3) / 1e9
        res["roofline"] = {"bound": "l2", "kernel": "k_dual4 + k_primal4 (one TGV iteration)", "achieved": l2a,
                           "peak": lp, "unit": "GB/s", "frac": l2a / lp, "peak_source": lp_src,
                           "basis": "physical: ncu lts__t_sectors_srcunit_tex x 32 B (the SMs' L2 traffic) per "
                                    "pixel-iteration x pixels / event time; ncu's DRAM bytes are cold-cache (flushed "
                                    "before each replay), an upper bound for the L2-resident chunks",
                           "avg_launch_ms": it_ms, "l2_bytes_per_pixel_iter": l2b, "dram_bytes_per_pixel_iter": drb,
                           "dram_achieved": drb * npx / (it_ms / 1e3) / 1e9,
                           "traffic": drb * npx, "sources": [nd["source"], npr["source"]]}
    else:
        res["roofline"] = {"bound": "l2", "kernel": "k_dual4 + k_primal4", "achieved": None, "peak": lp, "unit": "GB/s",
                           "frac": None, "peak_source": lp_src, "traffic": None, "basis": "no ncu capture"}
    if not args.no_cpu_baseline:
        import time as _t

        import oracle
        t0 = _t.perf_counter()
        oracle.stereo(IL[0].cpu().numpy(), IR[0].cpu().numpy(), D=128, outer=10, inner=20)
        dt_cpu = _t.perf_counter() - t0
        res["cpu_baseline"] = {"value": 1.0 / dt_cpu, "unit": "frames/s", "cores": 1, "kind": "oracle",
                               "sample": f"one 1240x376 pair, full solve, {dt_cpu:.1f} s on one host core"}
    return res


def pipeline_leg(args, dev):
    """The paper's pipeline (Fig. 2) on the device for the 61-frame street drive: stereo depth maps (§IV) →
    TSDF fusion (§III-A) → regularisation (§III-C, street solver parameters) → surface extraction."""
    import torch

    import paper_1604_03734_b200 as P
    from synth.stereo import street_pair
    from synth.scenes import TAU_DEFAULT
    IL, IR, dt, poses, intr, B = street_pair(seed=args.seed, frames=tuple(range(61)), device=dev, return_rig=True)
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def run():
        ev[0].record(stream)
        d = P.stereo.stereo(IL, IR, n_disp=128)
        z = P.stereo.disparity_to_depth(d, float(intr[0]) * B, d_min=0.5)
        ev[1].record(stream)
        xyz, first, f, W = P.fuse(z, poses, intr, 0.05, 0.3, 25.0, 30.0)
        ev[2].record(stream)
        vol = P.Volume(xyz, f, W, stream=stream)
        ev[3].record(stream)
        vol.regularise(0.8, 0.01, TAU_DEFAULT, TAU_DEFAULT, 300)
        ev[4].record(stream)
        T = vol.extract(0.05)
        ev[5].record(stream)
        torch.cuda.synchronize(dev)
        n = vol.n_local
        vol.close()
        return n, int(T.shape[0])

    run()
    n_blocks, ntri = run()
    names = ["stereo+depth", "fuse", "create", "regularise", "extract"]
    ms = {k: ev[i].elapsed_time(ev[i + 1]) for i, k in enumerate(names)}
    total = ev[0].elapsed_time(ev[5])
    return {"workload": "street drive: 61 stereo pairs 1240x376 -> depth -> fuse (v = 5 cm) -> 300 Huber-TV "
                        "iterations -> extraction", "frames": 61, "blocks": n_blocks, "voxels": 512 * n_blocks,
            "triangles": ntri, "ms": ms, "ms_total": total, "frames_per_s": 61 / (total / 1e3)}


# ------------------------------------------------------------------------------ CPU oracle timing

def platform_cpu() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def time_oracle(scene, iters: int, omp: bool = False, precision: str = "f64", nbr=None):
    """Wall time of `iters` oracle iterations over the whole scene — the -O3 -march=native timing build of
    the oracle (bitwise the parity build), one thread or OpenMP over all host threads."""
    import oracle
    coords, f, W = scene.numpy()
    if nbr is None:
        nbr = oracle.neighbours(coords)
    t0 = time.perf_counter()
    oracle.regularise(coords, f, W, scene.lam, scene.eps, scene.tau, scene.sigma, iters, theta=scene.theta,
                      data_term=scene.data_term, init=scene.init, precision=precision, nbr=nbr, omp=omp, native=True)
    return time.perf_counter() - t0


def cpu_baselines(scene):
    """SURVEY §8(d) CPU baselines on the box's host cores, each a bounded sample (~10 s) of the same volume:
    the fp64 oracle on one thread (`cpu_baseline`), on all host threads (`cpu_baseline_omp`), and the fp32
    oracle on one thread (`cpu_baseline_f32`)."""
    import oracle
    sc = scene.to("cpu")
    nbr = oracle.neighbours(sc.coords)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    host = {"cpu_model": platform_cpu(), "nproc": os.cpu_count(), "build": "gcc -O3 -march=native -ffp-contract=off"}
    out = {}
    for key, omp, prec in (("cpu_baseline", False, "f64"), ("cpu_baseline_omp", True, "f64"),
                           ("cpu_baseline_f32", False, "f32")):
        k = 1
        t = time_oracle(sc, k, omp=omp, precision=prec, nbr=nbr)
        while t < 5.0:   # grow the sample to ~10 s (the first short runs include thread start-up)
            k = max(2 * k, int(k * 10.0 / max(t, 1e-3)))
            t = time_oracle(sc, k, omp=omp, precision=prec, nbr=nbr)
        cores = threads if omp else 1
        out[key] = dict({"value": sc.n_alloc * k / t, "unit": "voxel-updates/s", "cores": cores,
                         "kind": "oracle" + (" (OpenMP)" if omp else ""), "precision": prec,
                         "sample": f"{k} {prec} oracle iteration(s) over the whole {scene.name} volume "
                                   f"({sc.n_alloc} voxels), {t:.1f} s on {cores} host thread(s)"}, **host)
    return out


def reference_arm(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg = args.config or ("street" if world == 1 else "city")   # the same workload as our arm
    if cfg == "city-weak":
        cfg = f"city-weak:{world}"
    if cfg.startswith("city"):
        from synth.scenes import Scene
        plan = route_plan(cfg, args.seed, dev)
        c, f, W = shard_generate(plan, 1, 0)
        scene = Scene(cfg, c.cpu(), f.cpu(), W.cpu(), lam=0.8, eps=0.01, iters=200, meta=plan.meta())
    else:
        scene = make_scene(cfg, 1, args.seed, dev).to("cpu")
    n_alloc = scene.n_alloc
    # 8 iterations per step: the oracle call's fixed cost (array conversion, its own table build, ~1 s on the
    # street) would otherwise dominate a 1-iteration sample and understate its throughput ~4x; the untimed
    # warm-up steps run one iteration each (they only page in the library and the arrays)
    per_step_iters = 8 if n_alloc < 50_000_000 else 2   # city: 2 (the whole run stays within a few minutes)
    for _ in range(args.warmup):
        time_oracle(scene, 1)
    times = [time_oracle(scene, per_step_iters) for _ in range(args.steps)]
    t = sum(times) / len(times)
    val = n_alloc * per_step_iters / t
    sample = f"{per_step_iters} oracle iteration(s) over the whole {scene.name} volume ({n_alloc} voxels) per step"
    line = {"impl": "reference", "metric": "voxel-updates/s", "value": val, "unit": "voxel-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t,
            "higher_is_better": True, "scaling": "strong" if cfg in ("city", "city-heavy") else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": scene.name, "n_alloc": n_alloc, "blocks": scene.n_blocks,
                                            "iters_per_step": per_step_iters},
            "cpu_baseline": {"value": val, "unit": "voxel-updates/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "voxel-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ our arm

def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    from paper_1604_03734_b200 import Volume
    from paper_1604_03734_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    sharded = world > 1 or args.sharded
    if sharded:
        if "MASTER_ADDR" not in os.environ:   # plain `python bench.py --sharded`: a one-rank group
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ.get("MASTER_PORT", "29531"),
                              RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    # workload: config 2 (street) on one GPU; BASELINE configs[4] (config 5) at N > 1 — the 1 km city route
    # at a fixed size (strong scaling), or `--config city-weak` (125 m of route per GPU, weak scaling)
    cfg = args.config or ("street" if world == 1 else "city")
    if cfg == "city-weak":
        cfg = f"city-weak:{world}"
    gen_s = None
    if cfg.startswith("city"):
        # per-shard generation: each rank generates only the blocks of its arc range
        from synth.scenes import Scene
        t_gen = time.perf_counter()
        plan = route_plan(cfg, args.seed, dev)
        coords_r, f_r, W_r = shard_generate(plan, world, rank)
        coords_all = gather_coords(coords_r, world, dev) if world > 1 else [coords_r]
        sh = shard_assemble(plan, world, rank, coords_all, coords_r, f_r, W_r)
        del coords_r, f_r, W_r, coords_all
        gen_s = time.perf_counter() - t_gen
        scene = Scene(cfg if not cfg.startswith("city-weak") else f"city-weak ({125 * world} m)", sh["coords"],
                      sh["f"], sh["W"], lam=0.8, eps=0.01, iters=200, meta=plan.meta())
        coords = sh["coords"]
        f_loc, W_loc = sh["f"], sh["W"]
        part = torch.from_numpy(sh["part"]) if sharded else None
        n_moved = sh["moved"]
    else:
        scene = make_scene(cfg, world, args.seed, dev)
        coords = scene.coords.contiguous()
        if sharded:
            part = partition(scene, world)
            mine = (part == rank).nonzero().squeeze(1).to(dev)
            f_loc, W_loc = scene.f[mine].contiguous(), scene.W[mine].contiguous()
        else:
            part = None
            f_loc, W_loc = scene.f, scene.W
        n_moved = 0
    iters = scene.iters if args.iters is None else args.iters
    n_local_vox = f_loc.shape[0] * 512
    scaling = "strong" if cfg in ("city", "city-heavy") else "weak"
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if sharded:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    kw = dict(part=part, group=group) if sharded else {}
    u_out = torch.empty(f_loc.shape[0], 512, device=dev)
    ev_a = torch.cuda.Event(enable_timing=True)
    ev_b = torch.cuda.Event(enable_timing=True)
    iter_ms = []

    shard_t = []
    host_us = []

    def step(c, f, W, out, record, freeze=bool(args.freeze), rec=None, exchange=True):
        vol = Volume(c, f, W, stream=stream, **kw)
        if sharded and args.transport == "peer" and world > 1:
            vol.connect_peers(group)
        vol.regularise(scene.lam, scene.eps, scene.tau, scene.sigma, 0, theta=scene.theta,
                       data_term=scene.data_term, init=scene.init, kernel=args.kernel)
        ev_a.record(stream)
        th = time.perf_counter()
        vol.regularise(scene.lam, scene.eps, scene.tau, scene.sigma, iters, theta=scene.theta,
                       data_term=scene.data_term, resume=True, kernel=args.kernel, freeze=freeze, exchange=exchange)
        host_us.append(1e6 * (time.perf_counter() - th) / iters)   # host issue time (asynchronous call)
        ev_b.record(stream)
        if sharded and record and rec is None:
            shard_t.append(vol.shard_timing())   # last iteration: interior A, halo chain, boundary B
        E = vol.energy(scene.lam, scene.eps, scene.data_term)
        vol.read_u(out)
        if record:
            ev_b.synchronize()
            (iter_ms if rec is None else rec).append(ev_a.elapsed_time(ev_b) / iters)
        vol.close()
        return E

    # warm-up (also validates the run end to end)
    for _ in range(max(3, args.warmup)):
        E = step(coords, f_loc, W_loc, u_out, False)
    barrier()
    launches0 = N.lib().vol_total_launches()
    clocks = ClockSampler(local_rank)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0.record(stream)
    for _ in range(args.steps):
        E = step(coords, f_loc, W_loc, u_out, True)
    t1.record(stream)
    barrier()
    clk = clocks.stop()
    launches = (N.lib().vol_total_launches() - launches0) // args.steps
    ms = t0.elapsed_time(t1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    it_t = torch.tensor([statistics.median(iter_ms)], device=dev)
    if sharded:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(it_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    it_ms = float(it_t.item())
    n_alloc_total = scene.n_alloc
    value = n_alloc_total * iters / (ms / 1e3)
    n_omega_t = torch.tensor([int((W_loc > 0).sum())], device=dev, dtype=torch.int64)
    if sharded:
        dist.all_reduce(n_omega_t)
    n_omega_total = int(n_omega_t.item())

    # transparency: the same step with opts.freeze = 0 (every Ω voxel recomputed and rewritten)
    nf = None
    if args.freeze and args.kernel != 1:
        nf_ms = []
        step(coords, f_loc, W_loc, u_out, False, freeze=False)
        barrier()
        t0.record(stream)
        nsteps = max(2, args.steps // 2)
        for _ in range(nsteps):
            step(coords, f_loc, W_loc, u_out, True, freeze=False, rec=nf_ms)
        t1.record(stream)
        barrier()
        nfm = torch.tensor([t0.elapsed_time(t1) / nsteps, statistics.median(nf_ms)], device=dev)
        if sharded:
            dist.all_reduce(nfm, op=dist.ReduceOp.MAX)
        nf = {"value": scene.n_alloc * iters / (float(nfm[0]) / 1e3), "ms_per_step": float(nfm[0]),
              "avg_launch_ms": float(nfm[1]), "steps": nsteps}

    # SURVEY 8(d) multi-GPU: exposed halo = T_iter(exchange on) - T_iter(exchange replaced by a no-op with the
    # same partition), and the per-stream durations of the last iteration (interior launch A, halo chain on
    # the communication stream, boundary launch B), max over ranks
    halo = None
    if sharded:
        off_ms = []
        step(coords, f_loc, W_loc, u_out, False, exchange=False)
        barrier()
        for _ in range(max(2, args.steps // 2)):
            step(coords, f_loc, W_loc, u_out, True, rec=off_ms, exchange=False)
        barrier()
        tt = torch.tensor([statistics.median(off_ms)] + [statistics.median(x[i] for x in shard_t) for i in range(3)],
                          device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        hu = torch.tensor([statistics.median(host_us)], device=dev)
        dist.all_reduce(hu, op=dist.ReduceOp.MAX)
        halo = {"exposed_us_per_iter": 1e3 * (it_ms - float(tt[0])), "iter_ms_exchange_off": float(tt[0]),
                "host_issue_us_per_iter": float(hu.item()), "gpu_us_per_iter": 1e3 * it_ms,
                "interior_ms": float(tt[1]), "exchange_chain_ms": float(tt[2]), "boundary_ms": float(tt[3]),
                "transport": ("direct stores into the peers' ghost rows by the boundary launch (CUDA IPC over NVLink), "
                              "per-source arrival counters, inside the CUDA graph of the skewed loop"
                              if args.transport == "peer" and world > 1 else
                              "NCCL send/recv per peer on the comm stream (fork/join inside the CUDA graph of the "
                              "skewed loop), pack/unpack kernels"),
                "note": "max over ranks; chain overlaps the interior launch"}

    # end to end from pinned host buffers through the same API
    e2e = None
    if not args.no_e2e:
        hc = coords.cpu().pin_memory()
        hf = f_loc.cpu().pin_memory()
        Wc = W_loc.cpu()
        # W is an observation count (Eq. 1): exact small integers go over PCIe as 8-bit counts
        # (vol_create_w8, bit-identical to the fp32 call), a quarter of the weight bytes
        w_u8 = bool(((Wc == Wc.round()) & (Wc >= 0) & (Wc <= 255)).all())
        hW = (Wc.to(torch.uint8) if w_u8 else Wc).pin_memory()
        hu = torch.empty(u_out.shape, dtype=torch.float32).pin_memory()
        hus = [hu, torch.empty_like(hu).pin_memory()]

        def e2e_pipelined(nsteps):
            ss = [stream, torch.cuda.Stream(dev)]
            start, end, join = (torch.cuda.Event(enable_timing=True) for _ in range(3))

            def make(i):
                v = Volume(hc, hf, hW, stream=ss[i % 2], **kw)
                v.regularise(scene.lam, scene.eps, scene.tau, scene.sigma, iters, theta=scene.theta,
                             data_term=scene.data_term, init=scene.init, kernel=args.kernel, freeze=bool(args.freeze))
                return v
            barrier()
            start.record(ss[0])
            ss[1].wait_event(start)
            v = make(0)
            for i in range(nsteps):
                nxt = make(i + 1) if i + 1 < nsteps else None
                v.energy(scene.lam, scene.eps, scene.data_term)
                v.read_u(hus[i % 2])
                v.close()
                v = nxt
            join.record(ss[1])
            ss[0].wait_event(join)
            end.record(ss[0])
            barrier()
            return start.elapsed_time(end) / nsteps

        for _ in range(2):
            step(hc, hf, hW, hu, False)
        if not sharded:
            e2e_pipelined(2)   # warm-up of the pipelined form
        barrier()
        t0.record(stream)
        for _ in range(args.steps):
            step(hc, hf, hW, hu, False)
        t1.record(stream)
        barrier()
        ems = torch.tensor([t0.elapsed_time(t1) / args.steps], device=dev)
        if sharded:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        ems = float(ems.item())
        h2d = hc.numel() * 4 + hf.numel() * 4 + hW.numel() * hW.element_size()
        d2h = hu.numel() * 4 + 5 * 8
        e2e = {"value": n_alloc_total * iters / (ems / 1e3), "unit": "voxel-updates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": ems,
               "w_host_dtype": "u8" if w_u8 else "f32", "mode": "serial: one step at a time on one stream"}
        if not sharded:
            # The same steps pipelined over two streams, the way a caller processing a stream of volumes uses
            # the API: step i+1's host-to-device copies and volume build are issued while step i iterates,
            # and step i's energy and u read-back while step i+1 iterates.  Every step still copies its
            # inputs from pinned host memory and reads its result back inside the timed region.
            pms = e2e_pipelined(args.steps)
            e2e["serial"] = {"value": e2e["value"], "ms_per_step": ems}
            e2e.update({"value": n_alloc_total * iters / (pms / 1e3), "ms_per_step": pms,
                        "mode": "pipelined: two streams, step i+1's H2D + build and step i's energy + D2H "
                                "overlap the iterations"})

    fusion = None
    if not args.no_fusion and world == 1:
        fusion = fusion_leg(args, dev)
    extraction = None
    if not args.no_fusion and world == 1:
        extraction = extraction_leg(args, dev, scene, iters, stream)
    stereo_res = None
    pipeline = None
    if not args.no_fusion and world == 1:
        stereo_res = stereo_leg(args, dev)
        pipeline = pipeline_leg(args, dev)

    if rank != 0:
        dist.destroy_process_group()
        return 0

    peak, peak_src = load_peaks()
    kname = {0: "k_skew", 1: "k_dual+k_primal", 2: "k_skew", 3: "k_fused"}[args.kernel]
    n_omega_local = int((W_loc > 0).sum())
    ncu = ncu_inputs()

    def hbm_roofline(ms_launch, freeze):
        """Roofline position of the iteration kernel: physical DRAM bytes per launch (the committed ncu capture
        of this kernel on this workload) over the CUDA-event launch time; SURVEY §8(d)'s algorithmic 48 B per
        allocated voxel-iteration beside it (alg_*).  Without a capture of this workload the algorithmic
        figure is the position (basis says which)."""
        alg_bytes = ALG_BYTES_PER_VOXEL * n_local_vox
        alg = alg_bytes / (ms_launch / 1e3) / 1e9
        ni = ncu.get(f"{kname}/{scene.name}/{'freeze' if freeze else 'nofreeze'}") if not sharded else None
        r = {"bound": "hbm", "kernel": kname, "peak": peak, "unit": "GB/s", "peak_source": peak_src,
             "avg_launch_ms": ms_launch, "alg_bytes_per_launch": alg_bytes, "alg_achieved": alg,
             "alg_frac": alg / peak, "alg_frac_of_8TBps": alg / 8000.0}
        if ni:
            tr = ni["dram_bytes"]
            ach = tr / (ms_launch / 1e3) / 1e9
            r.update({"basis": "physical: ncu dram__bytes_read + dram__bytes_write per launch / CUDA-event launch time",
                      "achieved": ach, "frac": ach / peak, "frac_of_8TBps": ach / 8000.0, "traffic": tr,
                      "traffic_source": ni["source"], "bytes_per_alloc_voxel": tr / n_local_vox,
                      "bytes_per_omega_voxel": tr / max(n_omega_local, 1),
                      "l2_bytes_per_launch": ni.get("lts_bytes"), "warp_instructions_per_launch": ni.get("warp_instructions")})
        else:
            r.update({"basis": "algorithmic: 48 B per allocated voxel-iteration (no ncu capture of this workload)",
                      "achieved": alg, "frac": alg / peak, "frac_of_8TBps": alg / 8000.0, "traffic": None})
        return r

    roofline = hbm_roofline(it_ms, bool(args.freeze))
    if nf:
        nf["roofline"] = hbm_roofline(nf["avg_launch_ms"], False)
    cpus = cpu_baselines(scene) if (not args.no_cpu_baseline and world == 1) else {}
    line = {
        "metric": "voxel-updates/s", "value": value, "unit": "voxel-updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": scene.name, "n_alloc": n_alloc_total, "n_omega": n_omega_total,
                   "blocks": scene.n_blocks, "iters": iters, "lambda": scene.lam, "eps": scene.eps,
                   "data_term": "L1" if scene.data_term == 0 else "L2",
                   "step": "vol_create + vol_regularise(init + iters) + vol_energy + vol_read_u",
                   "l2": f"inputs larger than L2 ({n_alloc_total * 48 / 1e9:.2f} GB of state vs 126 MB L2)",
                   "parallelism": f"route-axis shards x{world}" if sharded else "single GPU",
                   "partition": ("vol_partition_route: arc length of the nearest camera-path point, equal "
                                 "block counts" if sharded else None),
                   "generation": ({"per_shard": True, "seconds": gen_s, "blocks_moved_at_rebalance": n_moved}
                                  if gen_s is not None else None),
                   "energy": {"primal": E[0], "dual": E[1]}},
        "omega_updates_per_s": n_omega_total * iters / (ms / 1e3),
        "roofline": roofline, "cpu_baseline": cpus.get("cpu_baseline"), "cpu_baseline_omp": cpus.get("cpu_baseline_omp"),
        "cpu_baseline_f32": cpus.get("cpu_baseline_f32"), "e2e": e2e, "halo": halo, "gpu_launches": int(launches),
        "freeze": bool(args.freeze), "no_freeze": nf,
        "clocks": clk, "fusion": fusion, "extraction": extraction, "stereo": stereo_res, "pipeline": pipeline,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
