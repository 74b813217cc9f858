"""Summaries of gpurun_out artefacts: bench JSON lines, ncu raw metrics, SASS hot spots, launch list."""
import collections
import csv
import json
import subprocess
import sys


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{path}: iter_ms={r['avg_launch_ms']:.4f} alg={r['achieved']:.0f} GB/s frac={r['frac']:.3f} "
          f"value={d['value']:.4g} ms/step={d['ms_per_step']:.2f} e2e={d['e2e'] and round(d['e2e']['value'] / 1e9, 2)}e9 "
          f"clocks={d['clocks']} launches={d['gpu_launches']}")


def raw(rep, idx=0):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(out.splitlines()))
    H, U, D = rows[0], rows[1], rows[2 + idx]
    print(f"  [{idx}] {D[H.index('Kernel Name')][:80]}")
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.per_cycle_active", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]
    vals = {}
    for w in want:
        if w in H:
            i = H.index(w)
            vals[w] = (D[i], U[i])
            print(f"  {w:60s} {D[i]:>14s} {U[i]}")
    st = []
    for i, h in enumerate(H):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(D[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    return vals


def sass(rep, top=20, idx=0):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                                   "--launch-skip", str(idx), "--launch-count", "1"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(out.splitlines()))
    H = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(H) and r[0] != "Address":
            data.append(r)
    si, ie, ss = H.index("Source"), H.index("Instructions Executed"), H.index("Warp Stall Sampling (All Samples)")
    ti = sum(int(r[ie]) for r in data)
    ts = sum(int(r[ss]) for r in data)
    print(f"  warp instructions {ti}, stall samples {ts}")
    op, ops = collections.Counter(), collections.Counter()
    for r in data:
        t = r[si].strip().split()
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += int(r[ie])
        ops[o] += int(r[ss])
    print("  ", ", ".join(f"{o}:{c / ti * 100:.1f}%/{ops[o] / ts * 100:.1f}%" for o, c in op.most_common(16)))
    for r in sorted(data, key=lambda r: -int(r[ss]))[:top]:
        print(f"   {r[ss]:>6} {r[ie]:>9} {r[0][-5:]} {r[si].strip()[:90]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[hdr]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
        agg[r[ki].split("(")[0]].append(v)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:45s} n={len(v):5d} total={sum(v):10.1f}us mean={sum(v) / len(v):8.2f}us share={sum(v) / tot:.3f}")


if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a.endswith(".log"):
            bench(a)
        elif ".ncu-rep" in a:   # report[@launch index]
            rep, _, i = a.partition("@")
            raw(rep, int(i or 0))
            sass(rep, idx=int(i or 0))
        elif a.endswith(".csv"):
            launches(a)
