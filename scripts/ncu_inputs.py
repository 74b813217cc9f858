"""Per-kernel ncu figures that bench.py's roofline objects quote (DRAM and L2 bytes, warp instructions per
launch), read from committed `ncu --set full` captures, written to profiles/ncu_inputs.json.

    python scripts/ncu_inputs.py KEY=REPORT:KERNEL_REGEX[:note] ...

Each KEY gets the per-launch mean over the report's captured launches of the matching kernel:
dram read / write bytes, lts (L2) bytes, warp instructions, duration (serialised, cold-cache replay:
a share, not a bench time) and the report path.  Keys already in the file and not named are kept."""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_inputs.json")
METRICS = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
           "lts__t_sectors.sum": "lts_sectors", "lts__t_sectors_srcunit_tex.sum": "lts_tex_sectors", "smsp__inst_executed.sum": "warp_instructions",
           "gpu__time_duration.sum": "duration_us", "launch__grid_size": "grid"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3, "second": 1e6, "sector": 1, "inst": 1, "": 1}


def read(report, kernel_re):
    out = subprocess.check_output(["ncu", "-i", report, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(out.splitlines()))
    H, U = rows[0], rows[1]
    kcol = H.index("Kernel Name")
    acc, n = {}, 0
    for D in rows[2:]:
        if not re.search(kernel_re, D[kcol]):
            continue
        n += 1
        for m, name in METRICS.items():
            if m in H:
                i = H.index(m)
                v = float(D[i].replace(",", "")) * SCALE.get(U[i], 1)
                acc[name] = acc.get(name, 0.0) + v
    if not n:
        raise SystemExit(f"{report}: no launch of {kernel_re}")
    r = {k: v / n for k, v in acc.items()}
    r["dram_bytes"] = r.get("dram_read_bytes", 0) + r.get("dram_write_bytes", 0)
    r["lts_bytes"] = 32 * r.pop("lts_sectors", 0)               # all L2 tag traffic (incl. cross-die fabric)
    r["lts_tex_bytes"] = 32 * r.pop("lts_tex_sectors", 0)       # requests from the SMs (L1 / TMA)
    r["launches_captured"] = n
    r["source"] = os.path.relpath(report, ROOT)
    return r


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for arg in sys.argv[1:]:
        key, spec = arg.split("=", 1)
        parts = spec.split(":")
        rep, kre = parts[0], parts[1]
        d = read(rep, kre)
        if len(parts) > 2:
            d["note"] = ":".join(parts[2:])
        data[key] = d
        print(key, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items()})
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
