#!/bin/bash
# A/B of alternative libvol builds (HVG_LIBVOL) on the street bench: fused kernel only, freeze on and off.
# usage: LIBS="lib_a.so lib_b.so" ROUNDS=2 scripts/ab_libs.sh   (outputs under gpurun_out/ab_*.log)
set -u
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
  for L in $LIBS; do
    for fr in 1 0; do
      HVG_LIBVOL=$PWD/paper_1604_03734_b200/$L timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e \
        --no-cpu-baseline --no-fusion --freeze $fr ${BENCH_ARGS:-} > gpurun_out/ab_${L}_f${fr}_r$r.log 2>&1
      echo "$L f$fr r$r rc=$?" >> gpurun_out/status.txt
    done
  done
done
python - <<'PY'
import glob, json, re
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    ls = [l for l in open(f) if l.startswith('{')]
    if not ls: print(f, 'no json'); continue
    d = json.loads(ls[-1]); r = d['roofline']
    print(f"{f:50s} launch_ms={r['avg_launch_ms']:.4f} frac={r['frac']:.3f} ms/step={d['ms_per_step']:.2f} sm={d['clocks']['sm_mhz']}")
PY
