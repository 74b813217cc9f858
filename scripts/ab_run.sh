#!/bin/bash
# A/B of prebuilt libvol variants (paper_1604_03734_b200/libvol_*.so): bitwise u after 300 street iterations
# (scripts/skew_ab.py, freeze on/off timing) and the bench's k_skew launch time (scripts/ab_libs.sh).
# usage (GPU box): LIBS="libvol_head.so libvol_x.so" scripts/ab_run.sh
set -u
mkdir -p gpurun_out
for L in $LIBS; do
  HVG_LIBVOL=$PWD/paper_1604_03734_b200/$L timeout 900 python scripts/skew_ab.py --config ${CONFIG:-street} --reps 5 --save /tmp/u_$L.npy >> gpurun_out/ab_skew.log 2>&1
  echo "$L rc=$?" >> gpurun_out/ab_skew.log
done
python - >> gpurun_out/ab_skew.log 2>&1 <<'PY'
import os, numpy as np
libs = os.environ["LIBS"].split()
a = np.load(f"/tmp/u_{libs[0]}.npy")
for L in libs[1:]:
    b = np.load(f"/tmp/u_{L}.npy")
    print(L, "bitwise equal to", libs[0], np.array_equal(a.view(np.uint32), b.view(np.uint32)))
PY
ROUNDS=${ROUNDS:-2} scripts/ab_libs.sh > gpurun_out/ab_libs_summary.txt 2>&1
