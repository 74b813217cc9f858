#!/bin/bash
# ncu captures of k_skew on the non-default workloads (city, street-outlier), freeze on and off, so that
# their bench lines quote a physical roofline (each plain run precedes its ncu run).
set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for C in street-outlier city; do
  python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/plain_$C.log 2>&1 || { echo "$C plain failed"; continue; }
  $NCU -k regex:k_skew -s 30 -c 1 -o gpurun_out/r02_skew_v11_${C}_freeze python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/ncu_${C}_f.log 2>&1
  echo "$C freeze rc=$?"
  $NCU -k regex:k_skew -s 150 -c 1 -o gpurun_out/r02_skew_v11_${C}_nofreeze python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/ncu_${C}_n.log 2>&1
  echo "$C nofreeze rc=$?"
done
