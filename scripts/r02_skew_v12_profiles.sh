#!/bin/bash
# ncu captures of the product k_skew (v12) on street, street-outlier and city, freeze on and off (each plain
# run precedes its ncu run); then python scripts/ncu_inputs.py refreshes profiles/ncu_inputs.json.
set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
for C in street street-outlier city; do
  python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/plain_$C.log 2>&1 || { echo "$C plain failed"; continue; }
  $NCU -k regex:k_skew -s 30 -c 1 -o gpurun_out/r02_skew_v12_${C}_freeze python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/ncu_${C}_f.log 2>&1
  echo "$C freeze rc=$?"
  $NCU -k regex:k_skew -s 150 -c 1 -o gpurun_out/r02_skew_v12_${C}_nofreeze python scripts/skew_ab.py --config $C --iters 60 --reps 1 > gpurun_out/ncu_${C}_n.log 2>&1
  echo "$C nofreeze rc=$?"
done
