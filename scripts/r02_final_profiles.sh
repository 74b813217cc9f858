#!/bin/bash
# Final-state evidence: ncu --set full of the product k_skew on the street (freeze on), and the launch list
# of one timed bench step — each ncu run after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
S="python scripts/skew_ab.py --config street --iters 60 --reps 1"
$S > gpurun_out/plain_street.log 2>&1 && $NCU -k regex:k_skew -s 30 -c 1 -o gpurun_out/r02_skew_final_street_freeze $S \
  > gpurun_out/ncu_street_f.log 2>&1
echo "skew rc=$?" >> gpurun_out/final_status.txt
B="python bench.py --steps 1 --warmup 3 --no-fusion --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_bench1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ \
  -s 966 -c 322 --csv --log-file gpurun_out/r02_launches_final.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/final_status.txt
