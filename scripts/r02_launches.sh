#!/bin/bash
# launch list of one timed bench step (share of each kernel in the step), then the plain bench line
set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-fusion --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_bench1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ \
  -s 966 -c 322 --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/r02_status.txt
