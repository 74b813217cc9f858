#!/bin/bash
# Round-2 ncu captures (run on the GPU box; each plain run precedes its ncu run, as B200_PROFILING.md asks).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
NCU="ncu --set full --clock-control none --import-source on"
run() {   # name, ncu args, command...
  local name=$1 nargs=$2; shift 2
  "$@" > gpurun_out/plain_$name.log 2>&1 && $NCU $nargs -o gpurun_out/r02_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/r02_status.txt
}
run skew_freeze "-k regex:k_skew -s 30 -c 1" python scripts/skew_ab.py --iters 60 --reps 1
run skew_nofreeze "-k regex:k_skew -s 150 -c 1" python scripts/skew_ab.py --iters 60 --reps 1
run extract "-k regex:k_extract -s 6 -c 2" python scripts/extract_timing.py
run fuse "-k regex:k_fuse_integrate -s 2 -c 1" python scripts/fuse_timing.py
run stereo "-k regex:k_dual4|k_primal4 -s 200 -c 2" python scripts/stereo_timing.py
B="python bench.py --steps 1 --warmup 3 --no-fusion --no-e2e --no-cpu-baseline"
# launch list of one timed step (each step issues ~310 launches; skip the 3 warm-up steps)
$B > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ \
  -s 940 -c 320 --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/r02_status.txt
