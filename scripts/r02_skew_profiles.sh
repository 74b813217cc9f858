#!/bin/bash
# ncu captures of the current k_skew on street (freeze on / off), each after the same plain run
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
NCU="ncu --set full --clock-control none --import-source on"
C="python scripts/skew_ab.py --iters 60 --reps 1"
$C > gpurun_out/plain_skew.log 2>&1 && $NCU -k regex:k_skew -s 30 -c 1 -o gpurun_out/r02_skew_v10_freeze $C > gpurun_out/ncu_v10a.log 2>&1
echo "freeze rc=$?" > gpurun_out/r02_v10_status.txt
$NCU -k regex:k_skew -s 150 -c 1 -o gpurun_out/r02_skew_v10_nofreeze $C > gpurun_out/ncu_v10b.log 2>&1
echo "nofreeze rc=$?" >> gpurun_out/r02_v10_status.txt
