#!/bin/bash
# GPU-box check used during development: parity tests, bench, two-kernel baseline, ncu launch list and
# one full ncu capture of the fused kernel (all outputs under gpurun_out/).
# usage: scripts/gpu_check.sh [tests] [bench] [k1] [ncu]
set -u
mkdir -p gpurun_out
: > gpurun_out/status.txt
for what in "$@"; do
  case $what in
    tests) timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt ;;
    smoke) timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt ;;
    bench) timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt ;;
    variants)
      for vv in 0 1; do HVG_FUSED_VARIANT=$vv timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v$vv.log 2>&1; echo "v$vv=$?" >> gpurun_out/status.txt; done ;;
    k1) timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --kernel 1 > gpurun_out/bench_k1.log 2>&1; echo "k1=$?" >> gpurun_out/status.txt ;;
    ncu)
      P="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
      $P > gpurun_out/plain.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 2000 --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
      echo "launch=$?" >> gpurun_out/status.txt
      ncu --set full --clock-control none --import-source on -k regex:"k_skew|k_fused" -s 100 -c 2 -o gpurun_out/prof_fused $P > gpurun_out/ncu_full.log 2>&1
      echo "full=$?" >> gpurun_out/status.txt ;;
  esac
done
# experiment: alternative builds selected with HVG_LIBVOL (names after 'libs')
if [ "${LIBS:-}" != "" ]; then
  for L in $LIBS; do HVG_LIBVOL=$PWD/paper_1604_03734_b200/$L timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$L.log 2>&1; echo "$L=$?" >> gpurun_out/status.txt; done
fi
