#!/bin/bash
# A/B of k_skew variants on one box: VARIANTS="name:lib.so:ENV=1 ..." scripts/skew_ab_multi.sh [config]
# (lib relative to paper_1604_03734_b200/, ENV optional); bitwise check of u against the first variant.
set -u
C=${1:-street}
for r in 1 2; do
  for v in $VARIANTS; do
    IFS=: read -r name lib envs <<< "$v"
    env ${envs:-HVG_NONE=1} HVG_LIBVOL=$PWD/paper_1604_03734_b200/$lib timeout 600 \
      python scripts/skew_ab.py --config $C --save /tmp/u_$name.npy 2>&1 | grep -v Warn | sed "s/^/$name /"
  done
done
python - <<PY
import numpy as np
names = [v.split(':')[0] for v in "$VARIANTS".split()]
a = np.load(f'/tmp/u_{names[0]}.npy')
for n in names[1:]:
    b = np.load(f'/tmp/u_{n}.npy')
    print(n, 'bitwise equal to', names[0], np.array_equal(a.view(np.uint32), b.view(np.uint32)))
PY
