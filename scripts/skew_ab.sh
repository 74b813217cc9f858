#!/bin/bash
# usage (on the GPU box): scripts/skew_ab.sh [config]   — TMA vs legacy k_skew, bitwise check + timing
set -u
C=${1:-street}
python -c "import __graft_entry__ as g; g.build()" || exit 1
for r in 1 2; do
  timeout 600 python scripts/skew_ab.py --config $C --save /tmp/u_tma.npy
  HVG_SKEW_LEGACY=1 timeout 600 python scripts/skew_ab.py --config $C --save /tmp/u_leg.npy
done
python -c "import numpy as np; a=np.load('/tmp/u_tma.npy'); b=np.load('/tmp/u_leg.npy'); print('bitwise equal:', np.array_equal(a.view(np.uint32), b.view(np.uint32)))"
