#!/bin/bash
# Build libvol.so of git revision REV into paper_1604_03734_b200/NAME (A/B against the working tree).
# usage: scripts/build_rev.sh REV NAME [DEFINE ...]
set -eu
REV=$1; NAME=$2; shift 2
T=$(mktemp -d)
git archive "$REV" paper_1604_03734_b200 include | tar -x -C "$T"
(cd "$T" && python - "$@" <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1604_03734_b200 import build as B
B.build(force=True, defines=sys.argv[1:])
PY
)
cp "$T/paper_1604_03734_b200/libvol.so" "paper_1604_03734_b200/$NAME"
rm -rf "$T"
echo "built $REV -> paper_1604_03734_b200/$NAME"
