#!/bin/bash
# Build libmrf.so variants for kernel experiments: scripts/build_variants.sh name "-DFLAG ..." ...
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2006_03512_b200/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  python - "$name" "$flags" <<'PY' &
import sys, os, shlex
sys.path.insert(0, os.getcwd())
from paper_2006_03512_b200 import _build
out = os.path.join(_build.HERE, "variants", f"libmrf_{sys.argv[1]}.so")
_build.LIB_SAVE = _build.LIB
_build.LIB = out
_build.build(force=True, extra=shlex.split(sys.argv[2]))
print("built", out)
PY
done
wait
