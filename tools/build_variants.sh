#!/bin/bash
# A/B builds of kernel variants (same sources, -D macros): variants/<name>.so
# usage: bash tools/build_variants.sh name1 "flags1" name2 "flags2" ...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  SPH_NVCC_EXTRA="$2" python -c "
from paper_2005_02656_b200 import _build
_build.build(force=True, out='variants/$1.so')" 2>&1 | grep -iE "error" ; echo "built variants/$1.so ($2)"
  shift 2
done
