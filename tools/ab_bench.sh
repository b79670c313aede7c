#!/bin/bash
# usage: bash tools/ab_bench.sh OUTPREFIX variant1 variant2 ...  (variants/<v>.so, SPH_LIB)
cd "$(dirname "$0")/.."
out=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "$@"; do
  SPH_LIB=$PWD/variants/$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${out}_$v.json 2> gpurun_out/${out}_$v.err
  python - "$v" "gpurun_out/${out}_$v.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    p = d["phases_ms_per_step"]
    print(f"{sys.argv[1]:12s} step {d['ms_per_step']:8.2f}  nbr {p.get('neighbors',0):6.2f} dens {p.get('density',0):6.2f} iad {p.get('iad',0):6.2f} mom {p.get('momentum',0):7.2f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
