# Evrard 1M: search-cell factor sweep around the default (variable h)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
for cf in 0.85 0.9 0.95 1.0 1.05 1.1 1.15; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload evrard --cell-factor $cf > gpurun_out/r2_evrard_sweep_cf$cf.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r2_evrard_sweep_cf$cf.json').read().strip().splitlines()[-1]); p=d['phases_ms_per_step']; print('evrard cf $cf', round(d['ms_per_step'],2), '%.3g'%d['value'], 'nbr', p['neighbors'], 'dens', p['density'], 'iad', p['iad'], 'mom', p['momentum'])"
done
