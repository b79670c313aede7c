# final capture of the round-2 kernels (1 GPU): bench line, reference arm, Evrard / 1M,
# ncu launch list and one --set full launch per pair kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python bench.py > gpurun_out/r2z_bench_27M.json 2> gpurun_out/r2z_bench_27M.err; tail -c 300 gpurun_out/r2z_bench_27M.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2z_bench_reference.json 2> gpurun_out/r2z_bench_reference.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload evrard > gpurun_out/r2z_evrard.json 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload patch1m > gpurun_out/r2z_patch1m.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_search|k_expand_rows|k_density_c|k_iad_c" -s 20 -c 5 -o gpurun_out/r2z_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_ncu_full.log 2>&1
for f in gpurun_out/r2z_bench_27M.json gpurun_out/r2z_evrard.json gpurun_out/r2z_patch1m.json gpurun_out/r2z_bench_reference.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d.get('phases_ms_per_step', {}); print('$f', d['n_gpus'], round(d['ms_per_step'],2), '%.4g'%d['value'], p)"; done
