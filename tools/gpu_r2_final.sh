# final evidence of the round-2 kernels: bench (N=1 default), reference arm, Evrard /
# 1M workloads, ncu launch list and one --set full launch per pair kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; tail -c 600 gpurun_out/r2_bench_final.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; tail -c 400 gpurun_out/r2_bench_reference.json
for cf in 1.0 1.25 1.5; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload evrard --cell-factor $cf > gpurun_out/r2_evrard_cf$cf.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r2_evrard_cf$cf.json').read().strip().splitlines()[-1]); print('evrard cf $cf', d['ms_per_step'], d['value'], d['phases_ms_per_step'])"
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload patch1m > gpurun_out/r2_patch1m.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r2_patch1m.json').read().strip().splitlines()[-1]); print('patch1m', d['ms_per_step'], d['value'], d['phases_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_launch_final.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_search|k_expand_rows|k_density_c|k_iad_c" -s 20 -c 5 -o gpurun_out/r2_full_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_full_final.log 2>&1
ls -la gpurun_out | tail -8
