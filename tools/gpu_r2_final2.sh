# final round-2 evidence on a 4-GPU box: 1-GPU bench + reference arm + ncu of the final
# kernels, 1/2/4-GPU scaling, and the f1 validation decomposed over 2 and 4 GPUs
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python bench.py > gpurun_out/r2f_bench_27M.json 2> gpurun_out/r2f_bench_27M.err; tail -c 300 gpurun_out/r2f_bench_27M.json
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload evrard > gpurun_out/r2f_evrard.json 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload patch1m > gpurun_out/r2f_patch1m.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_search|k_expand_rows|k_density_c|k_iad_c" -s 20 -c 5 -o gpurun_out/r2f_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_full.log 2>&1
P=29650
for G in 2 4; do
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $P bench.py --gpus $G --steps 10 --warmup 3 > gpurun_out/r2f_scale_weak_$G.json 2>/dev/null
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $P bench.py --gpus $G --steps 10 --warmup 3 --workload patch27m > gpurun_out/r2f_scale_strong_$G.json 2>/dev/null
done
for f in gpurun_out/r2f_bench_27M.json gpurun_out/r2f_evrard.json gpurun_out/r2f_patch1m.json gpurun_out/r2f_scale_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d['phases_ms_per_step']; print('$f', d['n_gpus'], round(d['ms_per_step'],2), '%.4g'%d['value'], 'mom', p.get('momentum'), 'halo', p.get('halo'))"; done
bash tools/gpu_r2_validate_mgpu.sh
