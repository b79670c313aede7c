set -x
N=${1:-4}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_multigpu.py -x -q -m gpu > gpurun_out/r2_mgpu_tests_$N.log 2>&1
tail -3 gpurun_out/r2_mgpu_tests_$N.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_scale_weak_1.json 2>/dev/null
P=29600
for G in 2 $N; do
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $P bench.py --gpus $G --steps 10 --warmup 3 > gpurun_out/r2_scale_weak_$G.json 2>/dev/null
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port $P bench.py --gpus $G --steps 10 --warmup 3 --workload patch27m > gpurun_out/r2_scale_strong_$G.json 2>/dev/null
done
for f in gpurun_out/r2_scale_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], round(d['ms_per_step'],2), '%.4g'%d['value'], 'halo', d['phases_ms_per_step'].get('halo'))"; done
