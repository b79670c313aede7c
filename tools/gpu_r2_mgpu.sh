set -x
N=${1:-2}
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_multigpu.py -x -q -m gpu > gpurun_out/r2_mgpu_tests_$N.log 2>&1
tail -5 gpurun_out/r2_mgpu_tests_$N.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_weak_1.json 2> gpurun_out/r2_bench_weak_1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2_bench_weak_$N.json 2> gpurun_out/r2_bench_weak_$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus $N --steps 10 --warmup 3 --workload patch27m > gpurun_out/r2_bench_strong_$N.json 2> gpurun_out/r2_bench_strong_$N.err
for f in gpurun_out/r2_bench_weak_1.json gpurun_out/r2_bench_weak_$N.json gpurun_out/r2_bench_strong_$N.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], d['ms_per_step'], d['value'], d['phases_ms_per_step'].get('halo'))"; done
