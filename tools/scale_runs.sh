# Multi-GPU evidence run (gpurun --gpus 4): bit-identity tests, weak 1/2/4, strong (27M) 1/2/4,
# and the weak 4-GPU run with lazy re-decomposition (splitters every 10 steps).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/pytest_mg.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_w1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --workload patch27m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/strong1.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_w$n.log 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --workload patch27m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/strong$n.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --redecomp-every 10 > gpurun_out/scale_w4_lazy.log 2>&1
tail -2 gpurun_out/pytest_mg.log
for f in scale_w1 strong1 scale_w2 strong2 scale_w4 strong4 scale_w4_lazy; do grep '^{' gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['n_gpus'], d['ms_per_step'], d['value'])"; done
