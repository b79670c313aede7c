mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_mg.log 2>&1; echo rc=$? >> gpurun_out/pytest_mg.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_w1.log 2>&1
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_w$n.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29580 bench.py --gpus 4 --workload patch27m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/strong4.log 2>&1
