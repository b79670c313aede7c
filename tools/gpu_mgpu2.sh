python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu2.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_mgpu2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w2.log 2>&1
tail -3 gpurun_out/pytest_mgpu2.log; tail -1 gpurun_out/bench_w2.log | cut -c1-400
