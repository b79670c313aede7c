python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu2.log
for ub in 2 1 0; do SPH_UNIT_BITS=$ub timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ub$ub.log 2>&1; done
tail -3 gpurun_out/pytest_gpu2.log
for ub in 2 1 0; do tail -1 gpurun_out/bench_ub$ub.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($ub, d['ms_per_step'], d['phases_ms_per_step'])"; done
