python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu3.log
for ub in 2 0; do SPH_UNIT_BITS=$ub timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3_ub$ub.log 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_density_c|k_iad_c|k_search" -s 12 -c 4 -o gpurun_out/src3_25m -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_src3.log 2>&1
tail -3 gpurun_out/pytest_gpu3.log
for ub in 2 0; do tail -1 gpurun_out/bench3_ub$ub.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($ub, d['ms_per_step'], d['phases_ms_per_step'])"; done
tail -2 gpurun_out/ncu_src3.log
