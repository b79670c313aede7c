SPH_LIB=$PWD/_v_pf/libsph.so python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu14.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu14.log
SPH_LIB=$PWD/_v_pf/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_pf.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14_main.log 2>&1
tail -3 gpurun_out/pytest_gpu14.log
for v in pf main; do tail -1 gpurun_out/bench14_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
