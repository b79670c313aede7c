SPH_LIB=$PWD/_v_s4/libsph.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_gpu20.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu20.log
SPH_LIB=$PWD/_v_s4/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench20_s4.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench20_main.log 2>&1
tail -3 gpurun_out/pytest_gpu20.log
for v in s4 main; do tail -1 gpurun_out/bench20_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
