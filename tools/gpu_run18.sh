SPH_LIB=$PWD/_v_ring/libsph.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_gpu18.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu18.log
SPH_LIB=$PWD/_v_ring/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench18_ring.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench18_main.log 2>&1
tail -3 gpurun_out/pytest_gpu18.log
for v in ring main; do tail -1 gpurun_out/bench18_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
