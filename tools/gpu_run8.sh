python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu8.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_main.log 2>&1
SPH_LIB=$PWD/_v_ts32/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8_prev.log 2>&1
tail -3 gpurun_out/pytest_gpu8.log
for v in main prev; do tail -1 gpurun_out/bench8_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
