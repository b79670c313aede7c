SPH_LIB=$PWD/_v_rec/libsph.so python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu9.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu9.log
SPH_LIB=$PWD/_v_rec/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9_rec.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9_main.log 2>&1
tail -3 gpurun_out/pytest_gpu9.log
for v in rec main; do tail -1 gpurun_out/bench9_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
