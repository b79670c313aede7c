SPH_LIB=$PWD/_v_uc2/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench25_uc2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench25_main.log 2>&1
SPH_LIB=$PWD/_v_uc2/libsph.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench25_uc2b.log 2>&1
for v in uc2 main uc2b; do tail -1 gpurun_out/bench25_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['phases_ms_per_step'])"; done
