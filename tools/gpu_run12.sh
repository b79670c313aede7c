python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu12.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu12.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench12.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/l12.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu12.log
tail -1 gpurun_out/bench12.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms_per_step'])"
