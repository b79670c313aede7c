python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu15.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu15.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench15.log 2>&1
tail -3 gpurun_out/pytest_gpu15.log
tail -1 gpurun_out/bench15.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms_per_step'], d['roofline']['frac'])"
