set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_local_multirank.py -x -q -m gpu --durations=10 > gpurun_out/r2_local_mr.log 2>&1
tail -30 gpurun_out/r2_local_mr.log
timeout 1800 python -m pytest tests -q -m gpu --durations=15 --ignore=tests/test_local_multirank.py > gpurun_out/r2_gpu_all.log 2>&1
tail -30 gpurun_out/r2_gpu_all.log
