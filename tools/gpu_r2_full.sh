set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python -m pytest tests/test_local_multirank.py -x -q -m gpu > gpurun_out/r2_local_mr.log 2>&1
tail -5 gpurun_out/r2_local_mr.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 --ignore=tests/test_local_multirank.py > gpurun_out/r2_gpu_all.log 2>&1
tail -25 gpurun_out/r2_gpu_all.log
