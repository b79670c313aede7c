set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab6 cur seprec
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest_gpu_ab6.log 2>&1; tail -3 gpurun_out/r2_pytest_gpu_ab6.log
