set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab11 base cur base cur
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r2_ab11_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2_ab11_pytest_gpu.log
