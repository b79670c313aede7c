set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab7 cur noexp d512
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py tests/test_gpu_parity_extra.py -x -q -m gpu > gpurun_out/r2_ab7_parity.log 2>&1; tail -3 gpurun_out/r2_ab7_parity.log
