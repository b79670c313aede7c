set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab8 nopf cur grponly rowonly
bash tools/ab_bench.sh ab8b nopf cur
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py -x -q -m gpu > gpurun_out/r2_ab8_parity.log 2>&1; tail -3 gpurun_out/r2_ab8_parity.log
