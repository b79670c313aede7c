set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab12 base exp1wave base exp1wave
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_ab12_parity.log 2>&1; tail -2 gpurun_out/r2_ab12_parity.log
