set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab15 m2 m3 m2 m3
SPH_LIB=$PWD/variants/m3.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_ab15_parity.log 2>&1; tail -2 gpurun_out/r2_ab15_parity.log
