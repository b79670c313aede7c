set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab14 ring3 d4 d4i4 ring3 d4i4
SPH_LIB=$PWD/variants/d4i4.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_ab14_parity.log 2>&1; tail -2 gpurun_out/r2_ab14_parity.log
