set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py -x -q -m gpu > gpurun_out/r2_ab4_parity_cur.log 2>&1; tail -2 gpurun_out/r2_ab4_parity_cur.log
SPH_LIB=$PWD/variants/p2_384.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2_ab4_parity_p2.log 2>&1; tail -2 gpurun_out/r2_ab4_parity_p2.log
bash tools/ab_bench.sh ab4 cur p2_384 p2_256 casmem
