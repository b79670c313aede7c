set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
bash tools/ab_bench.sh ab9 cur poly9 cur poly9
SPH_LIB=$PWD/variants/poly9.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_extra.py tests/test_gpu_fullsize.py -q -m gpu > gpurun_out/r2_ab9_parity_poly9.log 2>&1; tail -3 gpurun_out/r2_ab9_parity_poly9.log
