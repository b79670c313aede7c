set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 900 python -m pytest tests/test_gpu_parity_extra.py -x -q -m gpu -k "wide_rows or rows_grow" > gpurun_out/r2_widetest.log 2>&1; tail -30 gpurun_out/r2_widetest.log
