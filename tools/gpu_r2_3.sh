set -x
python -c "import __graft_entry__ as g; g.build()"
# fail fast on a hang (a 27M bench step is ~0.25 s)
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py -x -q -m gpu > gpurun_out/r2_seg_parity.log 2>&1
tail -15 gpurun_out/r2_seg_parity.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_seg_bench.json 2> gpurun_out/r2_seg_bench.err
tail -c 3000 gpurun_out/r2_seg_bench.json; tail -5 gpurun_out/r2_seg_bench.err
