set -x
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests/test_gpu_parity_extra.py -x -q -m gpu --durations=20 > gpurun_out/r2_extra.log 2>&1
tail -30 gpurun_out/r2_extra.log
