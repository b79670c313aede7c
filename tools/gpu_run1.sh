set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_density_c" -s 6 -c 2 -o gpurun_out/src_25m -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_src.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log; tail -3 gpurun_out/ncu_src.log
