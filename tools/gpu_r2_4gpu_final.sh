# 4-GPU box: the whole -m gpu suite (multi-GPU NCCL cases included) and the f1
# validation on 1 / 2 / 4 GPUs
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_pytest_gpu_4gpubox.log 2>&1; tail -3 gpurun_out/r2_pytest_gpu_4gpubox.log
bash tools/gpu_r2_validate_mgpu.sh
