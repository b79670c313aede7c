# round-end multi-GPU check of the committed state: NCCL bit-identity cases on 2 GPUs
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -m gpu > gpurun_out/r2_end_pytest_multigpu_2.log 2>&1; tail -2 gpurun_out/r2_end_pytest_multigpu_2.log
