python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log
tail -3 gpurun_out/pytest_final.log; tail -2 gpurun_out/smoke_final.log
