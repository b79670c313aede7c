# round-end check of the committed state: smoke(), the whole -m gpu suite, one bench line
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 120 python tools/dbg_hang.py > gpurun_out/dbg_hang.log 2>&1 || { cat gpurun_out/dbg_hang.log; exit 3; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_end_smoke.log 2>&1; tail -2 gpurun_out/r2_end_smoke.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_end_pytest_gpu.log 2>&1; tail -2 gpurun_out/r2_end_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_end_bench.json 2> gpurun_out/r2_end_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r2_end_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['phases_ms_per_step'])"
