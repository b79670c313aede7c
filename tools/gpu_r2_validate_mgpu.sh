# f1 validation (square patch 100^3 to t = 0.5 s) on 1, 2 and 4 GPUs: the decomposed runs
# must reproduce the 1-GPU history (bit-identical decomposition)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/validate_square_patch.py --n 100 --out gpurun_out/r2_val_mgpu1_100.json > gpurun_out/r2_val_mgpu1_100.log 2>&1
for G in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2971$G \
    tools/validate_square_patch.py --side 100 --out gpurun_out/r2_val_mgpu${G}_100.json > gpurun_out/r2_val_mgpu${G}_100.log 2>&1
done
python - <<'PY'
import json
for g in (1, 2, 4):
    try:
        d = json.load(open(f"gpurun_out/r2_val_mgpu{g}_100.json"))
        print(g, d["gpus"], d["steps"], repr(d["t"]), repr(d["Lz_end"]), "%.4f%%" % (100 * d["rel_to_paper"]),
              "E drift %.3e" % d["E_drift_rel_after_startup"], "wall %.1f s" % d["wall_s"])
    except Exception as e:
        print(g, "FAILED", e)
PY
