# f1 validation decomposed over 4 GPUs, and the late-time sensitivity check on 1 GPU
# (positions scaled by 1 + 1e-15 / 1e-14: the same run up to the last bits)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29744 \
  tools/validate_square_patch.py --side 100 --out gpurun_out/r2_val_mgpu4_100.json > gpurun_out/r2_val_mgpu4_100.log 2>&1
timeout 900 python tools/validate_square_patch.py --side 100 --out gpurun_out/r2_val_mgpu1_100.json > gpurun_out/r2_val_mgpu1_100.log 2>&1
for e in 1e-15 1e-14; do
  timeout 900 python tools/validate_square_patch.py --side 100 --perturb $e --out gpurun_out/r2_val_perturb_$e.json > gpurun_out/r2_val_perturb_$e.log 2>&1
done
python - <<'PY'
import json
for f in ("r2_val_mgpu1_100", "r2_val_mgpu4_100", "r2_val_perturb_1e-15", "r2_val_perturb_1e-14"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["gpus"], d["steps"], repr(d["t"]), repr(d["Lz_end"]), "%.4f%%" % (100 * d["rel_to_paper"]),
              "E drift %.3e" % d["E_drift_rel_after_startup"], "p %.1e" % max(abs(v) for v in d["momentum_rel_to_sum_m_abs_v"]),
              "wall %.1f s" % d["wall_s"])
    except Exception as e:
        print(f, "FAILED", e)
PY
