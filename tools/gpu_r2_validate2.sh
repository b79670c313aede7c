set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/validate_square_patch.py --n 100 --h-max-factor 2 --out gpurun_out/val_gpu_100_hmax2.json > gpurun_out/val_gpu_100_hmax2.log 2>&1
timeout 600 python tools/validate_square_patch.py --n 100 --symmetric 1 --h-max-factor 2 --out gpurun_out/val_gpu_100_sym_hmax2.json > gpurun_out/val_gpu_100_sym_hmax2.log 2>&1
timeout 300 python tools/validate_square_patch.py --n 30 --symmetric 1 --h-max-factor 2 --every 100 --out gpurun_out/val_gpu_30_sym_hmax2.json > gpurun_out/val_gpu_30_sym_hmax2.log 2>&1
timeout 1500 python tools/shadow_window.py --n 100 --s0 3900 --k 8 --out gpurun_out/shadow_100_3900.json > gpurun_out/shadow_100_3900.log 2>&1
for f in gpurun_out/val_gpu_*hmax2*.log; do echo "== $f"; tail -1 $f | cut -c1-900; done
tail -9 gpurun_out/shadow_100_3900.log | cut -c1-400
