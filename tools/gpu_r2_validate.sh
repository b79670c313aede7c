set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/validate_square_patch.py --n 30 --every 100 --out gpurun_out/val_gpu_30.json > gpurun_out/val_gpu_30.log 2>&1
timeout 300 python tools/validate_square_patch.py --n 30 --every 100 --symmetric 1 --out gpurun_out/val_gpu_30_sym.json > gpurun_out/val_gpu_30_sym.log 2>&1
timeout 600 python tools/validate_square_patch.py --n 100 --out gpurun_out/val_gpu_100.json > gpurun_out/val_gpu_100.log 2>&1
timeout 600 python tools/validate_square_patch.py --n 100 --symmetric 1 --out gpurun_out/val_gpu_100_sym.json > gpurun_out/val_gpu_100_sym.log 2>&1
timeout 600 python tools/validate_square_patch.py --n 60 --out gpurun_out/val_gpu_60.json > gpurun_out/val_gpu_60.log 2>&1
for f in gpurun_out/val_gpu_*.log; do echo "== $f"; tail -1 $f | cut -c1-600; done
