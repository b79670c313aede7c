set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_v1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_search|k_expand_rows|k_density_c|k_iad_c" -s 20 -c 5 -o gpurun_out/r2_full_v1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_full.log 2>&1
ls -la gpurun_out/
