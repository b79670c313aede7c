# Round evidence on 1 B200: bench line (with cpu_baseline), reference arm, other configs,
# smoke, ncu launch list and one --set full capture of the pair kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo rc=$? >> gpurun_out/ev_smoke.log
timeout 600 python bench.py > gpurun_out/ev_bench_w1.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1
timeout 300 python bench.py --workload patch1m --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_1m.log 2>&1
timeout 300 python bench.py --workload evrard --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_evrard.log 2>&1
timeout 600 python bench.py --workload patch27m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench_27m.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_momentum_c|k_density_c|k_iad_c|k_search" -s 12 -c 4 -o gpurun_out/ev_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_full.log 2>&1
for f in ev_smoke ev_bench_w1 ev_bench_ref ev_bench_1m ev_bench_evrard ev_bench_27m ev_ncu_full; do echo "== $f"; tail -1 gpurun_out/$f.log | cut -c1-300; done
