# A/B timing of in-tree variant builds (_v_<name>/libsph.so) against the main build.
# usage: bash tools/ab_variants.sh name1 name2 ...   (main = paper_2005_02656_b200/libsph.so)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = main ]; then lib=$PWD/paper_2005_02656_b200/libsph.so; else lib=$PWD/_v_$v/libsph.so; fi
  CUDA_VISIBLE_DEVICES=0 SPH_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
done
