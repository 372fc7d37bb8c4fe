#!/bin/bash
# Small-problem CG schedules, abl/libhofem_old.so vs the working-tree build.
out=${1:-gpurun_out/ab_cg_small.txt}; : > $out
for rep in 1 2; do for lib in abl/libhofem_old.so paper_2402_15940_b200/libhofem.so; do
  echo "== $(basename $(dirname $lib))" >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 5 --ns 4,8,12,16,24 --modes persistent,fused --iters 100 >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp1 --ps 5 --ns 20 --modes persistent,fused --iters 100 >> $out
done; done
