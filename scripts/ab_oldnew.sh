#!/bin/bash
# A/B of the working-tree build against abl/libhofem_old.so (a copy of the
# previous build): brick-kernel times for BP3 p=4..7, config 5, BP5, BP1, and
# persistent / fused CG at small sizes.  usage: bash scripts/ab_oldnew.sh <outdir>
out=${1:-gpurun_out/ab_oldnew}
mkdir -p $out
: > $out/apply.txt; : > $out/cg.txt
for rep in 1 2; do
  for lib in abl/libhofem_old.so paper_2402_15940_b200/libhofem.so; do
    t=$(basename $(dirname $lib))
    for a in "--bench bp3 --p 4" "--bench bp3 --p 5" "--bench bp3 --p 6" "--bench bp3 --p 7" \
             "--bench bp3 --p 5 --slab 200,200,25" "--bench bp5 --p 5" "--bench bp1 --p 5" "--bench bp1 --p 3"; do
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py $a --tag $t >> $out/apply.txt 2>&1
    done
    echo "== $t" >> $out/cg.txt
    HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 5 --ns 8,12,62 --modes persistent,fused,separate --iters 50 >> $out/cg.txt
    HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp1 --ps 5 --ns 20 --modes persistent,fused --iters 100 >> $out/cg.txt
  done
done
