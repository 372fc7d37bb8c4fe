#!/bin/bash
# A/B of BP3 p=5 brick shapes: default vs scratch/shapes/libhofem_p6_s*.so (62^3 and config 5)
out=${1:-gpurun_out/ab_shapes.txt}
: > $out
for rep in 1 2; do
  python scripts/time_apply.py --bench bp3 --p 5 --tag default >> $out 2>&1
  python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag default >> $out 2>&1
  for lib in scratch/shapes/*.so; do
    t=$(basename $lib .so | sed 's/libhofem_//')
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 --tag $t >> $out 2>&1
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag $t >> $out 2>&1
  done
done
