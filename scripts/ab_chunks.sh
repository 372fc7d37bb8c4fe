#!/bin/bash
out=${1:-gpurun_out/ab_chunks.txt}
: > $out
for rep in 1 2; do
  python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag default >> $out 2>&1
  for lib in scratch/chunks/*.so; do
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag $(basename $lib .so | sed 's/libhofem_//') >> $out 2>&1
  done
done
