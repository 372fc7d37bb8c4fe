#!/bin/bash
# A/B of the SIMT stage layouts: default vs scratch/libhofem_p<P1>_<name>.so
out=${1:-gpurun_out/ab_layout.txt}
: > $out
for rep in 1 2; do
for p in 2 4 5 6 8; do
  for b in bp3 bp1 bp5; do
    python scripts/time_apply.py --bench $b --p $p --tag default >> $out 2>&1
  done
done
for lib in scratch/libhofem_p*.so; do
  P1=$(echo $lib | sed 's/.*libhofem_p\([0-9]\)_.*/\1/'); p=$((P1-1))
  for b in bp3 bp1 bp5; do
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench $b --p $p --tag $(basename $lib .so | sed 's/libhofem_//') >> $out 2>&1
  done
done
done
