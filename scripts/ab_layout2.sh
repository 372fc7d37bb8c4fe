#!/bin/bash
out=${1:-gpurun_out/ab_layout2.txt}
: > $out
for rep in 1 2; do
for lib in default scratch/libhofem_p*.so; do
  for P1 in 2 4 8; do
    case $lib in default) ;; *) [ "$(echo $lib | sed 's/.*libhofem_p\([0-9]\)_.*/\1/')" = "$P1" ] || continue;; esac
    p=$((P1-1))
    for b in bp3 bp1 bp5; do
      if [ $lib = default ]; then python scripts/time_apply.py --bench $b --p $p --tag default >> $out 2>&1
      else HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench $b --p $p --tag $(basename $lib .so | sed 's/libhofem_//') >> $out 2>&1; fi
    done
  done
done
done
