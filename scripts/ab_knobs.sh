#!/bin/bash
# A/B of per-P1 kernel knobs: default vs scratch/libhofem_p<P1>_<name>.so (BP3 + BP5, 30M dofs)
out=${1:-gpurun_out/ab_knobs.txt}
: > $out
for rep in 1 2; do
for lib in default scratch/libhofem_p*.so; do
  for P1 in 5 6 7; do
    case $lib in default) ;; *) [ "$(echo $lib | sed 's/.*libhofem_p\([0-9]\)_.*/\1/')" = "$P1" ] || continue;; esac
    p=$((P1-1))
    for b in bp3 bp5; do
      if [ $lib = default ]; then python scripts/time_apply.py --bench $b --p $p --tag default >> $out 2>&1
      else HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench $b --p $p --tag $(basename $lib .so | sed 's/libhofem_//') >> $out 2>&1; fi
    done
  done
done
done
