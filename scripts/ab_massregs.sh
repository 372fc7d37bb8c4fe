#!/bin/bash
# BP1 (mass) brick kernel register cap: the mass kernels inherited the diffusion
# caps (96-232); ptxas fits them in 64-96 without spills -> more CTAs per SM.
# Built ON the box.  usage: bash scripts/ab_massregs.sh <outfile>
out=${1:-gpurun_out/ab_massregs.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/mr
# P1 BX BY NT (current mass shape)
for v in "2 4 4 160" "3 4 2 128" "4 3 2 160" "5 2 2 160" "6 1 3 160" "7 1 1 64" "8 1 1 96" "9 1 1 128"; do
  set -- $v
  for r in 64 80 96; do
    name=m$1_r$r
    python scripts/build_pvariant.py $name $1 -DHOFEM_SM_P1=$1 -DHOFEM_SM_BX=$2 -DHOFEM_SM_BY=$3 \
      -DHOFEM_SM_NT=$4 -DHOFEM_SM_MAXR=$r -DHOFEM_SM_CPS=16 > /dev/null 2>&1 \
      && mv scratch/libhofem_$name.so scratch/mr/ || echo FAIL $name >> $out
  done
done
for rep in 1 2; do
  for P1 in 2 3 4 5 6 7 8 9; do
    p=$((P1 - 1))
    python scripts/time_apply.py --bench bp1 --p $p --reps 200 --tag default >> $out 2>&1
    for lib in scratch/mr/libhofem_m${P1}_*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp1 --p $p --reps 200 --tag $t >> $out 2>&1
    done
  done
done
