#!/bin/bash
# Knobs on top of the P1 = 6 1x3 / 160-thread brick (built ON the box), and the
# 1x3 shape for BP1 p=5.  usage: bash scripts/ab_p6x3.sh <outfile>
out=${1:-gpurun_out/ab_p6x3.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/p6x3
for v in "dla1 -DHOFEM_EO_DLA=1" "t2qx0 -DHOFEM_SIMT_T2QX=0" "pre1 -DHOFEM_EO_PRE=1" "endbar1 -DHOFEM_SIMT_ENDBAR=1" \
         "m1x3 -DHOFEM_SM_P1=6 -DHOFEM_SM_BX=1 -DHOFEM_SM_BY=3 -DHOFEM_SM_NT=160 -DHOFEM_SM_MAXR=128 -DHOFEM_SM_CPS=8"; do
  set -- $v; name=$1; shift
  python scripts/build_pvariant.py p6_$name 6 "$@" > /dev/null 2>&1 \
    && mv scratch/libhofem_p6_$name.so scratch/p6x3/ || echo FAIL $name >> $out
done
for rep in 1 2; do
  for mesh in "--n 62" "--n 60" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out 2>&1
    for lib in scratch/p6x3/*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      [ $t = p6_m1x3 ] && continue
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag $t >> $out 2>&1
    done
  done
  python scripts/time_apply.py --bench bp1 --p 5 --tag default >> $out 2>&1
  HOFEM_LIB_PATH=scratch/p6x3/libhofem_p6_m1x3.so python scripts/time_apply.py --bench bp1 --p 5 --tag m1x3 >> $out 2>&1
done
