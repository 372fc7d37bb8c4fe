#!/bin/bash
# D pairs in flight / register cap on the P1 = 6 1x3 brick (built ON the box).
out=${1:-gpurun_out/ab_p6dla.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/p6dla
S="-DHOFEM_SS_P1=6 -DHOFEM_SS_BX=1 -DHOFEM_SS_BY=3 -DHOFEM_SS_NT=160 -DHOFEM_SS_CPS=8"
for v in "r136 -DHOFEM_SS_MAXR=136" "dla3 -DHOFEM_SS_MAXR=128 -DHOFEM_EO_DLA=3" "dla4 -DHOFEM_SS_MAXR=128 -DHOFEM_EO_DLA=4" \
         "r136dla3 -DHOFEM_SS_MAXR=136 -DHOFEM_EO_DLA=3" "r136dla4 -DHOFEM_SS_MAXR=136 -DHOFEM_EO_DLA=4"; do
  set -- $v; name=$1; shift
  python scripts/build_pvariant.py p6_$name 6 $S "$@" > /dev/null 2>&1 \
    && mv scratch/libhofem_p6_$name.so scratch/p6dla/ || echo FAIL $name >> $out
done
for rep in 1 2; do
  for mesh in "--n 62" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out 2>&1
    for lib in scratch/p6dla/*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag $t >> $out 2>&1
    done
  done
  python scripts/time_apply.py --bench bp1 --p 5 --tag default >> $out 2>&1
  for lib in scratch/p6dla/*.so; do
    t=$(basename $lib .so | sed 's/libhofem_//')
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp1 --p 5 --tag $t >> $out 2>&1
  done
done
