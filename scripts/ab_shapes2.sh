#!/bin/bash
# A/B of BP3 p=5 (P1 = 6) brick shapes at 128 registers (item counts vs thread
# counts: S1 36 NE, S2 42 NE, S3 49 NE items), built ON the box.
# usage: bash scripts/ab_shapes2.sh <outfile>
out=${1:-gpurun_out/ab_shapes2.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/shapes2
for v in "1 3 160 128" "3 1 160 128" "1 5 256 128" "1 4 224 128" "2 2 224 128" "1 2 96 128" "1 3 160 112" "5 1 256 128"; do
  set -- $v; name=p6_s$1x$2_$3_$4
  python scripts/build_pvariant.py $name 6 -DHOFEM_SS_P1=6 -DHOFEM_SS_BX=$1 -DHOFEM_SS_BY=$2 \
    -DHOFEM_SS_NT=$3 -DHOFEM_SS_MAXR=$4 -DHOFEM_SS_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/shapes2/ || echo FAIL $v >> $out
done
for rep in 1 2; do
  for mesh in "--n 62" "--n 60" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out 2>&1
    for lib in scratch/shapes2/*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag $t >> $out 2>&1
    done
  done
done
