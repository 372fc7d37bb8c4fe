#!/bin/bash
# P1 = 6: 1x5 bricks / 256 threads (S1 / S2 / S3 180 / 210 / 245 items, epilogue
# 156 rows; 2 CTAs/SM = 16 warps, 10 elements in flight) vs the 1x3 / 160 default.
out=${1:-gpurun_out/ab_p6x5.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/x5
for v in "1 5 256 128" "5 1 256 128" "1 5 224 128"; do
  set -- $v; name=p6_s$1x$2_$3_$4
  python scripts/build_pvariant.py $name 6 -DHOFEM_SS_P1=6 -DHOFEM_SS_BX=$1 -DHOFEM_SS_BY=$2 \
    -DHOFEM_SS_NT=$3 -DHOFEM_SS_MAXR=$4 -DHOFEM_SS_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/x5/ || echo FAIL $v >> $out
done
for rep in 1 2; do
  for mesh in "--n 62" "--n 60" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out 2>&1
    for lib in scratch/x5/*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag $t >> $out 2>&1
    done
  done
done
