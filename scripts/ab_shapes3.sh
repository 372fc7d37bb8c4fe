#!/bin/bash
# Brick-shape A/B for P1 = 5, 7, 8 (BP3) and BP5 P1 = 7 (item counts vs thread
# counts), built ON the box.  usage: bash scripts/ab_shapes3.sh <outfile>
out=${1:-gpurun_out/ab_shapes3.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/shapes3
# kind(SS|SC) P1 BX BY NT MAXR
for v in "SS 5 1 4 160 102" "SS 5 2 2 160 102" "SS 5 1 2 96 102" "SS 5 3 2 224 102" "SS 5 1 3 128 102" \
         "SS 7 1 2 128 168" "SS 7 1 3 192 168" "SS 8 1 2 192 168" "SC 7 1 3 160 128" "SC 7 3 1 160 128"; do
  set -- $v; name=${1}${2}_s$3x$4_$5_$6
  python scripts/build_pvariant.py $name $2 -DHOFEM_$1_P1=$2 -DHOFEM_$1_BX=$3 -DHOFEM_$1_BY=$4 \
    -DHOFEM_$1_NT=$5 -DHOFEM_$1_MAXR=$6 -DHOFEM_$1_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/shapes3/ || echo FAIL $v >> $out
done
run() {  # bench p mesh-args prefix
  python scripts/time_apply.py --bench $1 --p $2 $3 --tag default >> $out 2>&1
  for lib in scratch/shapes3/libhofem_$4_*.so; do
    t=$(basename $lib .so | sed 's/libhofem_//')
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench $1 --p $2 $3 --tag $t >> $out 2>&1
  done
}
for rep in 1 2; do
  run bp3 4 "--n 78" SS5; run bp3 4 "--n 80" SS5
  run bp3 6 "--n 52" SS7; run bp3 6 "--n 48" SS7
  run bp3 7 "--n 44" SS8; run bp3 7 "--n 42" SS8
  run bp5 6 "--n 52" SC7; run bp5 6 "--n 48" SC7
done
