#!/bin/bash
# BP5 (collocated) brick shapes whose epilogue fits in one round of the CTA
# (rows per column padded to 32; 2x2 at P1 = 6 and 3x2 at P1 = 5 need two).
out=${1:-gpurun_out/ab_bp5shapes.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/bp5s
for v in "6 1 3 128 128" "6 1 4 160 128" "6 1 2 96 128" "5 1 6 160 102" "5 1 4 128 102" "5 1 3 96 102"; do
  set -- $v; name=SC$1_s$2x$3_$4_$5
  python scripts/build_pvariant.py $name $1 -DHOFEM_SC_P1=$1 -DHOFEM_SC_BX=$2 -DHOFEM_SC_BY=$3 \
    -DHOFEM_SC_NT=$4 -DHOFEM_SC_MAXR=$5 -DHOFEM_SC_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/bp5s/ || echo FAIL $v >> $out
done
run() {  # p mesh prefix
  python scripts/time_apply.py --bench bp5 --p $1 $2 --tag default >> $out 2>&1
  for lib in scratch/bp5s/libhofem_$3_*.so; do
    t=$(basename $lib .so | sed 's/libhofem_//')
    HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp5 --p $1 $2 --tag $t >> $out 2>&1
  done
}
for rep in 1 2; do
  run 5 "--n 62" SC6; run 5 "--n 60" SC6; run 5 "--slab 200,200,25" SC6
  run 4 "--n 78" SC5; run 4 "--n 80" SC5
done
