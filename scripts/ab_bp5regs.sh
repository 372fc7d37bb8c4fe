#!/bin/bash
# BP5 (collocated) register caps: the kernels fit in 96-102 registers without
# spills (ptxas), more CTAs per SM where shared memory allows.  Built ON the box.
out=${1:-gpurun_out/ab_bp5regs.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/b5r
# P1 BX BY NT MAXR
for v in "5 3 2 160 96" "7 2 1 128 102" "7 2 1 128 96" "8 2 1 128 102" "8 2 1 128 96" "9 1 1 96 102" "6 2 2 160 102"; do
  set -- $v; name=SC$1_r$5
  python scripts/build_pvariant.py $name $1 -DHOFEM_SC_P1=$1 -DHOFEM_SC_BX=$2 -DHOFEM_SC_BY=$3 \
    -DHOFEM_SC_NT=$4 -DHOFEM_SC_MAXR=$5 -DHOFEM_SC_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/b5r/ || echo FAIL $v >> $out
done
for rep in 1 2; do
  for P1 in 5 6 7 8 9; do
    p=$((P1 - 1))
    python scripts/time_apply.py --bench bp5 --p $p --tag default >> $out 2>&1
    for lib in scratch/b5r/libhofem_SC${P1}_*.so; do
      [ -e $lib ] || continue
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp5 --p $p --tag $t >> $out 2>&1
    done
  done
done
