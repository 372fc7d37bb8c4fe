#!/bin/bash
# BP5: one-round epilogues by more threads at a lower register cap (built ON the box).
out=${1:-gpurun_out/ab_bp5nt.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/b5n
for v in "6 2 2 192 102" "6 2 2 192 96" "5 3 2 192 96" "5 3 2 192 84"; do
  set -- $v; name=SC$1_s$2x$3_$4_$5
  python scripts/build_pvariant.py $name $1 -DHOFEM_SC_P1=$1 -DHOFEM_SC_BX=$2 -DHOFEM_SC_BY=$3 \
    -DHOFEM_SC_NT=$4 -DHOFEM_SC_MAXR=$5 -DHOFEM_SC_CPS=8 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/b5n/ || echo FAIL $v >> $out
done
for rep in 1 2; do
  for P1 in 5 6; do
    p=$((P1 - 1))
    for mesh in "" "--n 60"; do
      python scripts/time_apply.py --bench bp5 --p $p $mesh --tag default >> $out 2>&1
      for lib in scratch/b5n/libhofem_SC${P1}_*.so; do
        t=$(basename $lib .so | sed 's/libhofem_//')
        HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp5 --p $p $mesh --tag $t >> $out 2>&1
      done
    done
  done
done
