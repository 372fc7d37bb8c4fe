#!/bin/bash
# A/B on the box: fully matrix-free batch shapes (NE elements, NT threads), p = 3, 5, 7
out=${1:-gpurun_out/ab_mf.txt}
mkdir -p scratch
python -m paper_2402_15940_b200.build > /dev/null
for v in "4 4 128" "4 2 96" "6 2 128" "6 4 224" "8 2 160" "8 1 96"; do
  set -- $v
  python scripts/build_pvariant.py --src mf_p mf_p$1_ne$2_nt$3 $1 -DHOFEM_MF_NE=$2 -DHOFEM_MF_NT=$3 > /dev/null || echo FAIL $v
done
: > $out
for rep in 1 2; do
  python scripts/time_mf.py 3,5,7 | sed 's/^/default /' >> $out 2>&1
  for lib in scratch/libhofem_mf_p*.so; do
    P1=$(echo $lib | sed 's/.*mf_p\([0-9]\)_.*/\1/'); p=$((P1-1))
    HOFEM_LIB_PATH=$lib python scripts/time_mf.py $p | sed "s|^|$(basename $lib .so) |" >> $out 2>&1
  done
done
