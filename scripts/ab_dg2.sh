#!/bin/bash
# A/B on the box: DG batch shapes at P1 = 2, 8, 9 (default vs NE/NT variants)
out=${1:-gpurun_out/ab_dg2.txt}
mkdir -p scratch
python -m paper_2402_15940_b200.build > /dev/null
for v in "9 1 128" "8 1 96" "8 4 352" "2 32 288" "2 8 96"; do
  set -- $v
  python scripts/build_pvariant.py --src dg_p dg_p$1_ne$2_nt$3 $1 -DHOFEM_DG_NE=$2 -DHOFEM_DG_NT=$3 > /dev/null || echo FAIL $v
done
: > $out
for rep in 1 2; do
  python scripts/time_dg.py 1,7,8 | sed 's/^/default /' >> $out
  for lib in scratch/libhofem_dg_p*.so; do
    P1=$(echo $lib | sed 's/.*dg_p\([0-9]\)_.*/\1/'); p=$((P1-1))
    HOFEM_LIB_PATH=$lib python scripts/time_dg.py $p | sed "s|^|$(basename $lib .so) |" >> $out
  done
done
