#!/bin/bash
# A/B on the box: current defaults vs the previous P1=6 / P1=7 knobs
out=${1:-gpurun_out/ab_p6.txt}
mkdir -p scratch
python -m paper_2402_15940_b200.build --force > /dev/null
python scripts/build_pvariant.py p6_prev 6 -DHOFEM_EO_DLA=1 -DHOFEM_EO_PRE=0 > /dev/null
python scripts/build_pvariant.py p7_prev 7 -DHOFEM_SIMT_T2QX=0 > /dev/null
: > $out
for rep in 1 2; do
  for b in bp1 bp3 bp5; do
    python scripts/time_apply.py --bench $b --p 5 --tag default >> $out 2>&1
    HOFEM_LIB_PATH=scratch/libhofem_p6_prev.so python scripts/time_apply.py --bench $b --p 5 --tag p6_prev >> $out 2>&1
    python scripts/time_apply.py --bench $b --p 6 --tag default >> $out 2>&1
    HOFEM_LIB_PATH=scratch/libhofem_p7_prev.so python scripts/time_apply.py --bench $b --p 6 --tag p7_prev >> $out 2>&1
  done
  python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag default >> $out 2>&1
  HOFEM_LIB_PATH=scratch/libhofem_p6_prev.so python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag p6_prev >> $out 2>&1
done
