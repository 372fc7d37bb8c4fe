#!/bin/bash
# evict_last policy on the qdata L2 prefetch at P1 = 5, 7, 8, 9 (adopted at 6).
out=${1:-gpurun_out/ab_pfpol.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/pf
for P1 in 5 7 8 9; do
  python scripts/build_pvariant.py p${P1}_pfpol1 $P1 -DHOFEM_L2PF_POL=1 > /dev/null 2>&1 \
    && mv scratch/libhofem_p${P1}_pfpol1.so scratch/pf/ || echo FAIL $P1 >> $out
done
for rep in 1 2; do
  for P1 in 5 7 8 9; do
    p=$((P1 - 1))
    for b in bp3 bp5; do
      python scripts/time_apply.py --bench $b --p $p --tag default >> $out 2>&1
      HOFEM_LIB_PATH=scratch/pf/libhofem_p${P1}_pfpol1.so python scripts/time_apply.py --bench $b --p $p --tag pfpol1 >> $out 2>&1
    done
  done
done
