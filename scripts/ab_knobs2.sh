#!/bin/bash
# A/B on the box of the stage-3 D-load knobs at P1 = 3, 4, 5, 7, 8 (both kinds)
out=${1:-gpurun_out/ab_knobs2.txt}
mkdir -p scratch
python -m paper_2402_15940_b200.build > /dev/null
for P1 in 3 4 5 7 8; do
  python scripts/build_pvariant.py p${P1}_dla2 $P1 -DHOFEM_EO_DLA=2 > /dev/null
  python scripts/build_pvariant.py p${P1}_pre1 $P1 -DHOFEM_EO_PRE=1 > /dev/null
  python scripts/build_pvariant.py p${P1}_pre0 $P1 -DHOFEM_EO_PRE=0 > /dev/null
done
: > $out
for rep in 1 2; do
  for P1 in 3 4 5 7 8; do
    p=$((P1-1))
    for b in bp3 bp5 bp1; do
      python scripts/time_apply.py --bench $b --p $p --tag default >> $out 2>&1
      for v in dla2 pre1 pre0; do
        HOFEM_LIB_PATH=scratch/libhofem_p${P1}_$v.so python scripts/time_apply.py --bench $b --p $p --tag p${P1}_$v >> $out 2>&1
      done
    done
  done
done
