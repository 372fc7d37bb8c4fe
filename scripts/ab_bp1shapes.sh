#!/bin/bash
# A/B on the box: BP1 (~1M dofs, L2-resident) brick shapes, p = 3, 5, 8
out=${1:-gpurun_out/ab_bp1shapes.txt}
mkdir -p scratch
python -m paper_2402_15940_b200.build > /dev/null
# P1 BX BY NT MAXR CPS
for v in "4 1 1 64 128 8" "4 2 1 96 128 5" "6 1 1 64 128 8" "6 1 2 128 128 4" "6 2 1 128 128 4" "9 1 1 96 128 5"; do
  set -- $v
  python scripts/build_pvariant.py bp1_p$1_s$2x$3_$4 $1 -DHOFEM_SM_P1=$1 -DHOFEM_SM_BX=$2 -DHOFEM_SM_BY=$3 \
    -DHOFEM_SM_NT=$4 -DHOFEM_SM_MAXR=$5 -DHOFEM_SM_CPS=$6 > /dev/null || echo FAIL $v
done
: > $out
for rep in 1 2; do
  for P1 in 4 6 9; do
    p=$((P1-1))
    python scripts/time_apply.py --bench bp1 --p $p --tag default >> $out 2>&1
    python scripts/cg_modes.py --bench bp1 --ps $p --iters 100 --modes fused | sed 's/^/default /' >> $out 2>&1
    for lib in scratch/libhofem_bp1_p${P1}_*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp1 --p $p --tag $t >> $out 2>&1
      HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp1 --ps $p --iters 100 --modes fused | sed "s/^/$t /" >> $out 2>&1
    done
  done
done
