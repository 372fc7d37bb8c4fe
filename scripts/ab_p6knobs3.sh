#!/bin/bash
# Memory-policy knobs re-checked on the P1 = 6 1x3 brick (built ON the box).
out=${1:-gpurun_out/ab_p6knobs3.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
mkdir -p scratch/k3
for v in "dpol1 -DHOFEM_EO_DPOL=1" "dpol2 -DHOFEM_EO_DPOL=2" "pfpol1 -DHOFEM_L2PF_POL=1" "pf2 -DHOFEM_L2PF_AHEAD=2" "zo0 -DHOFEM_EO_ZO=0"; do
  set -- $v; name=$1; shift
  python scripts/build_pvariant.py p6_$name 6 "$@" > /dev/null 2>&1 \
    && mv scratch/libhofem_p6_$name.so scratch/k3/ || echo FAIL $name >> $out
done
for rep in 1 2; do
  for mesh in "--n 62" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out 2>&1
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --opt L2_PREFETCH=0 --tag nopf >> $out 2>&1
    for lib in scratch/k3/*.so; do
      t=$(basename $lib .so | sed 's/libhofem_//')
      HOFEM_LIB_PATH=$lib python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag $t >> $out 2>&1
    done
  done
done
