#!/bin/bash
# A/B of partial D staging (HOFEM_SIMT_DSP: outer z point pairs of D in shared
# memory, bulk-copied one brick ahead) for the BP3 brick kernel, built ON the box.
# usage: bash scripts/ab_dsp.sh <outfile>
out=${1:-gpurun_out/ab_dsp.txt}
: > $out
python -m paper_2402_15940_b200.build > /dev/null
for v in "5 1" "5 2" "6 1" "6 2" "7 1" "7 2"; do
  set -- $v
  python scripts/build_pvariant.py p$1_dsp$2 $1 -DHOFEM_SIMT_DSP=$2 > /dev/null || echo FAIL $v >> $out
done
for rep in 1 2; do
  for P1 in 5 6 7; do
    p=$((P1 - 1))
    python scripts/time_apply.py --bench bp3 --p $p --tag default >> $out 2>&1
    for d in 1 2; do
      HOFEM_LIB_PATH=scratch/libhofem_p${P1}_dsp$d.so python scripts/time_apply.py --bench bp3 --p $p --tag dsp$d >> $out 2>&1
    done
  done
  python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag default >> $out 2>&1
  for d in 1 2; do
    HOFEM_LIB_PATH=scratch/libhofem_p6_dsp$d.so python scripts/time_apply.py --bench bp3 --p 5 --slab 200,200,25 --tag dsp$d >> $out 2>&1
  done
done
# parity of every variant (fused apply vs the oracle, CG iterates, full-size samples)
for lib in scratch/libhofem_p*_dsp*.so; do
  echo "== parity $lib" >> $out
  HOFEM_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "fused_and_unfused or cg_iterates_small or sampled_points_full_size or bitwise" >> $out 2>&1
done
