#!/bin/bash
# partial D staging (DSP=1) on the P1=6 1x3 brick: time + ncu source capture
out=${1:-gpurun_out/ab_dsp2}
mkdir -p $out
python -m paper_2402_15940_b200.build > /dev/null
python scripts/build_pvariant.py p6_dsp1 6 -DHOFEM_SIMT_DSP=1 > /dev/null
for rep in 1 2; do
  for mesh in "--n 62" "--slab 200,200,25"; do
    python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag default >> $out/t.txt 2>&1
    HOFEM_LIB_PATH=scratch/libhofem_p6_dsp1.so python scripts/time_apply.py --bench bp3 --p 5 $mesh --tag dsp1 >> $out/t.txt 2>&1
  done
done
HOFEM_LIB_PATH=scratch/libhofem_p6_dsp1.so ncu --clock-control none --set full --import-source on -c 1 -k regex:fused_elem \
  -o $out/dsp1_p5 python scripts/prof_apply.py --p 5 > /dev/null 2>&1
