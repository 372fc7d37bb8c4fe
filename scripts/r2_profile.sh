#!/bin/bash
# Round-2 profiling pass (one GPU; never under torchrun):
#   1. the ncu launch list of a short bench run (no sweep) -> kernel shares of the step
#   2. ncu --set full of the dominant kernel at the bench config and of the
#      kernels SURVEY §8(d) asks FP64 figures for (BP3 p=7,8; BP1 p=5,8), plus the
#      f3 (matrix-free) and f4 (DG) kernels.
# usage: bash scripts/r2_profile.sh <tag>   (writes gpurun_out/<tag>/)
tag=${1:-r2g}
out=gpurun_out/$tag
mkdir -p $out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sweep > $out/launch_run.log 2>&1
FULL="$NCU --set full --import-source on -c 1"
$FULL -k regex:fused_elem -o $out/simt_p5_200x200x25 python scripts/prof_apply.py --p 5 --slab 200,200,25 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p5 python scripts/prof_apply.py --p 5 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p4 python scripts/prof_apply.py --p 4 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p6 python scripts/prof_apply.py --p 6 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/bp5_p5 python scripts/prof_apply.py --bench bp5 --p 5 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p7 python scripts/prof_apply.py --p 7 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p8 python scripts/prof_apply.py --p 8 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/bp1_p5 python scripts/prof_apply.py --bench bp1 --p 5 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/bp1_p8 python scripts/prof_apply.py --bench bp1 --p 8 > /dev/null 2>&1
$FULL -k regex:mf_diffusion -o $out/mf_p5 python scripts/prof_apply.py --p 5 --mf > /dev/null 2>&1
$FULL -k regex:dg_mass -o $out/dg_p5 python scripts/prof_apply.py --bench dg --p 5 > /dev/null 2>&1
ls -la $out
