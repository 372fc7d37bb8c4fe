#!/bin/bash
# Profiling pass after the P1=6 shape change (one GPU): launch list of a short
# bench run + ncu --set full of the BP3 p=5 kernel (config-5 slab, 62^3) and BP1 p=5.
tag=${1:-r2v}
out=gpurun_out/$tag
mkdir -p $out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sweep > $out/launch_run.log 2>&1
FULL="$NCU --set full --import-source on -c 1"
$FULL -k regex:fused_elem -o $out/simt_p5_200x200x25 python scripts/prof_apply.py --p 5 --slab 200,200,25 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/simt_p5 python scripts/prof_apply.py --p 5 > /dev/null 2>&1
$FULL -k regex:fused_elem -o $out/bp1_p5 python scripts/prof_apply.py --bench bp1 --p 5 > /dev/null 2>&1
python scripts/make_profiles.py $tag > /dev/null 2>&1
ls -la $out
