#!/bin/bash
# Final captures of the round (one GPU): launch list of the bench config, ncu
# --set full of the headline kernel (config-5 slab, 62^3), BP3 p=4/6/7/8, BP5 p=5,
# BP1 p=5, then the summaries (profiles/<tag>_*) and traffic.json.
tag=${1:-r2w}
out=gpurun_out/$tag
mkdir -p $out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sweep > $out/launch_run.log 2>&1
FULL="$NCU --set full --import-source on -c 1 -k regex:fused_elem"
$FULL -o $out/simt_p5_200x200x25 python scripts/prof_apply.py --p 5 --slab 200,200,25 > /dev/null 2>&1
$FULL -o $out/simt_p5 python scripts/prof_apply.py --p 5 > /dev/null 2>&1
$FULL -o $out/simt_p4 python scripts/prof_apply.py --p 4 > /dev/null 2>&1
$FULL -o $out/simt_p6 python scripts/prof_apply.py --p 6 > /dev/null 2>&1
$FULL -o $out/simt_p7 python scripts/prof_apply.py --p 7 > /dev/null 2>&1
$FULL -o $out/simt_p8 python scripts/prof_apply.py --p 8 > /dev/null 2>&1
$FULL -o $out/bp5_p5 python scripts/prof_apply.py --bench bp5 --p 5 > /dev/null 2>&1
$FULL -o $out/bp1_p5 python scripts/prof_apply.py --bench bp1 --p 5 > /dev/null 2>&1
mkdir -p $out/prof; cp profiles/traffic.json $out/prof/; python scripts/make_profiles.py $tag --out $out/prof > /dev/null 2>&1
ls -la $out $out/prof
