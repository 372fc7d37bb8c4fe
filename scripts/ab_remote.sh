#!/bin/bash
# Build the A/B variant libraries ON the GPU box (they are too large to ship),
# then run the A/B scripts.  usage: bash scripts/ab_remote.sh <outdir>
out=${1:-gpurun_out/ab}
mkdir -p $out scratch/shapes scratch/chunks
python -m paper_2402_15940_b200.build --force > /dev/null
for v in "6 pre1 -DHOFEM_EO_PRE=1" "6 dla2 -DHOFEM_EO_DLA=2" "6 dpol2 -DHOFEM_EO_DPOL=2" "6 l2pf2 -DHOFEM_L2PF_AHEAD=2" "5 t2qx -DHOFEM_SIMT_T2QX=1" "7 t2qx -DHOFEM_SIMT_T2QX=1"; do
  set -- $v; P1=$1; name=$2; shift 2
  python scripts/build_pvariant.py p${P1}_$name $P1 "$@" > /dev/null || echo FAIL $v
done
for v in "1 3 160 102 4" "3 1 160 102 4" "2 1 128 128 4" "1 2 160 102 4" "2 2 224 96 3"; do
  set -- $v; name=p6_s$1x$2_$3_$4
  python scripts/build_pvariant.py $name 6 -DHOFEM_SS_P1=6 -DHOFEM_SS_BX=$1 -DHOFEM_SS_BY=$2 \
    -DHOFEM_SS_NT=$3 -DHOFEM_SS_MAXR=$4 -DHOFEM_SS_CPS=$5 > /dev/null 2>&1 \
    && mv scratch/libhofem_$name.so scratch/shapes/ || echo FAIL $v
done
for c in 2 3 5; do
  python scripts/build_pvariant.py --src fused ch$c 0 -DHOFEM_CHUNKS_MIN=$c > /dev/null \
    && mv scratch/libhofem_ch$c.so scratch/chunks/ || echo FAIL ch$c
done
timeout 900 bash scripts/ab_knobs.sh $out/ab_knobs.txt
timeout 900 bash scripts/ab_shapes.sh $out/ab_shapes.txt
timeout 600 bash scripts/ab_chunks.sh $out/ab_chunks.txt
