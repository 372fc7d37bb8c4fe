#!/bin/bash
# A/B of DG batch shapes: default library vs scratch/libhofem_dg_p<P1>_ne<NE>_nt<NT>.so
out=${1:-gpurun_out/ab_dg.txt}
python scripts/time_dg.py 3,4,5,6,7,8 | sed 's/^/default /' > $out
for lib in scratch/libhofem_dg_p*.so; do
  P1=$(echo $lib | sed 's/.*dg_p\([0-9]\)_.*/\1/'); p=$((P1-1))
  HOFEM_LIB_PATH=$lib python scripts/time_dg.py $p | sed "s|^|$(basename $lib) |" >> $out
done
