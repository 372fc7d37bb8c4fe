#!/bin/bash
# Build SIMT-shape variants: each arg "name P1 BX BY NT MAXR CPS".
cd "$(dirname "$0")/.."
for v in "$@"; do
  set -- $v
  python scripts/build_variant.py $1 -DHOFEM_SS_P1=$2 -DHOFEM_SS_BX=$3 -DHOFEM_SS_BY=$4 \
    -DHOFEM_SS_NT=$5 -DHOFEM_SS_MAXR=$6 -DHOFEM_SS_CPS=$7 2>&1 | tail -1
done
python -c "from paper_2402_15940_b200 import build; build.build(force=True)"
