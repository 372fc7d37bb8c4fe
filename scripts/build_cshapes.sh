#!/bin/bash
# Build collocated SIMT shape variants: each arg "name P1 BX BY NT MAXR CPS".
cd "$(dirname "$0")/.."
for v in "$@"; do
  set -- $v
  python scripts/build_variant.py $1 -DHOFEM_SC_P1=$2 -DHOFEM_SC_BX=$3 -DHOFEM_SC_BY=$4 \
    -DHOFEM_SC_NT=$5 -DHOFEM_SC_MAXR=$6 -DHOFEM_SC_CPS=$7 2>&1 | tail -1
done
python -c "from paper_2402_15940_b200 import build; build.build(force=True)"
