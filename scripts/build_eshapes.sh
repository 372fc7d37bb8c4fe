#!/bin/bash
# Build DMMA-shape variants: each arg "name P1 BX BY MINB".
cd "$(dirname "$0")/.."
for v in "$@"; do
  set -- $v
  python scripts/build_variant.py $1 -DHOFEM_SE_P1=$2 -DHOFEM_SE_BX=$3 -DHOFEM_SE_BY=$4 \
    -DHOFEM_SE_MINB=$5 2>&1 | tail -1
done
python -c "from paper_2402_15940_b200 import build; build.build(force=True)"
