#!/bin/bash
# A/B the fused kernel variants (HOFEM_FUSED=mma|simt) on BP3/BP1 applies.
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-mma simt}; do
  for spec in ${SPECS:-"bp3 3" "bp3 4" "bp3 5" "bp3 6" "bp3 7" "bp1 3" "bp1 5" "bp1 7"}; do
    set -- $spec
    HOFEM_FUSED=$v python scripts/time_apply.py --bench $1 --p $2 --tag "$v"
  done
done
