#!/bin/bash
# A/B timing of libhofem variants in scratch/ (run on the GPU box).
cp paper_2402_15940_b200/libhofem.so /tmp/libhofem_orig.so
for f in "$@"; do
  cp scratch/libhofem_$f.so paper_2402_15940_b200/libhofem.so
  timeout 300 python scripts/time_apply.py --p ${P:-5} --bench ${BENCH:-bp3} --tag $f 2>&1 | tail -1
done
cp /tmp/libhofem_orig.so paper_2402_15940_b200/libhofem.so
