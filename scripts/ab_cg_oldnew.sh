mkdir -p gpurun_out/s4b; out=gpurun_out/s4b/cg.txt; : > $out
for rep in 1 2; do for lib in abl/libhofem_old.so paper_2402_15940_b200/libhofem.so; do
  echo "== $(basename $(dirname $lib))" >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 5 --ns 8,12 --modes persistent --iters 100 >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp1 --ps 5 --ns 20 --modes persistent --iters 100 >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 5 --ns 62 --modes separate --iters 30 >> $out
done; done
