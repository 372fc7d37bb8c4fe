mkdir -p gpurun_out/s3t
out=gpurun_out/s3t/t.txt; : > $out
for rep in 1 2; do
for lib in abl/libhofem_old.so paper_2402_15940_b200/libhofem.so; do
  echo "== $lib" >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 5 --ns 6,8,12,16 --modes persistent,fused --iters 100 >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp1 --ps 5 --ns 8,12,20 --modes persistent,fused --iters 100 >> $out
  HOFEM_LIB_PATH=$lib python scripts/cg_modes.py --bench bp3 --ps 3,7 --ns 8 --modes persistent,fused --iters 100 >> $out
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "cg" > gpurun_out/s3t/cgtest.txt 2>&1
