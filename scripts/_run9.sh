mkdir -p gpurun_out
for rep in 1 2; do for lib in paper_1009_0854_b200/libmact_cuda.so paper_1009_0854_b200/libmact_cuda_a*.so; do
  echo -n "$(basename $lib) corr: "; MACT_LIB=$PWD/$lib timeout 120 python scripts/prof_kernel.py --op all --input corr --iters 20 --time
done; for lib in paper_1009_0854_b200/libmact_cuda.so paper_1009_0854_b200/libmact_cuda_l*.so; do
  echo -n "$(basename $lib) corr: "; MACT_LIB=$PWD/$lib timeout 120 python scripts/prof_kernel.py --op lab --input corr --iters 30 --time
done; done > gpurun_out/all_sweep2.txt 2>&1
