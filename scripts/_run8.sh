mkdir -p gpurun_out
for rep in 1 2; do for lib in paper_1009_0854_b200/libmact_cuda.so paper_1009_0854_b200/libmact_cuda_a*.so; do
  echo -n "$(basename $lib) corr: "; MACT_LIB=$PWD/$lib timeout 120 python scripts/prof_kernel.py --op all --input corr --iters 20 --time
done; done > gpurun_out/all_sweep.txt 2>&1
for w in c2 c5; do timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline --workload $w > gpurun_out/b_$w.json 2>&1; done
