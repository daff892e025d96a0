mkdir -p gpurun_out; : > gpurun_out/dbg_seq.log
for s in a c b a c; do timeout 40 python scripts/dbg_seq33.py $s >> gpurun_out/dbg_seq.log 2>&1; echo "seq $s rc=$?" >> gpurun_out/dbg_seq.log; done
grep -E "rc=" gpurun_out/dbg_seq.log
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -m gpu -q -p no:cacheprovider -o faulthandler_timeout=200 -k "one_sided or full_cube or c3_image or host_executor or planar or both_kernels" > gpurun_out/pytest_lut.log 2>&1; echo "pytest=$?"; grep -E "FAILED|passed|failed|Timeout" gpurun_out/pytest_lut.log | tail -8
