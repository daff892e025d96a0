for m in trilinear prism pyramidal tetrahedral; do timeout 120 python scripts/prof_kernel.py --op lut17 --method $m --iters 20 --time; done
timeout 900 python -m pytest tests/test_gpu_exact_lut.py -x -q -k "lut17 or interp" 2>&1 | tail -2
