#!/bin/bash
# C5 (edge-pair kernels): paired w*gz products (pairw, default) vs scalar (nopairw); unit coefficients as copies (always)
timeout 1800 python -m pytest tests/test_gpu_conv.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/pt_pairw3.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_pairw3.log
O=gpurun_out/ab_pairw3.jsonl; : > $O
for v in nopairw "" nopairw ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_pairw3.err
done
echo DONE
