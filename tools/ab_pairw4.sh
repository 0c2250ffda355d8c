#!/bin/bash
# double-backward family: v*y / v*db as one paired multiply (pairw, default) vs two (nopairw)
timeout 1800 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pt_pairw4.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_pairw4.log
O=gpurun_out/ab_pairw4.jsonl; : > $O
for v in nopairw "" nopairw ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2,c1 --dtypes f32 --ops dbwd --iters 3 >> $O 2>>gpurun_out/ab_pairw4.err
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops dbwd --dtypes f32 --modes det --iters 2 >> $O 2>>gpurun_out/ab_pairw4.err
done
echo DONE
