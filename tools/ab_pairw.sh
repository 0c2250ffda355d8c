#!/bin/bash
# forward: weight application of two merged chunks as fma.rn.f32x2 (pairw, default) vs scalar (nopairw)
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pt_pairw.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_pairw.log
O=gpurun_out/ab_pairw.jsonl; : > $O
for v in nopairw "" nopairw ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2,c1 --dtypes f32 --ops fwd --iters 5 >> $O 2>>gpurun_out/ab_pairw.err
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops fwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_pairw.err
done
echo DONE
