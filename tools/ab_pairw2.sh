#!/bin/bash
# backward: paired gz*w products and gW chains (pairw, default) vs scalar (nopairw)
timeout 1800 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -p no:cacheprovider -x > gpurun_out/pt_pairw2.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_pairw2.log
O=gpurun_out/ab_pairw2.jsonl; : > $O
for v in nopairw "" nopairw ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2,c1 --dtypes f32 --ops bwd --iters 5 >> $O 2>>gpurun_out/ab_pairw2.err
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops bwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_pairw2.err
done
echo DONE
