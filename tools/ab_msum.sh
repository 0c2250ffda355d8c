#!/bin/bash
# dy warp sums: recursive halving (default) vs one butterfly per value (CGF_GEN=nomsum)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/pt_msum.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pt_msum.log
O=gpurun_out/ab_msum.jsonl; : > $O
for v in nomsum ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --dtypes f32,f64 --ops bwd,dbwd --iters 3 >> $O 2>>gpurun_out/ab_msum.err
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c1 --dtypes f32,f64 --ops bwd,dbwd --iters 3 >> $O 2>>gpurun_out/ab_msum.err
  CGF_GEN="$v" timeout 1500 python tools/sweep_conv.py --cases c4,c5 --ops bwd,dbwd --dtypes f32,f64 --modes det >> $O 2>>gpurun_out/ab_msum.err
done
echo DONE
