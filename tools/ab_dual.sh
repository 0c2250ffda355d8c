#!/bin/bash
# Paired FP32 emission for the double-backward family (merged chunks): parity + timing.
mkdir -p gpurun_out
CGF_GEN=merge=2,joint,ffma2 python -m pytest tests/test_gpu_conv.py tests/test_gpu_tp.py -q -p no:cacheprovider -x -k "double or dbwd or grouped or fwd_bwd_dbwd or forward_backward_double" > gpurun_out/pytest_dual.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_dual.log
O=gpurun_out/ab_dual.jsonl; : > $O
for F in "" merge=2,joint,ffma2; do
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2,c1 --ops dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_dual.err
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_dual.err
done
echo DONE
