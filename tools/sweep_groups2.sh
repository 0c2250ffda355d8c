#!/bin/bash
# Group counts re-swept after the multi-value warp sums / unrolled stores
mkdir -p gpurun_out
O=gpurun_out/sweep_groups2.jsonl; : > $O
for G in 2 4 6 8 12; do
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
done
for G in 1 2 4; do
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
done
for G in 1 2 3; do
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c5 --ops dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c5 --ops bwd --dtypes f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
done
for G in 1 2 3 4 6 8; do
  CGF_ROW_GROUPS=$G timeout 900 python tools/sweep.py --configs c2,c1 --ops dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
done
for G in 1 2 3; do
  CGF_ROW_GROUPS_BWD=$G timeout 900 python tools/sweep.py --configs c2,c1 --ops bwd --dtypes f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups2.err
done
echo DONE
