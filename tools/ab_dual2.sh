#!/bin/bash
# double-backward family: merged chunks side by side (joint) with / without paired FP32 ops, after the multi-sums
O=gpurun_out/ab_dual2.jsonl; : > $O
for v in "" "merge=2,joint,ffma2" "merge=2,joint"; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2,c1 --dtypes f32 --ops dbwd --iters 3 >> $O 2>>gpurun_out/ab_dual2.err
  CGF_GEN="$v" timeout 1500 python tools/sweep_conv.py --cases c4,c5 --ops dbwd --dtypes f32 --modes det >> $O 2>>gpurun_out/ab_dual2.err
done
echo DONE
