#!/bin/bash
# C4 FP32 conv backward (by neighbour) and C1 FP32 dbl-bwd knob check
O=gpurun_out/ab_c4bwd.jsonl; : > $O
for v in "" "depth=1" "depth=2" "minb=3" "minb=2" ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_c4bwd.err
done
for v in "" "depth=3" "depth=4"; do
  CGF_GEN="$v" timeout 600 python tools/sweep.py --configs c1 --ops dbwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_c4bwd.err
done
echo DONE
