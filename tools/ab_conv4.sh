#!/bin/bash
# C4 FP64 forward: register cap for 3 CTAs / SM, with 2 or 3 edges per item
O=gpurun_out/ab_conv4.jsonl; : > $O
for v in "" "minb=3" "minb=3,epi=3" "minb=4" "minb=3" ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f64 --modes det --iters 3 >> $O 2>>gpurun_out/ab_conv4.err
done
CGF_GEN="minb=3" timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd --dtypes f64 --modes det --iters 3 >> $O 2>>gpurun_out/ab_conv4.err
timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd --dtypes f64 --modes det --iters 3 >> $O 2>>gpurun_out/ab_conv4.err
echo DONE
