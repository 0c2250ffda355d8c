#!/bin/bash
# conv knob re-check after the round-2 generator changes: edges per item, register caps, ring depth
O=gpurun_out/ab_conv3.jsonl; : > $O
for v in "" "epi=3" "epi=4" "epi=1" ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32,f64 --modes det --iters 3 >> $O 2>>gpurun_out/ab_conv3.err
done
for v in "" "minb=2" "minb=3" "depth=2" "depth=1"; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f64 --modes det --iters 2 >> $O 2>>gpurun_out/ab_conv3.err
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f64 --modes det --iters 3 >> $O 2>>gpurun_out/ab_conv3.err
done
echo DONE
