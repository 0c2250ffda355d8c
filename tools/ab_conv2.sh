#!/bin/bash
# Occupancy knobs for the conv kernels (CGF_GEN): chunk merging, min blocks
# per SM, ring depth, warps per CTA; with / without unit groups.
mkdir -p gpurun_out
O=gpurun_out/ab_conv2.jsonl; : > $O
for F in "" merge=1 minb=3 merge=1,minb=4 depth=3 warps=8 merge=1,warps=8; do
  for G in 1 2; do
    CGF_CONVI_GROUPS=$G CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_conv2.err
  done
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_conv2.err
done
echo DONE
