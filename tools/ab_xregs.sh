#!/bin/bash
# A/B of generator flags (CGF_GEN) on the conv and TP kernels: x chunks in
# registers once per item (xregs), y in registers once per item (yitem).
mkdir -p gpurun_out
O=gpurun_out/ab_xregs.jsonl; : > $O
for F in "" xregs yitem xregs,yitem; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_xregs.err
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_xregs.err
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2 --ops fwd,bwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_xregs.err
done
echo DONE
