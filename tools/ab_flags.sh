#!/bin/bash
# A/B of generator flags (CGF_GEN): L2 eviction hints in the conv loops
# (l2hint), x chunks / y in registers once per item (xregs, yitem).
mkdir -p gpurun_out
O=gpurun_out/ab_flags.jsonl; : > $O
for F in "" l2hint xregs,yitem l2hint,xregs,yitem; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_flags.err
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_flags.err
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2 --ops fwd,bwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_flags.err
done
echo DONE
