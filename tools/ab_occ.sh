#!/bin/bash
# Occupancy sweep for the small-TP (C5) conv kernels: ring depth x warps, with / without edge pairs.
mkdir -p gpurun_out
O=gpurun_out/ab_occ.jsonl; : > $O
for F in "" depth=1 depth=1,warps=8 depth=1,minb=4 depth=1,minb=5 pairedges,warps=8 pairedges,depth=1,warps=4 pairedges,depth=1,minb=3 pairedges,warps=6 pairedges,warps=2,depth=1; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd,dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_occ.err
done
for F in "" depth=1 depth=1,warps=8; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_occ.err
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2,c1 --ops fwd,bwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_occ.err
done
echo DONE
