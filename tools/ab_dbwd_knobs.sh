#!/bin/bash
# double-backward / FP64 kernels: register caps and ring depth
O=gpurun_out/ab_dbwd_knobs.jsonl; : > $O
for v in "" "minb=2" "minb=3" "minb=4" "depth=1" "depth=2"; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32,f64 --modes det --iters 2 >> $O 2>>gpurun_out/ab_dbwd_knobs.err
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --ops dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_dbwd_knobs.err
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c5 --ops bwd --dtypes f64 --modes det --iters 2 >> $O 2>>gpurun_out/ab_dbwd_knobs.err
done
echo DONE
