#!/bin/bash
# TP kernels: __launch_bounds__ min blocks per SM (register cap) sweep
O=gpurun_out/ab_minb.jsonl; : > $O
for v in "" "minb=2" "minb=3" "minb=4"; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --dtypes f32,f64 --ops fwd,bwd --iters 3 >> $O 2>>gpurun_out/ab_minb.err
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c1 --dtypes f32,f64 --ops fwd,bwd --iters 3 >> $O 2>>gpurun_out/ab_minb.err
done
echo DONE
