#!/bin/bash
# C2 FP64 batched backward at the bench size: ring depth
O=gpurun_out/ab_f64bwd.jsonl; : > $O
for v in "" "depth=1" "" "depth=1"; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --ops bwd --dtypes f64 --rows 1000000 --iters 3 >> $O 2>>gpurun_out/ab_f64bwd.err
done
echo DONE
