#!/bin/bash
# C2 FP32 batched double-backward: ring depth, register cap, group count combinations
O=gpurun_out/ab_c2dbwd.jsonl; : > $O
run() { env $1 CGF_GEN="$2" timeout 600 python tools/sweep.py --configs c2 --ops dbwd --dtypes f32 --iters 5 | sed "s/^{/{\"groups\": \"$1\", /" >> $O 2>>gpurun_out/ab_c2dbwd.err; }
run "X=0" ""
run "X=0" "depth=2"
run "X=0" "depth=3"
run "CGF_ROW_GROUPS=4" "depth=2"
run "CGF_ROW_GROUPS=3" "depth=2"
run "CGF_ROW_GROUPS=8" "depth=2"
run "X=0" "depth=2,minb=3"
run "X=0" "depth=2,nobarrier"
run "X=0" ""
run "X=0" "depth=2"
echo DONE
