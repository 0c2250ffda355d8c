#!/bin/bash
# staging issue: parallel bulk (pbulk, FP32 forward default) vs lane-0 bulk copies (bulk) vs lane cp.async (lanecopy,nopbulk)
O=gpurun_out/ab_bulk.jsonl; : > $O
for v in "" "bulk,nopbulk" "" "bulk,nopbulk"; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --dtypes f32 --ops fwd,bwd --iters 5 >> $O 2>>gpurun_out/ab_bulk.err
done
echo DONE
