#!/bin/bash
# A/B sweep of generator variants (CGF_GEN) on one GPU. Output: gpurun_out/ab_*.jsonl
mkdir -p gpurun_out
for v in "" "nobarrier" "yreg" "yreg,nobarrier" "depth=5" "warps=8" "nobarrier,depth=5,warps=8"; do
  tag=$(echo "base$v" | tr ',=' '__')
  CGF_GEN="$v" timeout 300 python tools/sweep.py --configs c2 --dtypes f32 --iters 3 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_tp.jsonl 2>&1
done
for v in "" "nobarrier" "depth=6" "depth=8,warps=8" "warps=2,depth=8"; do
  CGF_GEN="$v" timeout 300 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32 --iters 2 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_conv.jsonl 2>&1
done
