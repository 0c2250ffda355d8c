#!/bin/bash
# A/B sweep of generator variants (CGF_GEN) on one GPU. Output: gpurun_out/ab_*.jsonl
mkdir -p gpurun_out
TPV=${TPV:-" |nobarrier|yreg|minb=1|warps=8|depth=2"}
CV=${CV:-" |nobarrier|minb=1|depth=6|warps=8"}
IFS='|'
for v in $TPV; do
  v=$(echo $v | xargs)
  CGF_GEN="$v" timeout 400 python tools/sweep.py --configs ${TPCFG:-c2} --dtypes ${TPDT:-f32} --iters 3 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_tp.jsonl 2>&1
done
for v in $CV; do
  v=$(echo $v | xargs)
  CGF_GEN="$v" timeout 400 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32 --iters 2 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/ab_conv.jsonl 2>&1
done
