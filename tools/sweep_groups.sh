#!/bin/bash
# Group-count sweeps (run on the GPU box): the by-neighbour conv kernels
# (CGF_CONVI_GROUPS, C4 / C5 backward and double-backward), the batched
# double-backward (CGF_ROW_GROUPS, C2), and the host pipeline (chunk size,
# depth) of the e2e path. One JSON line per measurement.
mkdir -p gpurun_out
O=gpurun_out/sweep_groups.jsonl
: > $O
for G in 1 2 3 4 6 8; do
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c4 --ops bwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups.err
done
for G in 1 2 3; do
  CGF_CONVI_GROUPS=$G timeout 900 python tools/sweep_conv.py --cases c5 --ops bwd,dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/sweep_groups.err
done
for G in 1 2 3 4 6; do
  CGF_ROW_GROUPS=$G timeout 900 python tools/sweep.py --configs c2,c1 --ops dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/sweep_groups.err
done
timeout 600 python tools/e2e_sweep.py 32:3 64:3 128:3 256:3 512:3 64:4 128:4 256:4 128:2 >> gpurun_out/sweep_e2e.jsonl 2>>gpurun_out/sweep_groups.err
