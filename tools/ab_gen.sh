#!/bin/bash
# A/B of SIMT generator variants (CGF_GEN) on the C2 TP: args are variant strings
for v in "$@"; do
  CGF_GEN="$v" timeout 300 python tools/sweep.py --configs ${CFG:-c2} --dtypes ${DT:-f32} --ops ${OPS:-fwd,bwd} --iters 3 2>&1 | sed "s/^{/{\"variant\": \"$v\", /" | cut -c1-220
done
