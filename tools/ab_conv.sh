#!/bin/bash
# A/B of generator variants on the C4 conv: args are CGF_GEN variant strings
for v in "$@"; do
  CGF_GEN="$v" timeout 400 python tools/sweep_conv.py --cases c4 --ops ${OPS:-fwd,bwd} --dtypes ${DT:-f32} --iters 2 2>&1 | sed "s/^{/{\"variant\": \"$v\", /" | grep -o '"variant": "[^"]*".*"op": "[a-z]*".*"dtype": "[a-z0-9]*".*"ms": [0-9.]*'
done
