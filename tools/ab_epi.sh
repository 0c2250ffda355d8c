#!/bin/bash
# Multi-edge items (CGF_GEN=epi=N) for the by-output conv kernels: parity, then timing.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider -k "multi_edge or single_edge or grouped" > gpurun_out/pytest_epi.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_epi.log
O=gpurun_out/ab_epi.jsonl; : > $O
for E in 1 2 3 4; do
  CGF_GEN=epi=$E timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops fwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_epi.err
done
echo DONE
