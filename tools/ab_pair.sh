#!/bin/bash
# Edge-pair emission for the by-output forward (CGF_GEN=pairedges): parity, timing.
mkdir -p gpurun_out
CGF_GEN=pairedges python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pytest_pair.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_pair.log
O=gpurun_out/ab_pair.jsonl; : > $O
for F in "" pairedges; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops fwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_pair.err
done
echo DONE
