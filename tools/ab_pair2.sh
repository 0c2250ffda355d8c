#!/bin/bash
# Edge-pair emission for the by-neighbour backward (CGF_GEN=pairedges): parity, timing.
mkdir -p gpurun_out
CGF_GEN=pairedges python -m pytest tests/test_gpu_conv.py tests/test_gpu_dist.py -q -p no:cacheprovider -x > gpurun_out/pytest_pair2.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_pair2.log
O=gpurun_out/ab_pair2.jsonl; : > $O
for F in "" pairedges pairedges,warps=2 pairedges,warps=8; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_pair2.err
done
echo DONE
