#!/bin/bash
# Paired FP32 emission (CGF_GEN=joint,ffma2): parity of the TP and conv suites
# with it forced on, then timing against the default and joint-only.
mkdir -p gpurun_out
CGF_GEN=joint,ffma2 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pytest_ffma2.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_ffma2.log
O=gpurun_out/ab_ffma2.jsonl; : > $O
for F in "" joint joint,ffma2; do
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2 --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_ffma2.err
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_ffma2.err
done
echo DONE
