#!/bin/bash
# uvw forward: staged coalesced epilogue (CGF_UVW_EPI=1) and the bottleneck knobs (CGF_UVW_EXP)
mkdir -p gpurun_out
CGF_UVW_EPI=1 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pytest_uvw2.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pytest_uvw2.log
O=gpurun_out/ab_uvw2.jsonl; : > $O
for cfg in "EPI=0" "EPI=1" "EXP=1" "EXP=2" "EXP=4" "EXP=6" "EPI=1 EXP=2" "EPI=1 EXP=4"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 600 python tools/sweep.py --configs c3 --w-shared --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw2.err
done
echo DONE
