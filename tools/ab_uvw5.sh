#!/bin/bash
# uvw producers: x-slot release after the unit (CGF_UVW_XREL=1), per-thread
# arrives without __syncwarp (CGF_UVW_ARV=1); EXP=8 (no proxy fence) is timing only
mkdir -p gpurun_out
CGF_UVW_XREL=1 CGF_UVW_ARV=1 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pytest_uvw5.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pytest_uvw5.log
O=gpurun_out/ab_uvw5.jsonl; : > $O
for cfg in "XREL=0" "XREL=1" "ARV=1" "XREL=1 ARV=1" "EXP=8" "XREL=0"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 600 python tools/sweep.py --configs c3 --w-shared --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw5.err
done
echo DONE
