#!/bin/bash
# uvw: unit order within a segment (CGF_UVW_ORDER=1: channel-block-major) and
# the A-ring depth (CGF_UVW_NA), plus per-role wait counters (CGF_UVW_PROF)
mkdir -p gpurun_out
CGF_UVW_ORDER=1 CGF_UVW_NA=6 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pytest_uvw4.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pytest_uvw4.log
O=gpurun_out/ab_uvw4.jsonl; : > $O
for cfg in "ORDER=0" "ORDER=1" "NA=5" "NA=6" "ORDER=1 NA=5" "ORDER=1 NA=6" "ORDER=0"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 600 python tools/sweep.py --configs c3 --w-shared --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw4.err
done
for cfg in "ORDER=0" "ORDER=1" "ORDER=1 NA=6"; do
  echo "== PROF $cfg" >> gpurun_out/ab_uvw4_prof.txt
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') CGF_UVW_PROF=1 timeout 300 python tools/sweep.py --configs c3 --w-shared --ops fwd --dtypes f32 --iters 1 2>&1 | tail -12 >> gpurun_out/ab_uvw4_prof.txt
done
echo DONE
