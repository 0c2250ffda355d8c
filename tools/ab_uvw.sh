#!/bin/bash
# uvw forward producer configurations (CGF_UVW_PW producer warps, CGF_UVW_NX x ring, CGF_UVW_NW W ring)
mkdir -p gpurun_out
O=gpurun_out/ab_uvw.jsonl; : > $O
for cfg in "PW=8" "PW=4" "PW=16" "PW=4 NX=4" "PW=8 NX=4"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 600 python tools/sweep.py --configs c3 --w-shared --ops fwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw.err
done
CGF_UVW_PW=4 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pytest_uvw.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pytest_uvw.log
echo DONE
O=gpurun_out/ab_tpocc.jsonl; : > $O
for F in "" minb=3 minb=3,depth=3 depth=3 warps=8; do
  CGF_GEN=$F timeout 600 python tools/sweep.py --configs c2 --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw.err
done
echo DONE2
