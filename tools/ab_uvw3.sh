#!/bin/bash
# uvw: software-pipelined TMEM A stores (CGF_UVW_PIPE=1)
mkdir -p gpurun_out
CGF_UVW_PIPE=1 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pytest_uvw3.log 2>&1; echo PYTEST_EXIT $?; tail -2 gpurun_out/pytest_uvw3.log
O=gpurun_out/ab_uvw3.jsonl; : > $O
for cfg in "PIPE=0" "PIPE=1" "PIPE=1 NX=4" "PIPE=1 EXP=4" "PIPE=0 EXP=4"; do
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 600 python tools/sweep.py --configs c3 --w-shared --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_uvw3.err
done
echo DONE
