#!/bin/bash
# gW staging depths, round 2: z' stages (CGF_UVW_NZS) with 5-6 gz^T stages
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_gw3.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_gw3.log
for cfg in "NGZ=6 NZS=2" "NGZ=6 NZS=3" "NGZ=5 NZS=3" "NGZ=4 NZS=4"; do
  echo "== $cfg"
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_bwd python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "^  cgf|duration" | tail -16
done
python tools/sweep.py --configs c3 --w-shared --ops bwd --dtypes f32 --iters 5 2>/dev/null | tail -1
