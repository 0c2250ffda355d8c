#!/bin/bash
# gy kernel staging: half-tile gz ring depth (CGF_UVW_GY_NGH) and x ring (CGF_UVW_GY_NX)
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_gy.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_gy.log
for cfg in "GY_NGH=2 GY_NX=2" "GY_NGH=3 GY_NX=2" "GY_NGH=2 GY_NX=3" "GY_NGH=4 GY_NX=1"; do
  echo "== $cfg"
  env $(echo $cfg | sed 's/\([A-Z_]*\)=/CGF_UVW_\1=/g') timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_bwdy_f32$ python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
done
python tools/sweep.py --configs c3 --w-shared --ops bwd --dtypes f32 --iters 5 2>/dev/null | tail -1
