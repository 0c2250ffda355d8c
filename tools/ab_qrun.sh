#!/bin/bash
# uvw producers: CG.y coefficients once per instruction run (CGF_UVW_QRUN=1, default) vs per unit
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_qrun.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_qrun.log
for v in 0 1 0 1; do
  echo "== QRUN=$v"
  CGF_UVW_QRUN=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cgf_uvw_(fwd|bwdx)_f32$" python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
  CGF_UVW_QRUN=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cgf_uvw_bwdx_f32$" python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
done
