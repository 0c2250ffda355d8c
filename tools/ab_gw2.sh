#!/bin/bash
# gW staging depths: CGF_UVW_NGZ (gz^T tiles), CGF_UVW_NXB (x segments)
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_gw2.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_gw2.log
for cfg in "NGZ=2 NXB=2" "NGZ=4 NXB=2" "NGZ=6 NXB=2" "NGZ=4 NXB=3" "NGZ=6 NXB=3" "NGZ=8 NXB=2"; do
  echo "== $cfg"
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_bwdw[06]_f32$ python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -2
done
