#!/bin/bash
# gz planes pre-pass: 16 vs 32 batch rows per block (CGF_UVW_PLANE_ROWS)
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_planes.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_planes.log
for v in 32 16 32 16; do
  echo "== PLANE_ROWS=$v"
  CGF_UVW_PLANE_ROWS=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cgf_uvw_bwd_planes python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration|dram" | tail -3
done
