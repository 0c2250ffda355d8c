#!/bin/bash
# uvw forward: loaders' / epilogue's waits suspended in try_wait (CGF_UVW_NC_SLEEP ns) instead of spinning
python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 > gpurun_out/pt_ncs.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_ncs.log
for v in 0 500 2000 10000 0 2000; do
  echo "== NC_SLEEP=$v"
  CGF_UVW_NC_SLEEP=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cgf_uvw_(fwd|bwdx)_f32$" python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
done
