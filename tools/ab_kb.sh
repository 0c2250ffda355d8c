#!/bin/bash
# uvw forward producers re-checked with the current handshakes: 2 A blocks per TMEM-store round (KB), pipelined stores (PIPE)
for cfg in "KB=1" "KB=2" "PIPE=1" "KB=1" "KB=2"; do
  echo "== $cfg"
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cgf_uvw_fwd_f32$" python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
done
CGF_UVW_KB=2 python -m pytest tests/test_gpu_tp.py -q -p no:cacheprovider -k c3 2>&1 | tail -1
