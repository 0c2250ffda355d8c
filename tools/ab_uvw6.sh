#!/bin/bash
# (1) gW kernel bound after the staging fix: EXP 16 = no MMAs, 32 = no producer math
# (2) forward rings: x tiles (CGF_UVW_NX), W images (CGF_UVW_NW)
for e in 0 16 32; do
  echo "== gW EXP=$e"
  CGF_UVW_EXP=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_bwdw[06]_f32$ python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -2
done
for cfg in "NX=3 NW=6" "NX=2 NW=6" "NX=4 NW=4" "NX=3 NW=4" "NX=3 NW=8"; do
  echo "== fwd $cfg"
  env $(echo $cfg | sed 's/\([A-Z]*\)=/CGF_UVW_\1=/g') timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_fwd_f32$ python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 2>&1 | grep -E "duration" | tail -1
done
