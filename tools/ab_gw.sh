#!/bin/bash
# gW kernel bound: CGF_UVW_EXP 16 = no MMAs, 32 = producers skip z' (timing only)
for e in 0 16 32 48; do
  echo "== EXP=$e"
  CGF_UVW_EXP=$e timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cgf_uvw_bwdw[06]_f32$ python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "^  cgf_uvw|duration"
done
