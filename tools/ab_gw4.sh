#!/bin/bash
# gW kernel knock-outs: 64 = no x TMA, 128 = no gz TMA, 16 = no MMAs, 32 = no producer math (timing only)
for e in 0 64 128 192 240; do
  echo "== gW EXP=$e"
  CGF_UVW_EXP=$e timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:cgf_uvw_bwdw[06]_f32$ python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 2>&1 | grep -E "duration|dram" | tail -4
done
