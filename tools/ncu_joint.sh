#!/bin/bash
# ncu of the C4 conv forward with and without joint chunk emission
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -c 1 -s 1"
timeout 400 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/full_c4_convfwd_nojoint python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32 --iters 2 > /dev/null 2>&1
CGF_GEN=joint timeout 400 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/full_c4_convfwd_joint python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32 --iters 2 > /dev/null 2>&1
