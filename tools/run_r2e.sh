#!/bin/bash
# ncu captures for SASS-level instruction histograms (tools/ncu_sass_hist.py)
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/full_c4_f32_convfwd python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_convi_bwd_f32 -o gpurun_out/full_c4_f32_convbwd python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_convi_bwd_f32 -o gpurun_out/full_c5_f32_convbwd python tools/sweep_conv.py --cases c5 --ops bwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/full_c5_f32_convfwd python tools/sweep_conv.py --cases c5 --ops fwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_convi_dbwdx_f32_g0 -o gpurun_out/full_c4_f32_dbwdx python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_convo_dbwdz_f32 -o gpurun_out/full_c4_f32_dbwdz python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32 --iters 1 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_uvw_fwd_f32 -o gpurun_out/full_c3_f32_uvwfwd python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_uvw_bwdy -o gpurun_out/full_c3_f32_uvwbwdy python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 > /dev/null 2>&1
timeout 600 $P -k regex:cgf_tp_bwd_f32 -o gpurun_out/full_c2_f32_bwd2 python tools/prof_tp.py --config c2 --op bwd --rows 1000000 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
echo DONE
