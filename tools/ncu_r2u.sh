#!/bin/bash
# ncu --set full of the SIMT kernels after the multi-value warp sums (SASS histograms, stalls)
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -c 1 -s 1"
timeout 400 $P -k regex:cgf_convi_bwd_f64_g3 -o gpurun_out/u_c4_f64_convbwd python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f64 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convi_bwd_f32 -o gpurun_out/u_c4_f32_convbwd python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/u_c4_f32_convfwd python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convi_dbwdx_f32_g0 -o gpurun_out/u_c4_f32_dbwdx python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convo_dbwdz_f32 -o gpurun_out/u_c4_f32_dbwdz python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convi_bwd_f32 -o gpurun_out/u_c5_f32_convbwd python tools/sweep_conv.py --cases c5 --ops bwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convo_fwd_f32 -o gpurun_out/u_c5_f32_convfwd python tools/sweep_conv.py --cases c5 --ops fwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 300 $P -k regex:cgf_tp_dbwd_f32_g0 -o gpurun_out/u_c2_f32_dbwd python tools/prof_tp.py --config c2 --op dbwd --rows 1000000 > /dev/null 2>&1
timeout 300 $P -k regex:cgf_tp_bwd_f64 -o gpurun_out/u_c2_f64_bwd python tools/prof_tp.py --config c2 --op bwd --dtype f64 --rows 400000 > /dev/null 2>&1
ls -la gpurun_out/u_*.ncu-rep
