#!/bin/bash
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -c 1"
timeout 300 $P -k regex:cgf_tp_bwd_f64 -s 1 -o gpurun_out/full_c2_f64_bwd python tools/prof_tp.py --config c2 --op bwd --dtype f64 --rows 200000 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convo_fwd_f32 -s 1 -o gpurun_out/full_c4_f32_convfwd python tools/sweep_conv.py --cases c4 --ops fwd --dtypes f32 --iters 2 > /dev/null 2>&1
timeout 400 $P -k regex:cgf_convi_bwd_f64 -s 1 -o gpurun_out/full_c4_f64_convbwd python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f64 --iters 2 > /dev/null 2>&1
