#!/bin/bash
# ncu --set full of the C3 shared-W backward kernels (gW pass 0, gy, gx) and the forward
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -s 1 -c 1"
timeout 600 $P -k regex:cgf_uvw_bwdw0_f32$ -o gpurun_out/full_c3_f32_bwdw0 python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 > gpurun_out/ncu_c3bwdw.log 2>&1
timeout 600 $P -k regex:cgf_uvw_bwdx_f32$ -o gpurun_out/full_c3_f32_bwdx python tools/prof_tp.py --config c3 --op bwd --w-shared --rows 1000000 > gpurun_out/ncu_c3bwdx.log 2>&1
timeout 600 $P -k regex:cgf_uvw_fwd_f32$ -o gpurun_out/full_c3_f32_fwd python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 > gpurun_out/ncu_c3fwd.log 2>&1
echo DONE
