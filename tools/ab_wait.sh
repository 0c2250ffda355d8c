#!/bin/bash
# A/B: mbarrier waits with a suspend-time hint (uvw kernels: always on in this
# build; SIMT consumers: CGF_GEN=waitsleep).
mkdir -p gpurun_out
O=gpurun_out/ab_wait.jsonl; : > $O
timeout 900 python tools/sweep.py --configs c3 --w-shared --ops fwd,bwd --dtypes f32 --iters 5 >> $O 2>>gpurun_out/ab_wait.err
for F in "" waitsleep; do
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd,dbwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_wait.err
  CGF_GEN=$F timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --iters 3 >> $O 2>>gpurun_out/ab_wait.err
  CGF_GEN=$F timeout 900 python tools/sweep.py --configs c2 --ops fwd,bwd,dbwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/ab_wait.err
done
P="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $P -k regex:cgf_uvw_fwd_f32 -o gpurun_out/full_c3_f32_uvwfwd2 python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 > /dev/null 2>&1
echo DONE
