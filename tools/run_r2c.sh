#!/bin/bash
# GPU call: full parity suite, backward row-group sweep, ncu of the grouped kernels.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r2c.log 2>&1; echo PYTEST_EXIT $?
tail -15 gpurun_out/pytest_r2c.log
O=gpurun_out/sweep_rowbwd.jsonl; : > $O
for G in 1 2 3 4; do
  CGF_ROW_GROUPS_BWD=$G timeout 600 python tools/sweep.py --configs c2 --ops bwd --dtypes f32,f64 --iters 3 >> $O 2>>gpurun_out/sweep_rowbwd.err
done
P="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $P -k regex:cgf_convi_bwd_f64_g3of8 -o gpurun_out/full_c4_f64_convbwd_g python tools/sweep_conv.py --cases c4 --ops bwd --dtypes f64 --iters 1 > gpurun_out/ncu_c4bwd.log 2>&1
timeout 600 $P -k regex:cgf_tp_dbwd_f32_g2of6 -o gpurun_out/full_c2_f32_dbwd_g python tools/prof_tp.py --config c2 --op dbwd --rows 1000000 > gpurun_out/ncu_c2dbwd.log 2>&1
timeout 600 $P -k regex:cgf_tp_bwd_f64 -o gpurun_out/full_c2_f64_bwd python tools/prof_tp.py --config c2 --op bwd --dtype f64 --rows 400000 > gpurun_out/ncu_c2bwd64.log 2>&1
echo DONE
