#!/bin/bash
# One `ncu --set full` capture per benchmark kernel (1 launch each, after a
# warm-up launch) + the launch list of a short bench run. Outputs under
# gpurun_out/; tools/ncu_traffic.py turns them into profiles/ncu_traffic.json.
set -x
mkdir -p gpurun_out
P="ncu --set full --clock-control none --import-source on -s 1 -c 1"
timeout 600 $P -k regex:cgf_tp_fwd_f32 -o gpurun_out/full_c2_f32_fwd python tools/prof_tp.py --config c2 --op fwd --rows 1000000 > gpurun_out/ncu_c2fwd.log 2>&1
timeout 600 $P -k regex:cgf_tp_bwd_f32 -o gpurun_out/full_c2_f32_bwd python tools/prof_tp.py --config c2 --op bwd --rows 1000000 > gpurun_out/ncu_c2bwd.log 2>&1
timeout 600 $P -k regex:cgf_uvw_fwd -o gpurun_out/full_c3_f32_fwd python tools/prof_tp.py --config c3 --op fwd --w-shared --rows 1000000 > gpurun_out/ncu_c3fwd.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --conv-steps 1 --leg-steps 1 > gpurun_out/ncu_bench.log 2>&1
