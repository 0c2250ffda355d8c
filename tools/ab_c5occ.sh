#!/bin/bash
# C5 conv backward / forward occupancy knobs (registers vs warps)
O=gpurun_out/ab_c5occ.jsonl; : > $O
for v in "" "minb=4" "minb=2" "" "minb=4"; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c5 --ops fwd,bwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_c5occ.err
done
for v in "" "minb=4" "minb=3"; do
  CGF_GEN="$v" timeout 900 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f32 --modes det --iters 3 >> $O 2>>gpurun_out/ab_c5occ.err
done
echo DONE
