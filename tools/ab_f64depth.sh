#!/bin/bash
# FP64: new depth defaults (dbl-bwd family, by-neighbour backward) + TP fwd / bwd ring depth A/B
timeout 1800 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pt_f64d.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_f64d.log
O=gpurun_out/ab_f64depth.jsonl; : > $O
timeout 900 python tools/sweep_conv.py --cases c4 --ops dbwd --dtypes f64 --modes det --iters 2 >> $O 2>>gpurun_out/ab_f64depth.err
timeout 900 python tools/sweep_conv.py --cases c5 --ops bwd --dtypes f64 --modes det --iters 2 >> $O 2>>gpurun_out/ab_f64depth.err
timeout 900 python tools/sweep.py --configs c2,c1 --ops dbwd --dtypes f64 --iters 3 >> $O 2>>gpurun_out/ab_f64depth.err
for v in "" "depth=1" "depth=2" "depth=3"; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2,c1 --ops fwd,bwd --dtypes f64 --iters 3 >> $O 2>>gpurun_out/ab_f64depth.err
done
echo DONE
