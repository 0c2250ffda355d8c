#!/bin/bash
# staged output stores: compile-time-unrolled lane loops (default) vs runtime loops (CGF_GEN=loopstores)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tp.py tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pt_ustore.log 2>&1; echo PYTEST_EXIT $?; tail -1 gpurun_out/pt_ustore.log
O=gpurun_out/ab_ustore.jsonl; : > $O
for v in loopstores "" loopstores ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --dtypes f32 --ops fwd,bwd,dbwd --iters 5 >> $O 2>>gpurun_out/ab_ustore.err
done
for v in loopstores ""; do
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c2 --dtypes f64 --ops fwd,bwd,dbwd --iters 3 >> $O 2>>gpurun_out/ab_ustore.err
  CGF_GEN="$v" timeout 900 python tools/sweep.py --configs c1 --dtypes f32,f64 --ops fwd,bwd,dbwd --iters 3 >> $O 2>>gpurun_out/ab_ustore.err
  CGF_GEN="$v" timeout 1500 python tools/sweep_conv.py --cases c4,c5 --ops fwd,bwd,dbwd --dtypes f32 --modes det >> $O 2>>gpurun_out/ab_ustore.err
  CGF_GEN="$v" timeout 1500 python tools/sweep_conv.py --cases c4 --ops fwd,bwd --dtypes f64 --modes det >> $O 2>>gpurun_out/ab_ustore.err
done
echo DONE
