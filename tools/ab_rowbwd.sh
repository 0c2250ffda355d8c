#!/bin/bash
# conv backward traversal: by neighbour (default) vs row order (CGF_CONV_BWD=row:
# CSR-order edges, per-edge g_node_x partials + segmented sum)
mkdir -p gpurun_out
CGF_CONV_BWD=row timeout 900 python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider -x > gpurun_out/pytest_rowbwd.log 2>&1; echo PYTEST_EXIT $?; tail -3 gpurun_out/pytest_rowbwd.log
O=gpurun_out/ab_rowbwd.jsonl; : > $O
for v in nbr row; do
  CGF_CONV_BWD=$v timeout 900 python tools/sweep_conv.py --cases c4,c5 --ops bwd --dtypes f32,f64 --modes det >> $O 2>>gpurun_out/ab_rowbwd.err
done
echo DONE
