#!/bin/bash
# A/B of uvw generator knobs; each argument is "PW NX NW" (producer warps, x ring, W ring)
for cfg in "$@"; do
  set -- $cfg
  echo "=== PW=$1 NX=$2 NW=$3"
  export CGF_UVW_PW=$1 CGF_UVW_NX=$2 CGF_UVW_NW=$3
  timeout 60 python tools/uvw_probe.py 5000 2>&1 | grep -E "rel err" | cut -c1-100
  timeout 100 python tools/sweep.py --configs c3 --dtypes f32 --w-shared --ops fwd --iters 5 2>&1 | cut -c1-200
done
