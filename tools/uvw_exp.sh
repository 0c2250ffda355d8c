#!/bin/bash
# uvw forward experiment knobs (CGF_UVW_EXP bitmask), timing only
for e in 0 1 2 4 3 7; do
  echo -n "EXP=$e "; CGF_UVW_EXP=$e timeout 100 python tools/sweep.py --configs c3 --dtypes f32 --w-shared --ops fwd --iters 5 2>&1 | grep -o '"ms": [0-9.]*'
done
