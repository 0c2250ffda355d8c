"""e2e host-path sweep: TpPlan.forward_backward on pinned host arrays (C2
FP32, 131072 rows) for each CGF_HOST_CHUNK_MB / CGF_HOST_DEPTH setting given
on the command line (chunk MB : depth [: ramp 0/1, CGF_HOST_RAMP]), host
wall clock, best of 5.

    python tools/e2e_sweep.py 64:3 128:3 256:3 128:4 256:4 256:3:0
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402

plan = cgf.TpPlan(config_json("c2"))
R = 131_072
pin = lambda *s: torch.randn(s).pin_memory()
ins = [pin(R, d).numpy() for d in (plan.dim_x, plan.dim_y, plan.n_w, plan.dim_z)]
outs = tuple(torch.empty(R, d).pin_memory().numpy() for d in (plan.dim_z, plan.dim_x, plan.dim_y, plan.n_w))
nbytes = sum(a.nbytes for a in ins) + sum(a.nbytes for a in outs)
for spec in sys.argv[1:] or ["128:3"]:
    mb, depth, *rest = spec.split(":")
    ramp = rest[0] if rest else "1"
    os.environ["CGF_HOST_CHUNK_MB"], os.environ["CGF_HOST_DEPTH"], os.environ["CGF_HOST_RAMP"] = mb, depth, ramp
    plan.forward_backward(*ins, out=outs)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        plan.forward_backward(*ins, out=outs)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * min(ts)
    print(json.dumps({"chunk_mb": int(mb), "depth": int(depth), "ramp": int(ramp), "ms": ms, "GB/s_both_dirs": nbytes / ms / 1e6,
                      "GFLOP/s": (plan.flops_fwd + plan.flops_bwd) * R / ms / 1e6}), flush=True)
