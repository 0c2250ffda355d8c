"""Minimal launcher for ncu: runs `--iters` launches of one TP op (no other
kernels between them except input generation up front).

    ncu --set full -k regex:cgf_tp -s 1 -c 1 -o gpurun_out/prof python tools/prof_tp.py --config c2 --op bwd
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--op", default="fwd")
ap.add_argument("--dtype", default="f32")
ap.add_argument("--rows", type=int, default=262_144)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--w-shared", action="store_true")
a = ap.parse_args()
plan = cgf.TpPlan(config_json(a.config))
tdt = torch.float32 if a.dtype == "f32" else torch.float64
R = a.rows
nw = 1 if a.w_shared else R
t = lambda *s: torch.randn(s, device="cuda", dtype=tdt)
x, y, w, gz = t(R, plan.dim_x), t(R, plan.dim_y), t(nw, plan.n_w), t(R, plan.dim_z)
up = (t(R, plan.dim_x), t(R, plan.dim_y), t(nw, plan.n_w))
for _ in range(a.iters):
    if a.op == "fwd":
        plan.forward(x, y, w, w_shared=a.w_shared)
    elif a.op == "bwd":
        plan.backward(x, y, w, gz, w_shared=a.w_shared)
    else:
        plan.double_backward(x, y, w, gz, up, w_shared=a.w_shared)
torch.cuda.synchronize()
print("done", a)
