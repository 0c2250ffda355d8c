"""C2 FP32 forward timing alone vs interleaved with the backward (the bench step):
is the in-step forward slower because of the interleaving or because of power?"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402

plan = cgf.TpPlan(config_json("c2"))
R = 1_000_000
g = torch.Generator(device="cuda").manual_seed(1)
x, y, w, gz = (torch.randn((R, d), device="cuda", generator=g) for d in (plan.dim_x, plan.dim_y, plan.n_w, plan.dim_z))
z = torch.empty((R, plan.dim_z), device="cuda")
grads = plan.backward(x, y, w, gz)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def fwd():
    plan.forward(x, y, w, z=z)


def bwd():
    plan.backward(x, y, w, gz, out=grads)


out = {}
for name, seq in (("fwd_alone", [fwd] * 20), ("bwd_alone", [bwd] * 20), ("interleaved", [fwd, bwd] * 10),
                  ("fwd_alone_again", [fwd] * 20)):
    for f in seq[:4]:
        f()
    torch.cuda.synchronize()
    times = {"fwd": [], "bwd": []}
    for f in seq:
        a = ev()
        f()
        b = ev()
        torch.cuda.synchronize()
        times["fwd" if f is fwd else "bwd"].append(a.elapsed_time(b))
    out[name] = {k: round(sum(v) / len(v), 3) for k, v in times.items() if v}
print(json.dumps(out))
