"""Debug probe for the tcgen05 uvw path: one small forward, compared with the SIMT path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_13986_b200 as cgf  # noqa: E402
from oracle.oracle import config_json  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1
plan = cgf.TpPlan(config_json("c3"))
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randn((rows, plan.dim_x), device="cuda", generator=g)
y = torch.randn((rows, plan.dim_y), device="cuda", generator=g)
w = torch.randn((1, plan.n_w), device="cuda", generator=g)
os.environ["CGF_UVW"] = "0"
ref = plan.forward(x, y, w, w_shared=True)
torch.cuda.synchronize()
os.environ["CGF_UVW"] = "1"
print("launching uvw", rows, flush=True)
z = plan.forward(x, y, w, w_shared=True)
torch.cuda.synchronize()
err = ((z - ref).norm() / ref.norm()).item()
print("rows", rows, "rel err vs SIMT", err, flush=True)
print("z[0,:8]", z[0, :8].tolist(), "\nref", ref[0, :8].tolist())
