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
d = (z - ref).abs()
rowerr = d.max(dim=1).values / ref.abs().max()
bad_rows = torch.nonzero(rowerr > 1e-4).flatten()
print("bad rows:", bad_rows.numel(), "of", rows, "first:", bad_rows[:140].tolist())
if rows >= 128:
    m = torch.arange(rows, device=z.device) % 128
    per_m = torch.zeros(128, device=z.device).index_reduce_(0, m, rowerr, "amax")
    print("bad m (row % 128):", torch.nonzero(per_m > 1e-4).flatten().tolist())
colerr = d.max(dim=0).values / ref.abs().max()
bc = torch.nonzero(colerr > 1e-4).flatten().tolist()
print("bad cols:", len(bc), "segments (0-63 | 64-255 | 256-575):", sum(c < 64 for c in bc), sum(64 <= c < 256 for c in bc), sum(c >= 256 for c in bc))
if bad_rows.numel():
    r0 = bad_rows[0].item()
    e = (d[r0] / ref.abs().max()).tolist()
    print("row", r0, "err by col group of 8:", [round(max(e[i:i+8]), 4) for i in range(0, len(e), 8)])
