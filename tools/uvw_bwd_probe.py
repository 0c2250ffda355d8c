"""Debug probe for the tcgen05 uvw backward (shared W): gx / gy / gW against the oracle on a row sample."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_13986_b200 as cgf  # noqa: E402
from oracle import oracle as O  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 300
js = O.config_json("c3")
o, plan = O.Oracle(js), cgf.TpPlan(js)
x, y, w = O.random_batch(o, rows, 7, np.float32, w_shared=True)
gz = O.NormalGen(8).normal_vec(rows * o.dim_z, np.float32).reshape(rows, -1)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
gx, gy, gw = plan.backward(d(x), d(y), d(w), d(gz), w_shared=True)
torch.cuda.synchronize()
wx, wy, ww = o.backward(x, y, w, gz, w_shared=True)
for n, a, b in (("gx", gx, wx), ("gy", gy, wy), ("gW", gw, ww)):
    print(n, "rel err", O.rel_error(a.cpu().numpy().reshape(b.shape), b), flush=True)
