"""Fused-conv timing sweep (C4 / C5-on-one-GPU) with the SURVEY.md §8d
algorithmic byte counts: fwd |E|(dy+W) + |V|(dx+dz); bwd 2|E|(dy+W) +
|V|(2dx+dz); dbwd 3|E|(dy+W) + |V|(3dx+2dz) words.

    python tools/sweep_conv.py [--cases c4,c5] [--ops fwd,bwd,dbwd] [--dtypes f32,f64] [--modes det,atomic,unfused]

The atomic mode's algorithmic bytes are counted with the same compulsory
formula (its extra per-edge reductions are the price of non-determinism).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200 import dist as cdist  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402

CASES = {"c4": ("c2", 29), "c5": ("c1", 58), "c4_c1tp": ("c1", 29)}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c4")
    ap.add_argument("--ops", default="fwd,bwd,dbwd")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--modes", default="det")
    a = ap.parse_args()
    pk = peak()
    for case in a.cases.split(","):
        prob, n = CASES[case]
        nodes, src, nbr = cdist.lattice_radius_graph(n, 1.0, 3.0)
        plan = cgf.TpPlan(config_json(prob))
        cp = cgf.ConvPlan(plan)
        g = cgf.Graph(nodes, src, nbr)
        del src, nbr
        V, E = g.nodes, g.edges
        for dts in a.dtypes.split(","):
            tdt = torch.float32 if dts == "f32" else torch.float64
            es = 4 if dts == "f32" else 8
            t = lambda *s: torch.randn(s, device="cuda", dtype=tdt)
            nx, ey, ew = t(V, plan.dim_x), t(E, plan.dim_y), t(E, plan.n_w)
            gz = t(V, plan.dim_z)
            for mode_name, op in [(m, o) for m in a.modes.split(",") for o in a.ops.split(",")]:
                mode = cgf.ATOMIC if mode_name == "atomic" else cgf.DETERMINISTIC
                unf = mode_name == "unfused"
                if unf and op == "dbwd":
                    continue
                up = None
                if op == "fwd":
                    fn = (lambda: cp.unfused_forward(g, nx, ey, ew)) if unf else (lambda: cp.forward(g, nx, ey, ew, mode=mode))
                    words = E * (plan.dim_y + plan.n_w) + V * (plan.dim_x + plan.dim_z)
                    flops = plan.flops_fwd * E
                elif op == "bwd":
                    fn = (lambda: cp.unfused_backward(g, nx, ey, ew, gz)) if unf else (lambda: cp.backward(g, nx, ey, ew, gz, mode=mode))
                    words = 2 * E * (plan.dim_y + plan.n_w) + V * (2 * plan.dim_x + plan.dim_z)
                    flops = plan.flops_bwd * E
                else:
                    try:
                        up = (t(V, plan.dim_x), t(E, plan.dim_y), t(E, plan.n_w))
                    except torch.OutOfMemoryError:
                        print(json.dumps({"case": case, "op": op, "dtype": dts, "error": "OOM"}))
                        continue
                    fn = lambda: cp.double_backward(g, nx, ey, ew, gz, up, mode=mode)
                    words = 3 * E * (plan.dim_y + plan.n_w) + V * (3 * plan.dim_x + 2 * plan.dim_z)
                    flops = plan.flops_dbwd * E
                try:
                    r = fn()
                    del r
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(a.iters):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        r = fn()
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                        del r
                    ms = statistics.median(ts)
                    gbs = words * es / (ms / 1e3) / 1e9
                    rec = {"case": case, "tp": prob, "mode": mode_name, "env": {k: v for k, v in os.environ.items()
                                                                               if k.startswith("CGF_")}, "nodes": V, "edges": E, "op": op, "dtype": dts, "ms": ms,
                           "edges/s": E / (ms / 1e3), "GB/s": gbs, "frac_hbm": gbs / pk,
                           "GFLOP/s": flops / (ms / 1e3) / 1e9}
                except Exception as exc:
                    rec = {"case": case, "op": op, "dtype": dts, "error": repr(exc)[:300]}
                print(json.dumps(rec), flush=True)
                del up
                torch.cuda.empty_cache()
            del nx, ey, ew, gz
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
