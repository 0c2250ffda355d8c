"""Times every TP op of the benchmark configurations on one GPU and prints a
roofline table (CUDA events on the launching stream, inputs > L2, median of
`--iters` launches after warm-up). Algorithmic bytes follow SURVEY.md §8d.

    python tools/sweep.py [--configs c1,c2,c3] [--ops fwd,bwd,dbwd] [--dtypes f32,f64]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2501_13986_b200 as cgf  # noqa: E402
from paper_2501_13986_b200.configs import config_json  # noqa: E402

ROWS = {"c1": 50_000, "c2": 1_000_000, "c3": 1_000_000}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2")
    ap.add_argument("--ops", default="fwd,bwd,dbwd")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--w-shared", action="store_true")
    args = ap.parse_args()
    pk = peak()
    for cname in args.configs.split(","):
        plan = cgf.TpPlan(config_json(cname))
        for dts in args.dtypes.split(","):
            tdt = torch.float32 if dts == "f32" else torch.float64
            es = 4 if dts == "f32" else 8
            R = args.rows or ROWS[cname]
            if dts == "f64" and cname == "c2":
                R = min(R, 400_000)  # FP64 C2 double-backward needs ~226 GB at 1M rows
            ws = args.w_shared
            nw_rows = 1 if ws else R
            t = lambda *s: torch.randn(s, device="cuda", dtype=tdt)
            x, y, w, gz = t(R, plan.dim_x), t(R, plan.dim_y), t(nw_rows, plan.n_w), t(R, plan.dim_z)
            for op in args.ops.split(","):
                if op == "fwd":
                    fn = lambda: plan.forward(x, y, w, w_shared=ws)
                    words = R * (plan.dim_x + plan.dim_y + plan.dim_z) + nw_rows * plan.n_w
                    flops = plan.flops_fwd * R
                elif op == "bwd":
                    fn = lambda: plan.backward(x, y, w, gz, w_shared=ws)
                    words = R * (2 * plan.dim_x + 2 * plan.dim_y + plan.dim_z) + 2 * nw_rows * plan.n_w
                    flops = plan.flops_bwd * R
                else:
                    up = (t(R, plan.dim_x), t(R, plan.dim_y), t(nw_rows, plan.n_w))
                    fn = lambda: plan.double_backward(x, y, w, gz, up, w_shared=ws)
                    words = R * (3 * plan.dim_x + 3 * plan.dim_y + 2 * plan.dim_z) + 3 * nw_rows * plan.n_w
                    flops = plan.flops_dbwd * R
                try:
                    for _ in range(2):
                        fn()
                    torch.cuda.synchronize()
                    # short kernels are timed as a burst of back-to-back calls between
                    # two events, so host launch overhead does not count
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    r = fn()
                    b.record()
                    torch.cuda.synchronize()
                    del r
                    burst = max(1, min(100, int(10.0 / max(a.elapsed_time(b), 1e-3))))
                    ts = []
                    for _ in range(args.iters):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        for _ in range(burst):
                            r = fn()
                        b.record()
                        torch.cuda.synchronize()
                        ts.append(a.elapsed_time(b) / burst)
                        del r
                    ms = statistics.median(ts)
                    gbs = words * es / (ms / 1e3) / 1e9
                    rec = {"config": cname, "op": op, "dtype": dts, "rows": R, "w_shared": ws, "ms": ms, "burst": burst,
                           "env": {k: v for k, v in os.environ.items() if k.startswith("CGF_")},
                           "GB/s": gbs, "frac_hbm": gbs / pk, "GFLOP/s": flops / (ms / 1e3) / 1e9,
                           "rows/s": R / (ms / 1e3)}
                except Exception as exc:
                    rec = {"config": cname, "op": op, "dtype": dts, "error": repr(exc)[:300]}
                print(json.dumps(rec), flush=True)
                if op == "dbwd":
                    del up
            del x, y, w, gz
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
