"""Graph construction on the device vs the unmodified reference on the host
(conv.cpp:64-151): radius_graph of the C4 / C5 lattices, make_graph of a
shuffled edge list with duplicates, and the transposed CSR. Device times are
CUDA-event medians; the reference is timed through oracle/_ref (1 thread).

    python tools/sweep_graph.py [--cases c4,c5] [--iters 5]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2501_13986_b200 as cgf  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = {"c4": 29, "c5": 58}


def dev_ms(fn, iters):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c4,c5")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    for case in a.cases.split(","):
        n = CASES[case]
        pos = torch.from_numpy(O.cubic_lattice(n)).cuda()
        dg = cgf.radius_graph_device(pos, 3.0)
        rec = {"case": case, "nodes": dg.nodes, "edges": dg.edges}
        rec["radius_graph_ms"] = dev_ms(lambda: cgf.radius_graph_device(pos, 3.0), a.iters)
        perm = torch.randperm(dg.edges, device="cuda")
        src = torch.cat([dg.src[perm], dg.src[: dg.edges // 4]])
        dst = torch.cat([dg.nbr[perm], dg.nbr[: dg.edges // 4]])
        rec["make_graph_ms"] = dev_ms(lambda: cgf.make_graph_device(dg.nodes, src, dst), a.iters)
        rec["make_graph_input_edges"] = int(src.numel())

        def tr():
            dg._t = None
            dg._transpose()
        rec["transpose_ms"] = dev_ms(tr, a.iters)
        if O.ref_available():
            L = O.ref_lib()
            t0 = time.perf_counter()
            ne = L.cgr_lattice_graph(n, 1.0, 3.0, None, None, 0)  # cubic_lattice + radius_graph (+ make_graph)
            rec["reference_radius_graph_host_ms"] = (time.perf_counter() - t0) * 1e3
            rec["reference_edges"] = int(ne)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
