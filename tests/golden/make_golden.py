"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libcgforge_ref.so, built by `make -C oracle ref` from
/root/reference). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Fixtures (all outputs computed by the reference itself):
  cg_blocks.json        every real-basis CG block with l1,l2 <= 5, l3 <= 6
                        (cg.cpp:58-134), values as 17-digit decimals
  listing_coeffs.json   the coefficients printed in the reference's own golden
                        IR listings (proj/tests/golden/*.txt) + their (l1,l2,l3)
  tp_<name>_<dtype>.npz TpPlan forward / backward / double_backward outputs
                        on random_batch(seed=1234) inputs, gz NormalGen(1235),
                        da/db/dC NormalGen(1236/1237/1238) (cgforge.cpp:357-386)
  conv_<name>_<dtype>.npz ConvPlan forward / backward (deterministic, 1 chunk)
                        on radius_graph(cubic_lattice(3), 1.1), float64 only
"""
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

from oracle import oracle as O  # noqa: E402
from problems import random_problem  # noqa: E402

REF_TESTS = "/root/reference/proj/tests/golden"

TP_CASES = {
    "scalar": (O.config_json("scalar"), 4),
    "paper": (O.config_json("paper"), 3),
    "c1": (O.config_json("c1"), 3),
    "c2": (O.config_json("c2"), 1),
    "c3": (O.config_json("c3"), 2),
    "rand301": (random_problem(301), 3),
    "rand311": (random_problem(311), 3),
    "rand2": (random_problem(2), 3),
    "rand3": (random_problem(3), 3),
}
CONV_CASES = ["paper", "c1"]


def inputs(ref, rows, dt):
    g = O.NormalGen(1234)
    x = g.normal_vec(rows * ref.dim_x, dt).reshape(rows, -1)
    y = g.normal_vec(rows * ref.dim_y, dt).reshape(rows, -1)
    w = g.normal_vec(rows * ref.n_w, dt).reshape(rows, -1)
    gz = O.NormalGen(1235).normal_vec(rows * ref.dim_z, dt).reshape(rows, -1)
    da = O.NormalGen(1236).normal_vec(x.size, dt).reshape(x.shape)
    db = O.NormalGen(1237).normal_vec(y.size, dt).reshape(y.shape)
    dc = O.NormalGen(1238).normal_vec(w.size, dt).reshape(w.shape)
    return x, y, w, gz, da, db, dc


def main():
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    blocks = []
    for l1 in range(6):
        for l2 in range(6):
            for l3 in range(abs(l1 - l2), min(l1 + l2, 6) + 1):
                i, j, k, v = O.ref_cg_block(l1, l2, l3)
                blocks.append({"l": [l1, l2, l3],
                               "entries": [[int(a), int(b), int(c), float(d)]
                                           for a, b, c, d in zip(i, j, k, v)]})
    with open(os.path.join(HERE, "cg_blocks.json"), "w") as f:
        json.dump(blocks, f, separators=(",", ":"))

    if os.path.isdir(REF_TESTS):
        # l triple per listing: (name -> (l1,l2,l3)), test_kernelgen.cpp golden cases
        triples = {"b_fwd_000": (0, 0, 0), "b_fwd_111": (1, 1, 1), "b_bwd_111": (1, 1, 1),
                   "c_fwd_110": (1, 1, 0), "c_bwd_110": (1, 1, 0)}
        lst = {}
        for name, tri in triples.items():
            txt = open(os.path.join(REF_TESTS, name + ".txt")).read()
            co = [float(m) for m in re.findall(r"\+= (-?[0-9.e+-]+) \*", txt)]
            lst[name] = {"l": tri, "coeffs": co, "lines": txt.count("\n")}
        with open(os.path.join(HERE, "listing_coeffs.json"), "w") as f:
            json.dump(lst, f, indent=1)

    for name, (js, rows) in TP_CASES.items():
        ref = O.RefPlan(js)
        for dt in (np.float32, np.float64):
            x, y, w, gz, da, db, dc = inputs(ref, rows, dt)
            z = ref.forward(x, y, w)
            gx, gy, gw = ref.backward(x, y, w, gz)
            ox, oy, ow, ogz = ref.double_backward(x, y, w, gz, da, db, dc)
            np.savez_compressed(os.path.join(HERE, f"tp_{name}_{np.dtype(dt).name}.npz"),
                                problem=js, rows=rows, z=z, gx=gx, gy=gy, gw=gw, ox=ox, oy=oy,
                                ow=ow, ogz=ogz, flops=np.array(ref.traffic))

    g = O.radius_graph(O.cubic_lattice(3), 1.1)
    for name in CONV_CASES:
        js = O.config_json(name)
        ref = O.RefPlan(js)
        for dt in (np.float64,):
            gen = O.NormalGen(1234)
            nx = gen.normal_vec(g.nodes * ref.dim_x, dt).reshape(g.nodes, -1)
            ey = gen.normal_vec(g.edges * ref.dim_y, dt).reshape(g.edges, -1)
            ew = gen.normal_vec(g.edges * ref.n_w, dt).reshape(g.edges, -1)
            z = ref.conv_forward(g, nx, ey, ew, chunks=1)
            gnz = O.NormalGen(1235).normal_vec(z.size, dt).reshape(z.shape)
            gx, gy, gw = ref.conv_backward(g, nx, ey, ew, gnz, chunks=1)
            np.savez_compressed(os.path.join(HERE, f"conv_{name}_{np.dtype(dt).name}.npz"),
                                problem=js, src=g.src, nbr=g.nbr, z=z, gx=gx, gy=gy, gw=gw)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
