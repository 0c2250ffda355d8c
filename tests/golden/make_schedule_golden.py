"""Regenerates the schedule / counter / listing fixtures from the UNMODIFIED
reference (oracle/_ref/libcgforge_ref.so; `make -C oracle ref`). Run here,
where /root/reference exists:

    python tests/golden/make_schedule_golden.py

  listings/<name>.txt   kernelgen::emit_text of the reference's golden-listing
                        problems (test_kernelgen.cpp:148-156), checked equal to
                        the reference's own proj/tests/golden/<name>.txt
  schedules.json        per (problem, budget): sha256 + length of
                        scheduler::schedule_to_json, the strategy, and the
                        ExecStats of forward / backward / double_backward on 3
                        rows (engine.cpp:224-392); the "paper" problem's JSON
                        text in full
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))

from oracle import oracle as O  # noqa: E402
from problems import random_problem  # noqa: E402

REF_TESTS = "/root/reference/proj/tests/golden"

# test_kernelgen.cpp:148-156: single-instruction problems (l1, l2, l3, kind, b', b)
LISTING_PROBLEMS = {
    "b_fwd_000": ({"x": "1x0e", "y": "1x0e", "z": "1x0e", "instructions": [[1, 1, 1, "B"]]}, False),
    "b_fwd_111": ({"x": "32x1o", "y": "1x1o", "z": "32x1e", "instructions": [[1, 1, 1, "B"]]}, False),
    "b_bwd_111": ({"x": "32x1o", "y": "1x1o", "z": "32x1e", "instructions": [[1, 1, 1, "B"]]}, True),
    "c_fwd_110": ({"x": "32x1o", "y": "1x1o", "z": "16x0e", "instructions": [[1, 1, 1, "C"]]}, False),
    "c_bwd_110": ({"x": "32x1o", "y": "1x1o", "z": "16x0e", "instructions": [[1, 1, 1, "C"]]}, True),
}

BUDGETS = (100000, 4096, 2000, 1642)


def schedule_cases():
    cases = {n: O.config_json(n) for n in ("c1", "c2", "c3", "scalar", "paper")}
    for seed in (2, 3, 7, 11, 31, 32, 33, 301, 311):
        cases[f"rand{seed}"] = random_problem(seed)
    return cases


def main():
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    for name, (prob, bwd) in LISTING_PROBLEMS.items():
        txt = O.RefPlan(json.dumps(prob)).emit_text(0, backward=bwd)
        ref_file = os.path.join(REF_TESTS, name + ".txt")
        if os.path.exists(ref_file):
            assert open(ref_file).read() == txt, name
        with open(os.path.join(HERE, "listings", name + ".txt"), "w") as f:
            f.write(txt)
    out = {"listing_problems": {k: v[0] for k, v in LISTING_PROBLEMS.items()}, "cases": {}}
    for name, js in schedule_cases().items():
        for budget in BUDGETS:
            try:
                ref = O.RefPlan(js, budget=budget)
            except ValueError as e:
                out["cases"][f"{name}@{budget}"] = {"problem": js, "budget": budget, "error": str(e)}
                continue
            text = ref.schedule_json()
            g = O.NormalGen(1234)
            x = g.normal_vec(3 * ref.dim_x).reshape(3, -1)
            y = g.normal_vec(3 * ref.dim_y).reshape(3, -1)
            w = g.normal_vec(3 * ref.n_w).reshape(3, -1)
            gz = g.normal_vec(3 * ref.dim_z).reshape(3, -1)
            stats = {}
            ref.forward(x, y, w)
            stats["forward"] = ref.last_stats
            ref.backward(x, y, w, gz)
            stats["backward"] = ref.last_stats
            ref.double_backward(x, y, w, gz, x, y, w)
            stats["double_backward"] = ref.last_stats
            rec = {"problem": js, "budget": budget, "strategy": ref.strategy, "phases": ref.phases,
                   "schedule_sha256": hashlib.sha256(text.encode()).hexdigest(), "schedule_len": len(text),
                   "stats_3_rows": stats}
            if name == "paper":
                rec["schedule_json"] = text
            out["cases"][f"{name}@{budget}"] = rec
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("schedule / listing fixtures written to", HERE)


if __name__ == "__main__":
    main()
