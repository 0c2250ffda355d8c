"""CPU tests of the product's counters and dumps:
the per-row schedule model behind ExecStats, schedule_to_json and the
emit_text listings are computed by libcgf (csrc/schedule.cpp) and must equal
the reference's — pinned by fixtures generated from the unmodified reference
(tests/golden/make_schedule_golden.py) and, where oracle/_ref was built, by
the live reference on more problems and budgets."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2501_13986_b200 as cgf
from oracle import oracle as O
from problems import random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")
REF_GOLDEN_DIR = "/root/reference/proj/tests/golden"
FIX = json.load(open(os.path.join(GOLD, "schedules.json")))
OPS = {"forward": cgf.OP_FORWARD, "backward": cgf.OP_BACKWARD, "double_backward": cgf.OP_DOUBLE_BACKWARD}


@pytest.mark.parametrize("case", sorted(FIX["cases"]))
def test_schedule_json_and_exec_stats_match_reference_fixture(case):
    rec = FIX["cases"][case]
    if "error" in rec:
        with pytest.raises(cgf.BudgetError) as ei:
            cgf.TpPlan(rec["problem"], budget=rec["budget"])
        assert str(ei.value) == rec["error"]
        return
    plan = cgf.TpPlan(rec["problem"], budget=rec["budget"])
    text = plan.schedule_json()
    assert len(text) == rec["schedule_len"]
    assert hashlib.sha256(text.encode()).hexdigest() == rec["schedule_sha256"]
    if "schedule_json" in rec:
        assert text == rec["schedule_json"]
    for op, want in rec["stats_3_rows"].items():
        assert plan.stats(OPS[op], 3) == tuple(want), op


@pytest.mark.parametrize("name", sorted(FIX["listing_problems"]))
def test_listing_byte_exact_against_reference_golden(name):
    """kernelgen::emit_text of the reference's golden-listing problems
    (test_kernelgen.cpp:148-156), byte for byte: the committed fixture, and the
    reference checkout's own file where it exists."""
    plan = cgf.TpPlan(json.dumps(FIX["listing_problems"][name]))
    txt = plan.listing(0, backward="_bwd_" in name)
    assert txt == open(os.path.join(GOLD, "listings", name + ".txt")).read()
    ref_file = os.path.join(REF_GOLDEN_DIR, name + ".txt")
    if os.path.exists(ref_file):
        assert txt == open(ref_file).read()


def test_budget_error_message_matches_reference():
    js = cgf.configs.config_json("c3")
    with pytest.raises(cgf.BudgetError) as ei:
        cgf.TpPlan(js, budget=700)
    assert str(ei.value) == "budget 700 words below working set 1089 of subkernel 0 (C, l=(0,0,0), b=32, b'=32)"


def test_forward_stats_equal_traffic_times_rows():
    """test_engine.cpp:350-363 on the paper problem, both budgets."""
    js = cgf.configs.config_json("paper")
    for budget in (100000, 1642):
        plan = cgf.TpPlan(js, budget=budget)
        rec = FIX["cases"][f"paper@{budget}"] if f"paper@{budget}" in FIX["cases"] else None
        loads, stores, flops = plan.stats(cgf.OP_FORWARD, 1)
        assert plan.stats(cgf.OP_FORWARD, 7) == (7 * loads, 7 * stores, 7 * flops)
        assert flops == plan.flops_fwd
        if rec:
            doc = json.loads(plan.schedule_json())
            assert (doc["traffic"]["loads_words"], doc["traffic"]["stores_words"], doc["traffic"]["flops"]) == \
                (loads, stores, flops)


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed", list(range(40, 70)))
def test_schedule_and_listings_match_live_reference_random(seed):
    js = random_problem(seed)
    for budget in (100000, 3000, 1200):
        try:
            ref = O.RefPlan(js, budget=budget)
        except ValueError as e:
            with pytest.raises(cgf.BudgetError) as ei:
                cgf.TpPlan(js, budget=budget)
            assert str(ei.value) == str(e)
            continue
        plan = cgf.TpPlan(js, budget=budget)
        assert plan.schedule_json() == ref.schedule_json()
        g = O.NormalGen(seed)
        x = g.normal_vec(2 * ref.dim_x).reshape(2, -1)
        y = g.normal_vec(2 * ref.dim_y).reshape(2, -1)
        w = g.normal_vec(2 * ref.n_w).reshape(2, -1)
        gz = g.normal_vec(2 * ref.dim_z).reshape(2, -1)
        ref.forward(x, y, w)
        assert plan.stats(cgf.OP_FORWARD, 2) == ref.last_stats
        ref.backward(x, y, w, gz)
        assert plan.stats(cgf.OP_BACKWARD, 2) == ref.last_stats
        ref.double_backward(x, y, w, gz, x, y, w)
        assert plan.stats(cgf.OP_DOUBLE_BACKWARD, 2) == ref.last_stats
    for pos in range(plan.n_split):
        for bwd in (False, True):
            assert plan.listing(pos, bwd) == ref.emit_text(pos, bwd)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_array_files_round_trip_and_match_reference_bytes(tmp_path, dt):
    """array_io (array_io.cpp:15-68): libcgf writes the reference's exact
    .bin / .json bytes, reads them back, and rejects a dtype mismatch and a
    short .bin like the reference."""
    a = np.random.default_rng(3).standard_normal((5, 7)).astype(dt)
    base = str(tmp_path / "ours")
    cgf.save_array(base, a)
    assert cgf.read_meta(base) == (5, 7, cgf.F64 if dt == np.float64 else cgf.F32)
    assert np.array_equal(cgf.load_array(base), a)
    if O.ref_available():
        import ctypes as C
        rb = str(tmp_path / "ref")
        assert O.ref_lib().cgr_save_array(rb.encode(), a.ctypes.data, 5, 7, int(dt == np.float64)) == 0
        for ext in (".bin", ".json"):
            assert open(base + ext, "rb").read() == open(rb + ext, "rb").read(), ext
    other = np.float32 if dt == np.float64 else np.float64
    import ctypes as C
    buf = np.empty(35, other)
    rc = cgf.lib().cgf_array_load(base.encode(), cgf.F32 if other == np.float32 else cgf.F64, buf.ctypes.data, 35, 0,
                                  None)
    assert rc != 0 and "expected" in cgf.lib().cgf_last_error().decode()
    with open(base + ".bin", "r+b") as f:
        f.truncate(8)
    with pytest.raises(cgf.CgfError, match="shorter"):
        cgf.load_array(base)
