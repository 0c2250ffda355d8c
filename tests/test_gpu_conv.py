"""GPU parity tests for the fused TP + graph convolution (deterministic,
row-owned, no atomics) against the CPU oracle's conv (reference semantics,
conv.cpp:234-528; double-backward composed per SURVEY.md §8c)."""
import numpy as np
import pytest

from oracle import oracle as O
from problems import config, random_problem

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}
DTYPES = [np.float32, np.float64]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def P():
    import paper_2501_13986_b200 as pkg
    return pkg


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def check(got, want, dt, what):
    err = O.rel_error(got, want)
    assert err <= TOL[dt], f"{what}: rel err {err:.3e} > {TOL[dt]:.0e}"


def conv_inputs(o, g, dt, seed=1234):
    gen = O.NormalGen(seed)
    nx = gen.normal_vec(g.nodes * o.dim_x, dt).reshape(g.nodes, -1)
    ey = gen.normal_vec(g.edges * o.dim_y, dt).reshape(g.edges, -1)
    ew = gen.normal_vec(g.edges * o.n_w, dt).reshape(g.edges, -1)
    gnz = O.NormalGen(seed + 1).normal_vec(g.nodes * o.dim_z, dt).reshape(g.nodes, -1)
    dgx = O.NormalGen(seed + 2).normal_vec(nx.size, dt).reshape(nx.shape)
    dgy = O.NormalGen(seed + 3).normal_vec(ey.size, dt).reshape(ey.shape)
    dgw = O.NormalGen(seed + 4).normal_vec(ew.size, dt).reshape(ew.shape)
    return nx, ey, ew, gnz, dgx, dgy, dgw


def graphs():
    g1 = O.radius_graph(O.cubic_lattice(4), 1.5)
    # ragged: a lattice with some nodes isolated (rows with no edges) and an
    # isolated neighbour set (nodes never read)
    g = O.radius_graph(O.cubic_lattice(5), 1.8)
    keep = (g.src % 7 != 3) & (g.nbr % 11 != 5)
    g2 = O.make_graph(g.nodes, g.src[keep], g.nbr[keep])
    return {"lat4": g1, "ragged5": g2}


CASES = [("paper", config("paper")), ("c1", config("c1")), ("c2", config("c2")),
         ("rand311", random_problem(311)), ("rand2", random_problem(2)), ("rand5", random_problem(5))]


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("gname", ["lat4", "ragged5"])
@pytest.mark.parametrize("name,js", CASES, ids=[c[0] for c in CASES])
def test_conv_fwd_bwd_dbwd(name, js, gname, dt):
    og = graphs()[gname]
    o, pkg = O.Oracle(js), P()
    plan = pkg.TpPlan(js)
    cp = pkg.ConvPlan(plan)
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, dgx, dgy, dgw = conv_inputs(o, og, dt)
    z = cp.forward(g, dev(nx), dev(ey), dev(ew))
    check(host(z), o.conv_forward(og, nx, ey, ew), dt, "conv forward")
    outs = cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gnz))
    for a, b, n in zip(outs, o.conv_backward(og, nx, ey, ew, gnz), ("g_node_x", "g_edge_y", "g_edge_w")):
        check(host(a), b, dt, n)
    outs = cp.double_backward(g, dev(nx), dev(ey), dev(ew), dev(gnz), (dev(dgx), dev(dgy), dev(dgw)))
    want = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    for a, b, n in zip(outs, want, ("dnode_x", "dedge_y", "dedge_w", "dg_node_z")):
        check(host(a), b, dt, n)


def test_golden_conv_fixture():
    d = np.load("tests/golden/conv_paper_float64.npz")
    js = str(d["problem"])
    o, pkg = O.Oracle(js), P()
    og = O.make_graph(27, d["src"], d["nbr"])
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, *_ = conv_inputs(o, og, np.float64)
    check(host(cp.forward(g, dev(nx), dev(ey), dev(ew))), d["z"], np.float64, "golden z")
    for a, k in zip(cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gnz)), ("gx", "gy", "gw")):
        check(host(a), d[k], np.float64, k)


@pytest.mark.parametrize("name", ["paper", "c2"])
def test_single_edge_conv_equals_tp_bitwise(name):
    """A single-edge conv is one TP, bit for bit (test_conv.cpp:162-180, 308-333)."""
    js = config(name)
    o, pkg = O.Oracle(js), P()
    plan = pkg.TpPlan(js)
    cp = pkg.ConvPlan(plan)
    g = pkg.Graph(2, [0], [1])
    gen = O.NormalGen(7)
    nx = gen.normal_vec(2 * o.dim_x).reshape(2, -1)
    ey = gen.normal_vec(o.dim_y).reshape(1, -1)
    ew = gen.normal_vec(o.n_w).reshape(1, -1)
    z = cp.forward(g, dev(nx), dev(ey), dev(ew))
    zt = plan.forward(dev(nx[1:2]), dev(ey), dev(ew))
    assert torch.equal(z[0], zt[0])
    assert not z[1].any()
    gz = O.NormalGen(8).normal_vec(2 * o.dim_z).reshape(2, -1)
    gx, gy, gw = cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gz))
    tx, ty, tw = plan.backward(dev(nx[1:2]), dev(ey), dev(ew), dev(gz[0:1]))
    assert torch.equal(gx[1], tx[0]) and torch.equal(gy, ty) and torch.equal(gw, tw)
    assert not gx[0].any()


def test_conv_deterministic_bitwise():
    js = config("c1")
    o, pkg = O.Oracle(js), P()
    og = O.radius_graph(O.cubic_lattice(6), 2.0)
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, *_ = conv_inputs(o, og, np.float64)
    a = cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gnz))
    b = cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gnz))
    for u, v in zip(a, b):
        assert torch.equal(u, v)


def test_unsorted_edges_rejected_by_deterministic_mode():
    """conv.cpp:240 / 371-374: only the deterministic mode checks the order."""
    pkg = P()
    js = config("paper")
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    o = O.Oracle(js)
    g = pkg.Graph(3, [1, 0], [0, 1])
    nx = torch.zeros((3, o.dim_x), device="cuda", dtype=torch.float64)
    ey = torch.zeros((2, o.dim_y), device="cuda", dtype=torch.float64)
    ew = torch.zeros((2, o.n_w), device="cuda", dtype=torch.float64)
    with pytest.raises(pkg.InvalidArgument):
        cp.forward(g, nx, ey, ew)
    cp.forward(g, nx, ey, ew, mode=pkg.ATOMIC)


# ---- atomic mode (Mode::atomic, conv.cpp:311-324 / 470-486): edges in any
# order, node outputs accumulated with float atomics.
ATOMIC_CASES = [("paper", config("paper")), ("c1", config("c1")), ("c2", config("c2")), ("rand5", random_problem(5))]


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("gname", ["lat4", "ragged5"])
@pytest.mark.parametrize("name,js", ATOMIC_CASES, ids=[c[0] for c in ATOMIC_CASES])
def test_atomic_conv_shuffled_edges(name, js, gname, dt):
    og = graphs()[gname]
    o, pkg = O.Oracle(js), P()
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    nx, ey, ew, gnz, dgx, dgy, dgw = conv_inputs(o, og, dt)
    perm = np.random.default_rng(5).permutation(og.edges)  # edge list in random order
    g = pkg.Graph(og.nodes, og.src[perm], og.nbr[perm])
    assert og.edges < 2 or not g.sorted
    A = pkg.ATOMIC
    z = cp.forward(g, dev(nx), dev(ey[perm]), dev(ew[perm]), mode=A)
    check(host(z), o.conv_forward(og, nx, ey, ew), dt, "atomic forward")
    gx, gy, gw = cp.backward(g, dev(nx), dev(ey[perm]), dev(ew[perm]), dev(gnz), mode=A)
    wx, wy, ww = o.conv_backward(og, nx, ey, ew, gnz)
    check(host(gx), wx, dt, "atomic g_node_x")
    check(host(gy), wy[perm], dt, "atomic g_edge_y")
    check(host(gw), ww[perm], dt, "atomic g_edge_w")
    outs = cp.double_backward(g, dev(nx), dev(ey[perm]), dev(ew[perm]), dev(gnz),
                              (dev(dgx), dev(dgy[perm]), dev(dgw[perm])), mode=A)
    want = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    for a, b, n in zip(outs, (want[0], want[1][perm], want[2][perm], want[3]),
                       ("dnode_x", "dedge_y", "dedge_w", "dg_node_z")):
        check(host(a), b, dt, "atomic " + n)


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_atomic_via_csr_entry_points(dt):
    """The CSR C ABI entries with CGF_CONV_ATOMIC expand row_ptr on the device
    and run the atomic kernels: within rounding of the deterministic mode
    (test_conv.cpp:247-258)."""
    import ctypes as C
    js = config("c1")
    o, pkg = O.Oracle(js), P()
    plan = pkg.TpPlan(js)
    og = graphs()["ragged5"]
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, *_ = conv_inputs(o, og, dt)
    tx, ty, tw = dev(nx), dev(ey), dev(ew)
    det = pkg.ConvPlan(plan).forward(g, tx, ty, tw)
    z = torch.empty_like(det)
    d = g.device(tx.device)
    ptr = lambda t: C.c_void_p(t.data_ptr())
    rc = pkg.lib().cgf_conv_forward(plan._h, pkg.F32 if dt == np.float32 else pkg.F64, g.nodes, g.edges,
                                    ptr(d["row_ptr"]), ptr(d["nbr"]), ptr(tx), ptr(ty), ptr(tw), ptr(z), pkg.ATOMIC,
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, pkg.lib().cgf_last_error()
    check(host(z), host(det), dt, "atomic (CSR entry) vs deterministic")


def test_atomic_empty_graph_and_isolated_nodes():
    js = config("paper")
    o, pkg = O.Oracle(js), P()
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(4, np.zeros(0, np.int64), np.zeros(0, np.int64))
    nx = torch.randn((4, o.dim_x), device="cuda", dtype=torch.float64)
    ey = torch.zeros((0, o.dim_y), device="cuda", dtype=torch.float64)
    ew = torch.zeros((0, o.n_w), device="cuda", dtype=torch.float64)
    z = cp.forward(g, nx, ey, ew, mode=pkg.ATOMIC)
    assert z.shape == (4, o.dim_z) and not z.any()
    gx, gy, gw = cp.backward(g, nx, ey, ew, torch.randn((4, o.dim_z), device="cuda", dtype=torch.float64),
                             mode=pkg.ATOMIC)
    assert not gx.any() and gy.shape == (0, o.dim_y) and gw.shape == (0, o.n_w)


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c4_full_graph_sampled(dt):
    """C4 at full size: C2 TP on radius_graph(cubic_lattice(29), 3.0) =
    24,389 nodes / 2,634,962 edges. Output rows sampled against the oracle."""
    js = config("c2")
    o, pkg = O.Oracle(js), P()
    og = O.radius_graph(O.cubic_lattice(29), 3.0)
    assert (og.nodes, og.edges) == (24389, 2634962)
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    gen = torch.Generator(device="cuda").manual_seed(3)
    nx = torch.randn((og.nodes, o.dim_x), device="cuda", dtype=tdt, generator=gen)
    ey = torch.randn((og.edges, o.dim_y), device="cuda", dtype=tdt, generator=gen)
    ew = torch.randn((og.edges, o.n_w), device="cuda", dtype=tdt, generator=gen)
    z = cp.forward(g, nx, ey, ew)
    rows = np.array([0, 1, 12194, 24388])
    keep = np.isin(og.src, rows)
    sub = O.make_graph(og.nodes, og.src[keep], og.nbr[keep])
    eidx = torch.from_numpy(np.nonzero(keep)[0]).cuda()
    want = o.conv_forward(sub, host(nx), host(ey[eidx]), host(ew[eidx]))
    check(host(z)[rows], want[rows], dt, "C4 sampled forward rows")
    gz = torch.randn((og.nodes, o.dim_z), device="cuda", dtype=tdt, generator=gen)
    gx, gy, gw = cp.backward(g, nx, ey, ew, gz)
    keep = np.isin(og.nbr, rows)
    sub = O.make_graph(og.nodes, og.src[keep], og.nbr[keep])
    eidx = torch.from_numpy(np.nonzero(keep)[0]).cuda()
    wx, wy, ww = o.conv_backward(sub, host(nx), host(ey[eidx]), host(ew[eidx]), host(gz))
    check(host(gx)[rows], wx[rows], dt, "C4 sampled g_node_x")
    check(host(gy[eidx]), wy, dt, "C4 sampled g_edge_y")
    check(host(gw[eidx]), ww, dt, "C4 sampled g_edge_w")


@pytest.mark.parametrize("groups", [1, 2, 3, 5])
@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_grouped_kernels_match_oracle(groups, dt, monkeypatch):
    """The by-neighbour conv kernels (backward, double-backward pass 2) and
    the batched TP double-backward run their units in G groups, one kernel
    each, with the per-edge / per-row dy summed in group order: any G gives
    the oracle's results (C2 TP on a ragged lattice graph, plus 300 TP rows)."""
    monkeypatch.setenv("CGF_CONVI_GROUPS", str(groups))
    monkeypatch.setenv("CGF_ROW_GROUPS", str(groups))
    js = config("c2")
    o, pkg = O.Oracle(js), P()
    plan = pkg.TpPlan(js)
    cp = pkg.ConvPlan(plan)
    og = graphs()["ragged5"]
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, dgx, dgy, dgw = conv_inputs(o, og, dt, seed=55)
    outs = cp.backward(g, dev(nx), dev(ey), dev(ew), dev(gnz))
    for got, want, n in zip(outs, o.conv_backward(og, nx, ey, ew, gnz), ("gx", "gy", "gw")):
        check(host(got), want, dt, f"G={groups} conv {n}")
    outs = cp.double_backward(g, dev(nx), dev(ey), dev(ew), dev(gnz), (dev(dgx), dev(dgy), dev(dgw)))
    want = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    for got, wv, n in zip(outs, want, ("dx", "dy", "dw", "dgz")):
        check(host(got), wv, dt, f"G={groups} conv double-backward {n}")
    rows = 300
    gen = O.NormalGen(77)
    x, y, w = (gen.normal_vec(rows * d, dt).reshape(rows, -1) for d in (o.dim_x, o.dim_y, o.n_w))
    gz, da = (gen.normal_vec(rows * d, dt).reshape(rows, -1) for d in (o.dim_z, o.dim_x))
    db, dc = (gen.normal_vec(rows * d, dt).reshape(rows, -1) for d in (o.dim_y, o.n_w))
    outs = plan.double_backward(dev(x), dev(y), dev(w), dev(gz), (dev(da), dev(db), dev(dc)))
    for got, wv, n in zip(outs, o.double_backward(x, y, w, gz, da, db, dc), ("dx", "dy", "dw", "dgz")):
        check(host(got), wv, dt, f"G={groups} TP double-backward {n}")


@pytest.mark.parametrize("epi", [2, 3])
@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("name", ["c1", "c2", "paper"])
def test_multi_edge_items_match_oracle(name, dt, epi, monkeypatch):
    """By-output conv kernels with EB consecutive edges of a row staged per
    item (CGF_GEN=epi=EB): ragged rows (edge counts not multiples of EB,
    isolated nodes) give the oracle's forward and double-backward dgz."""
    monkeypatch.setenv("CGF_GEN", f"epi={epi}")
    js = config(name)
    o, pkg = O.Oracle(js), P()
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    og = graphs()["ragged5"]
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, dgx, dgy, dgw = conv_inputs(o, og, dt, seed=66)
    check(host(cp.forward(g, dev(nx), dev(ey), dev(ew))), o.conv_forward(og, nx, ey, ew), dt, f"EB={epi} forward")
    outs = cp.double_backward(g, dev(nx), dev(ey), dev(ew), dev(gnz), (dev(dgx), dev(dgy), dev(dgw)))
    want = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    check(host(outs[3]), want[3], dt, f"EB={epi} double-backward dgz")


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("gname", ["lat4", "ragged5"])
@pytest.mark.parametrize("name", ["paper", "c1", "c2"])
def test_row_order_backward_matches_oracle(name, gname, dt, monkeypatch):
    """The row-order conv backward (CGF_CONV_BWD=row: edges in CSR order, per-edge
    g_node_x partial rows, segmented sum over the transposed CSR) against the
    oracle; deterministic (two calls bitwise equal), and a single edge is still
    one TP bit for bit."""
    monkeypatch.setenv("CGF_CONV_BWD", "row")
    js = config(name)
    og = graphs()[gname]
    o, pkg = O.Oracle(js), P()
    plan = pkg.TpPlan(js)
    cp = pkg.ConvPlan(plan)
    g = pkg.Graph(og.nodes, og.src, og.nbr)
    nx, ey, ew, gnz, *_ = conv_inputs(o, og, dt)
    args = (dev(nx), dev(ey), dev(ew), dev(gnz))
    outs = cp.backward(g, *args)
    for a, b, n in zip(outs, o.conv_backward(og, nx, ey, ew, gnz), ("g_node_x", "g_edge_y", "g_edge_w")):
        check(host(a), b, dt, n)
    for a, b in zip(outs, cp.backward(g, *args)):
        assert torch.equal(a, b)
    g1 = pkg.Graph(2, [0], [1])
    x1 = dev(nx[:2])
    gx, gy, gw = cp.backward(g1, x1, dev(ey[:1]), dev(ew[:1]), dev(gnz[:2]))
    tx, ty, tw = plan.backward(x1[1:2], dev(ey[:1]), dev(ew[:1]), dev(gnz[0:1]))
    assert torch.equal(gx[1], tx[0]) and torch.equal(gy, ty) and torch.equal(gw, tw)
    assert not gx[0].any()
