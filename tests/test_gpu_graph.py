"""GPU graph construction (conv.cpp:64-151 on the device) and the unfused
gather -> TP -> scatter comparator (conv.cpp:530-616). Integer outputs must
be bit-identical to the reference's host construction (the oracle's numpy
restatement, and the unmodified reference through oracle/_ref when built);
the unfused conv is checked against the oracle's conv at the §8c tolerances."""
import numpy as np
import pytest

from oracle import oracle as O
from problems import config, random_problem

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def P():
    import paper_2501_13986_b200 as pkg
    return pkg


def i32(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.int32))).cuda()


def same_graph(dg, og):
    assert dg.nodes == og.nodes and dg.edges == og.edges
    np.testing.assert_array_equal(dg.row_ptr.cpu().numpy(), og.row_ptr)
    np.testing.assert_array_equal(dg.nbr.cpu().numpy(), og.nbr)
    np.testing.assert_array_equal(dg.src.cpu().numpy(), og.src)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_make_graph_matches_reference(seed):
    rng = np.random.default_rng(seed)
    nodes = [1, 7, 300][seed]
    e = [0, 40, 20000][seed]
    src = rng.integers(0, nodes, e)
    dst = rng.integers(0, nodes, e)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    src = np.concatenate([src, src[: len(src) // 3]])  # duplicates, unsorted
    dst = np.concatenate([dst, dst[: len(dst) // 3]])
    dg = P().make_graph_device(nodes, i32(src), i32(dst))
    same_graph(dg, O.make_graph(nodes, src, dst))


def test_make_graph_self_loops_allowed():
    src, dst = [2, 1, 1, 0, 2], [2, 1, 0, 0, 2]
    dg = P().make_graph_device(3, i32(src), i32(dst), allow_self_loops=True)
    same_graph(dg, O.make_graph(3, src, dst, allow_self_loops=True))


def test_make_graph_errors_follow_first_bad_edge():
    pkg = P()
    with pytest.raises(pkg.InvalidArgument, match=r"self-loop \(1\)"):
        pkg.make_graph_device(4, i32([0, 1, 2, 5]), i32([1, 1, 2, 0]))
    with pytest.raises(pkg.InvalidArgument, match="out of range"):
        pkg.make_graph_device(4, i32([0, 7, 2]), i32([1, 1, 2]))


def test_transpose_matches_host_and_reference():
    pkg = P()
    og = O.radius_graph(O.cubic_lattice(6), 1.8)
    dg = pkg.make_graph_device(og.nodes, i32(og.src), i32(og.nbr))
    t_row_ptr, t_src, t_eid = dg._transpose()
    hg = pkg.Graph(og.nodes, og.src, og.nbr)  # host counting sort (cgf_conv_transpose_host)
    np.testing.assert_array_equal(t_row_ptr.cpu().numpy(), hg.t_row_ptr)
    np.testing.assert_array_equal(t_src.cpu().numpy(), hg.t_src[: og.edges])
    np.testing.assert_array_equal(t_eid.cpu().numpy(), hg.t_eid[: og.edges])
    perm = np.empty(og.edges, np.int64)
    perm[t_eid.cpu().numpy()] = np.arange(og.edges)
    np.testing.assert_array_equal(perm, O.transpose_permutation(og))


@pytest.mark.parametrize("n,r", [(1, 1.0), (4, 1.5), (5, 1.8), (7, 3.0)])
def test_radius_graph_lattice(n, r):
    pos = O.cubic_lattice(n)
    dg = P().radius_graph_device(torch.from_numpy(pos).cuda(), r)
    same_graph(dg, O.radius_graph(pos, r))


def test_radius_graph_random_positions():
    rng = np.random.default_rng(11)
    pos = rng.uniform(-2.0, 3.0, (3000, 3))
    dg = P().radius_graph_device(torch.from_numpy(pos).cuda(), 0.4)
    same_graph(dg, O.radius_graph(pos, 0.4))


def test_radius_graph_bad_cutoff():
    pkg = P()
    with pytest.raises(pkg.InvalidArgument):
        pkg.radius_graph_device(torch.zeros((3, 3), dtype=torch.float64, device="cuda"), 0.0)


@pytest.mark.parametrize("n,edges", [(29, 2634962), (58, 22416384)], ids=["c4", "c5"])
def test_radius_graph_benchmark_graphs(n, edges):
    """The C4 / C5 graphs built on the device: edge counts, and
    bit-identical CSR against the unmodified reference when oracle/_ref is
    built (else the numpy restatement for C4)."""
    pos = O.cubic_lattice(n)
    dg = P().radius_graph_device(torch.from_numpy(pos).cuda(), 3.0)
    assert dg.edges == edges
    if O.ref_available():
        same_graph(dg, O.ref_lattice_graph(n))
    elif n == 29:
        same_graph(dg, O.radius_graph(pos, 3.0))


# ---- unfused comparator ------------------------------------------------------

def conv_inputs(o, g, dt, seed=1234):
    gen = O.NormalGen(seed)
    nx = gen.normal_vec(g.nodes * o.dim_x, dt).reshape(g.nodes, -1)
    ey = gen.normal_vec(g.edges * o.dim_y, dt).reshape(g.edges, -1)
    ew = gen.normal_vec(g.edges * o.n_w, dt).reshape(g.edges, -1)
    gnz = O.NormalGen(seed + 1).normal_vec(g.nodes * o.dim_z, dt).reshape(g.nodes, -1)
    return nx, ey, ew, gnz


def check(got, want, dt, what):
    err = O.rel_error(got, want)
    assert err <= TOL[dt], f"{what}: rel err {err:.3e} > {TOL[dt]:.0e}"


CASES = [("paper", config("paper")), ("c1", config("c1")), ("c2", config("c2")), ("rand5", random_problem(5))]


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("name,js", CASES, ids=[c[0] for c in CASES])
def test_unfused_conv_matches_oracle(name, js, dt):
    og = O.radius_graph(O.cubic_lattice(5), 1.8)
    keep = (og.src % 7 != 3) & (og.nbr % 11 != 5)  # isolated rows and never-read nodes
    og = O.make_graph(og.nodes, og.src[keep], og.nbr[keep])
    o, pkg = O.Oracle(js), P()
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    nx, ey, ew, gnz = conv_inputs(o, og, dt)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for g in (pkg.Graph(og.nodes, og.src, og.nbr), pkg.make_graph_device(og.nodes, i32(og.src), i32(og.nbr))):
        z = cp.unfused_forward(g, d(nx), d(ey), d(ew))
        check(z.cpu().numpy(), o.conv_forward(og, nx, ey, ew), dt, "unfused forward")
        outs = cp.unfused_backward(g, d(nx), d(ey), d(ew), d(gnz))
        for a, b, n in zip(outs, o.conv_backward(og, nx, ey, ew, gnz), ("g_node_x", "g_edge_y", "g_edge_w")):
            check(a.cpu().numpy(), b, dt, "unfused " + n)


def test_unfused_empty_graph():
    js = config("paper")
    o, pkg = O.Oracle(js), P()
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(3, np.zeros(0, np.int64), np.zeros(0, np.int64))
    nx = torch.randn((3, o.dim_x), device="cuda", dtype=torch.float64)
    z = cp.unfused_forward(g, nx, torch.zeros((0, o.dim_y), device="cuda", dtype=torch.float64),
                           torch.zeros((0, o.n_w), device="cuda", dtype=torch.float64))
    assert z.shape == (3, o.dim_z) and not z.any()
