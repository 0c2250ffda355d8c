"""GPU parity at the BASELINE sizes for the
ops the smaller tests cover only at small sizes: sampled rows / nodes / edges
against the CPU oracle (rows and per-node outputs are independent given their
incident edges, so a sample is checked exactly), plus size-independent
properties over the whole batch (exact power-of-two scaling). Tolerances: the
north star's relative L2 1e-5 (FP32) / 1e-12 (FP64)."""
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O
from problems import config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}
DTYPES = [np.float32, np.float64]
ROWS = 1_000_000  # BASELINE configs[1] batch


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.empty_cache()


def P():
    import paper_2501_13986_b200 as pkg
    return pkg


def host(t):
    return t.detach().cpu().numpy()


def check(got, want, dt, what):
    err = O.rel_error(got, want)
    assert err <= TOL[dt], f"{what}: rel err {err:.3e} > {TOL[dt]:.0e}"


def tdtype(dt):
    return torch.float32 if dt == np.float32 else torch.float64


SAMPLE = np.array([0, 1, 2, 31, 32, 127, 128, 4095, ROWS // 3, ROWS // 2, ROWS - 129, ROWS - 2, ROWS - 1])


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c2_full_size_backward_sampled_and_exact_scaling(dt):
    """C2 backward over 1M rows (FP64: 126 GB resident): sampled rows against
    the oracle; gz -> 2 gz doubles gx, gy, gW bit for bit over every row."""
    js = config("c2")
    o, plan = O.Oracle(js), P().TpPlan(js)
    tdt = tdtype(dt)
    g = torch.Generator(device="cuda").manual_seed(21)
    x = torch.randn((ROWS, o.dim_x), device="cuda", dtype=tdt, generator=g)
    y = torch.randn((ROWS, o.dim_y), device="cuda", dtype=tdt, generator=g)
    w = torch.randn((ROWS, o.n_w), device="cuda", dtype=tdt, generator=g)
    gz = torch.randn((ROWS, o.dim_z), device="cuda", dtype=tdt, generator=g)
    idx = torch.from_numpy(SAMPLE).cuda()
    sx, sy, sw, sgz = (host(a[idx]) for a in (x, y, w, gz))
    gx, gy, gw = plan.backward(x, y, w, gz)
    for got, want, n in zip((gx, gy, gw), o.backward(sx, sy, sw, sgz), ("gx", "gy", "gw")):
        check(host(got[idx]), want, dt, f"C2 1M-row backward, sampled {n}")
    sums = [a.double().sum().item() for a in (gx, gy, gw)]
    gz.mul_(2)
    out = plan.backward(x, y, w, gz, out=(gx, gy, gw))
    for a, s, n in zip(out, sums, ("gx", "gy", "gw")):
        assert a.double().sum().item() == 2 * s, n  # exact: every product / sum scales by 2
    del x, y, w, gz, gx, gy, gw, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c2_full_size_forward_f64_and_double_backward(dt):
    """C2 at 1M rows: the FP64 forward (99.5 GB resident) and the
    double-backward — on the device in FP32 (126 GB), through the chunked host
    path in FP64 (226 GB of operands exceed one GPU's HBM) — sampled rows
    against the oracle."""
    js = config("c2")
    o, plan = O.Oracle(js), P().TpPlan(js)
    tdt = tdtype(dt)
    g = torch.Generator(device="cuda").manual_seed(22)
    idx = torch.from_numpy(SAMPLE).cuda()
    if dt == np.float64:
        x = torch.randn((ROWS, o.dim_x), device="cuda", dtype=tdt, generator=g)
        y = torch.randn((ROWS, o.dim_y), device="cuda", dtype=tdt, generator=g)
        w = torch.randn((ROWS, o.n_w), device="cuda", dtype=tdt, generator=g)
        z = plan.forward(x, y, w)
        check(host(z[idx]), o.forward(host(x[idx]), host(y[idx]), host(w[idx])), dt, "C2 1M-row FP64 forward")
        del x, y, w, z
        torch.cuda.empty_cache()
        psutil = pytest.importorskip("psutil")
        need = ROWS * (3 * (o.dim_x + o.dim_y + o.n_w) + 2 * o.dim_z) * 8 * 1.15
        if psutil.virtual_memory().available < need:
            # 1M FP64 rows need 226 GB of operands: more than one B200 (183 GB)
            # and than this host's RAM. Largest resident batch instead.
            _c2_f64_double_backward_device(o, plan, 600_000, g)
            return
        # operands generated on the device in row blocks, staged into host arrays
        shapes = [(o.dim_x,), (o.dim_y,), (o.n_w,), (o.dim_z,), (o.dim_x,), (o.dim_y,), (o.n_w,)]
        arrs = [np.empty((ROWS,) + s, np.float64) for s in shapes]
        blk = 65_536
        for r0 in range(0, ROWS, blk):
            n = min(blk, ROWS - r0)
            for a, s in zip(arrs, shapes):
                a[r0:r0 + n] = host(torch.randn((n,) + s, device="cuda", dtype=tdt, generator=g))
        outs = plan.double_backward(*arrs[:4], tuple(arrs[4:]))
        want = o.double_backward(*(a[SAMPLE] for a in arrs))
        for got, wv, n in zip(outs, want, ("dx", "dy", "dw", "dgz")):
            check(got[SAMPLE], wv, dt, f"C2 1M-row FP64 double-backward (host path), sampled {n}")
        return
    x = torch.randn((ROWS, o.dim_x), device="cuda", dtype=tdt, generator=g)
    y = torch.randn((ROWS, o.dim_y), device="cuda", dtype=tdt, generator=g)
    w = torch.randn((ROWS, o.n_w), device="cuda", dtype=tdt, generator=g)
    gz = torch.randn((ROWS, o.dim_z), device="cuda", dtype=tdt, generator=g)
    up = tuple(torch.randn(a.shape, device="cuda", dtype=tdt, generator=g) for a in (x, y, w))
    outs = plan.double_backward(x, y, w, gz, up)
    want = o.double_backward(*(host(a[idx]) for a in (x, y, w, gz) + up))
    for got, wv, n in zip(outs, want, ("dx", "dy", "dw", "dgz")):
        check(host(got[idx]), wv, dt, f"C2 1M-row double-backward, sampled {n}")
    del x, y, w, gz, up, outs
    torch.cuda.empty_cache()


def _c2_f64_double_backward_device(o, plan, rows, g):
    """FP64 double-backward of `rows` resident rows (600K: 136 GB), sampled rows vs the oracle."""
    tdt = torch.float64
    sample = np.array([0, 1, 31, 32, rows // 2, rows - 1])
    idx = torch.from_numpy(sample).cuda()
    x = torch.randn((rows, o.dim_x), device="cuda", dtype=tdt, generator=g)
    y = torch.randn((rows, o.dim_y), device="cuda", dtype=tdt, generator=g)
    w = torch.randn((rows, o.n_w), device="cuda", dtype=tdt, generator=g)
    gz = torch.randn((rows, o.dim_z), device="cuda", dtype=tdt, generator=g)
    up = tuple(torch.randn(a.shape, device="cuda", dtype=tdt, generator=g) for a in (x, y, w))
    outs = plan.double_backward(x, y, w, gz, up)
    want = o.double_backward(*(host(a[idx]) for a in (x, y, w, gz) + up))
    for got, wv, n in zip(outs, want, ("dx", "dy", "dw", "dgz")):
        check(host(got[idx]), wv, np.float64, f"C2 {rows}-row FP64 double-backward, sampled {n}")
    del x, y, w, gz, up, outs
    torch.cuda.empty_cache()


def _subgraph(og, keep):
    return O.make_graph(og.nodes, og.src[keep], og.nbr[keep]), torch.from_numpy(np.nonzero(keep)[0]).cuda()


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c4_full_graph_double_backward_sampled(dt):
    """C4 double-backward on the full graph (C2 TP, 2,634,962 edges): dL/dg_node_z
    at sampled output nodes, dL/dnode_x at sampled neighbour nodes and the
    per-edge dL/dy, dL/dW of their edges against the oracle's composed conv
    double-backward on the incident-edge subgraph."""
    js = config("c2")
    o, pkg = O.Oracle(js), P()
    from paper_2501_13986_b200 import dist as cdist
    nodes, src, nbr = cdist.lattice_radius_graph(29, 1.0, 3.0)
    og = SimpleNamespace(nodes=nodes, src=src, nbr=nbr, edges=int(src.size))
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(nodes, src, nbr)
    tdt = tdtype(dt)
    gen = torch.Generator(device="cuda").manual_seed(23)
    rnd = lambda *s: torch.randn(s, device="cuda", dtype=tdt, generator=gen)
    nx, ey, ew, gnz = rnd(nodes, o.dim_x), rnd(og.edges, o.dim_y), rnd(og.edges, o.n_w), rnd(nodes, o.dim_z)
    up = (rnd(nodes, o.dim_x), rnd(og.edges, o.dim_y), rnd(og.edges, o.n_w))
    ox, oy, ow, ogz = cp.double_backward(g, nx, ey, ew, gnz, up)
    sample = np.array([0, 1, 12194, nodes - 1])
    hx, hgz, hdx = host(nx), host(gnz), host(up[0])
    sub, eidx = _subgraph(og, np.isin(og.src, sample))  # every edge writing dgz at the sample
    want = o.conv_double_backward(sub, hx, host(ey[eidx]), host(ew[eidx]), hgz, hdx, host(up[1][eidx]),
                                  host(up[2][eidx]))
    check(host(ogz)[sample], want[3][sample], dt, "C4 dL/dg_node_z (sampled nodes)")
    sub, eidx = _subgraph(og, np.isin(og.nbr, sample))  # every edge writing dx at the sample
    want = o.conv_double_backward(sub, hx, host(ey[eidx]), host(ew[eidx]), hgz, hdx, host(up[1][eidx]),
                                  host(up[2][eidx]))
    check(host(ox)[sample], want[0][sample], dt, "C4 dL/dnode_x (sampled nodes)")
    check(host(oy[eidx]), want[1], dt, "C4 dL/dedge_y (sampled edges)")
    check(host(ow[eidx]), want[2], dt, "C4 dL/dedge_w (sampled edges)")


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c5_full_graph_sampled(dt):
    """C5 on one GPU (C1 TP on radius_graph(cubic_lattice(58), 3.0) = 195,112
    nodes / 22,416,384 edges, the bench's conv leg): forward at sampled
    output nodes; FP32 also the backward at sampled neighbour nodes and their
    edges (the FP64 backward's 176 GB of edge operands exceed one GPU)."""
    js = config("c1")
    o, pkg = O.Oracle(js), P()
    from paper_2501_13986_b200 import dist as cdist
    nodes, src, nbr = cdist.lattice_radius_graph(58, 1.0, 3.0)
    assert (nodes, src.size) == (195_112, 22_416_384)
    og = SimpleNamespace(nodes=nodes, src=src, nbr=nbr, edges=int(src.size))
    cp = pkg.ConvPlan(pkg.TpPlan(js))
    g = pkg.Graph(nodes, src, nbr)
    tdt = tdtype(dt)
    gen = torch.Generator(device="cuda").manual_seed(24)
    rnd = lambda *s: torch.randn(s, device="cuda", dtype=tdt, generator=gen)
    nx, ey, ew = rnd(nodes, o.dim_x), rnd(og.edges, o.dim_y), rnd(og.edges, o.n_w)
    z = cp.forward(g, nx, ey, ew)
    sample = np.array([0, 1, 3481, nodes // 2, nodes - 1])
    hx = host(nx)
    sub, eidx = _subgraph(og, np.isin(og.src, sample))
    check(host(z)[sample], o.conv_forward(sub, hx, host(ey[eidx]), host(ew[eidx]))[sample], dt,
          "C5 forward (sampled nodes)")
    del z
    if dt == np.float64:
        return
    gnz = rnd(nodes, o.dim_z)
    gx, gy, gw = cp.backward(g, nx, ey, ew, gnz)
    sub, eidx = _subgraph(og, np.isin(og.nbr, sample))
    wx, wy, ww = o.conv_backward(sub, hx, host(ey[eidx]), host(ew[eidx]), host(gnz))
    check(host(gx)[sample], wx[sample], dt, "C5 g_node_x (sampled nodes)")
    check(host(gy[eidx]), wy, dt, "C5 g_edge_y (sampled edges)")
    check(host(gw[eidx]), ww, dt, "C5 g_edge_w (sampled edges)")


def test_forward_backward_host_entry_matches_separate_calls():
    """cgf_tp_forward_backward_host (one pipelined pass, the e2e path) gives
    bit-identical results to forward_host + backward_host, over several row
    chunks (C2 FP32, 40K rows)."""
    js = config("c2")
    plan = P().TpPlan(js)
    rows = 40_000
    rng = np.random.default_rng(5)
    x, y, w, gz = (rng.standard_normal((rows, d)).astype(np.float32)
                   for d in (plan.dim_x, plan.dim_y, plan.n_w, plan.dim_z))
    z, gx, gy, gw = plan.forward_backward(x, y, w, gz)
    z2 = plan.forward(x, y, w)
    gx2, gy2, gw2 = plan.backward(x, y, w, gz)
    for a, b, n in ((z, z2, "z"), (gx, gx2, "gx"), (gy, gy2, "gy"), (gw, gw2, "gw")):
        assert np.array_equal(a, b), n
    o = O.Oracle(js)
    s = np.array([0, 1, rows // 2, rows - 1])
    check(z[s], o.forward(x[s], y[s], w[s]), np.float32, "fused host entry z")


@pytest.mark.parametrize("ramp", ["0", "1"])
def test_host_pipeline_chunking_is_bitwise_neutral(ramp, monkeypatch):
    """The host path's chunking (1024-row chunks here, CGF_HOST_CHUNK_MB=1; with
    CGF_HOST_RAMP the first / last chunks split into 1/8, 1/4, 1/2 pieces)
    changes nothing: forward_backward on host arrays equals the device calls
    bitwise (C1 FP32, 10,000 rows, a ragged last chunk)."""
    monkeypatch.setenv("CGF_HOST_CHUNK_MB", "1")
    monkeypatch.setenv("CGF_HOST_RAMP", ramp)
    plan = P().TpPlan(config("c1"))
    rows = 10_000
    rng = np.random.default_rng(9)
    x, y, w, gz = (rng.standard_normal((rows, d)).astype(np.float32)
                   for d in (plan.dim_x, plan.dim_y, plan.n_w, plan.dim_z))
    got = plan.forward_backward(x, y, w, gz)
    D = lambda a: torch.from_numpy(a).cuda()
    want = (plan.forward(D(x), D(y), D(w)),) + tuple(plan.backward(D(x), D(y), D(w), D(gz)))
    for a, b, n in zip(got, want, ("z", "gx", "gy", "gw")):
        assert np.array_equal(a, host(b)), n
