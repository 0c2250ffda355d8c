"""GPU parity tests: generated sm_100a TP kernels (through the C ABI) vs the
CPU oracle on identical seeded inputs. Tolerances are the north star's:
relative L2 error <= 1e-5 in FP32 and <= 1e-12 in FP64."""
import json

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


def inputs(o, rows, dt, seed=1234, w_shared=False):
    x, y, w = O.random_batch(o, rows, seed, dt, w_shared=w_shared)
    gz = O.NormalGen(seed + 1).normal_vec(rows * o.dim_z, dt).reshape(rows, -1)
    da = O.NormalGen(seed + 2).normal_vec(x.size, dt).reshape(x.shape)
    db = O.NormalGen(seed + 3).normal_vec(y.size, dt).reshape(y.shape)
    dc = O.NormalGen(seed + 4).normal_vec(w.size, dt).reshape(w.shape)
    return x, y, w, gz, da, db, dc


def check(got, want, dt, what):
    err = O.rel_error(got, want)
    assert err <= TOL[dt], f"{what}: rel err {err:.3e} > {TOL[dt]:.0e}"


CASES = [("scalar", config("scalar"), 7), ("paper", config("paper"), 33), ("c1", config("c1"), 257),
         ("c2", config("c2"), 64), ("c3", config("c3"), 16)] + \
        [(f"rand{s}", random_problem(s), 19) for s in (301, 311, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10)]


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("name,js,rows", CASES, ids=[c[0] for c in CASES])
def test_forward_backward_double_backward(name, js, rows, dt):
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, gz, da, db, dc = inputs(o, rows, dt)
    z = plan.forward(dev(x), dev(y), dev(w))
    check(host(z), o.forward(x, y, w), dt, "forward")
    gx, gy, gw = plan.backward(dev(x), dev(y), dev(w), dev(gz))
    for g, r, n in zip((gx, gy, gw), o.backward(x, y, w, gz), ("gx", "gy", "gw")):
        check(host(g), r, dt, n)
    outs = plan.double_backward(dev(x), dev(y), dev(w), dev(gz), (dev(da), dev(db), dev(dc)))
    for g, r, n in zip(outs, o.double_backward(x, y, w, gz, da, db, dc), ("dx", "dy", "dw", "dgz")):
        check(host(g), r, dt, n)


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_golden_fixture_c2(dt):
    """The committed reference outputs (tests/golden/tp_c2_*.npz) reproduce on the GPU."""
    d = np.load(f"tests/golden/tp_c2_{np.dtype(dt).name}.npz")
    o, plan = O.Oracle(str(d["problem"])), P().TpPlan(str(d["problem"]))
    x, y, w, gz, da, db, dc = inputs(o, int(d["rows"]), dt)
    # golden inputs: gz / da / db / dC come from seeds 1235..1238 as in make_golden.py
    gz = O.NormalGen(1235).normal_vec(gz.size, dt).reshape(gz.shape)
    da = O.NormalGen(1236).normal_vec(x.size, dt).reshape(x.shape)
    db = O.NormalGen(1237).normal_vec(y.size, dt).reshape(y.shape)
    dc = O.NormalGen(1238).normal_vec(w.size, dt).reshape(w.shape)
    check(host(plan.forward(dev(x), dev(y), dev(w))), d["z"], dt, "z")
    for g, k in zip(plan.backward(dev(x), dev(y), dev(w), dev(gz)), ("gx", "gy", "gw")):
        check(host(g), d[k], dt, k)
    outs = plan.double_backward(dev(x), dev(y), dev(w), dev(gz), (dev(da), dev(db), dev(dc)))
    for g, k in zip(outs, ("ox", "oy", "ow", "ogz")):
        check(host(g), d[k], dt, k)


def test_scalar_known_answers():
    plan = P().TpPlan(config("scalar"))
    t = lambda v: torch.tensor([[v]], dtype=torch.float64, device="cuda")
    assert plan.forward(t(2.0), t(3.0), t(0.5)).item() == 3.0
    gx, gy, gw = plan.backward(t(2.0), t(3.0), t(0.5), t(1.0))
    assert (gx.item(), gy.item(), gw.item()) == (1.5, 1.0, 6.0)


def test_empty_batch_and_host_path():
    plan = P().TpPlan(config("c1"))
    o = O.Oracle(config("c1"))
    z = plan.forward(*(torch.empty((0, d), device="cuda") for d in (o.dim_x, o.dim_y, o.n_w)))
    assert z.shape == (0, o.dim_z)
    x, y, w, gz, *_ = inputs(o, 5, np.float64)
    check(plan.forward(x, y, w), o.forward(x, y, w), np.float64, "host forward")
    for g, r in zip(plan.backward(x, y, w, gz), o.backward(x, y, w, gz)):
        check(g, r, np.float64, "host backward")


def test_unaligned_pointers_take_the_copy_path():
    """Views with a 4-byte offset cannot use the bulk-copy engine; results must not change."""
    js = config("c1")
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, *_ = inputs(o, 9, np.float32)
    def off(a):
        buf = torch.zeros(a.size + 1, dtype=torch.float32, device="cuda")
        buf[1:] = dev(a).reshape(-1)
        return buf[1:].view(a.shape)
    z = plan.forward(off(x), off(y), off(w))
    check(host(z), o.forward(x, y, w), np.float32, "unaligned forward")


def test_shape_errors_before_compute():
    pkg = P()
    plan = pkg.TpPlan(config("scalar"))
    with pytest.raises(pkg.ShapeError):
        plan.forward(torch.ones((2, 1), device="cuda"), torch.ones((1, 1), device="cuda"),
                     torch.ones((2, 1), device="cuda"))


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_c3_shared_weights_forward(dt):
    js = config("c3")
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, *_ = inputs(o, 40, dt, w_shared=True)
    z = plan.forward(dev(x), dev(y), dev(w), w_shared=True)
    check(host(z), o.forward(x, y, w, w_shared=True), dt, "shared-W forward")


def test_determinism_bitwise():
    js = config("c2")
    plan = P().TpPlan(js)
    o = O.Oracle(js)
    x, y, w, gz, *_ = inputs(o, 300, np.float64)
    a = plan.backward(dev(x), dev(y), dev(w), dev(gz))
    b = plan.backward(dev(x), dev(y), dev(w), dev(gz))
    for u, v in zip(a, b):
        assert torch.equal(u, v)


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
def test_full_size_c2_sampled_rows_and_linearity(dt):
    """BASELINE size (C2, 1M rows FP32 / 256K FP64): row-sampled parity against the
    oracle plus multilinearity z(2.5 x) = 2.5 z(x) over the full batch."""
    js = config("c2")
    o, plan = O.Oracle(js), P().TpPlan(js)
    rows = 1_000_000 if dt == np.float32 else 262_144
    tdt = torch.float32 if dt == np.float32 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((rows, o.dim_x), device="cuda", dtype=tdt, generator=g)
    y = torch.randn((rows, o.dim_y), device="cuda", dtype=tdt, generator=g)
    w = torch.randn((rows, o.n_w), device="cuda", dtype=tdt, generator=g)
    z = plan.forward(x, y, w)
    idx = torch.tensor([0, 1, 2, rows // 3, rows // 2, rows - 2, rows - 1], device="cuda")
    want = o.forward(host(x[idx]), host(y[idx]), host(w[idx]))
    check(host(z[idx]), want, dt, "sampled rows")
    z2 = plan.forward(x * 2.5, y, w)
    err = (z2 - 2.5 * z).norm() / (2.5 * z).norm()
    assert err.item() <= TOL[dt] * 10


@pytest.mark.parametrize("rows", [1, 127, 128, 1000, 128 * 150 + 37])
def test_c3_shared_w_tensor_core_forward(rows):
    """uvw (kind C) with shared W on tcgen05 (3xTF32): one-tile, tail tile and
    more tiles than SMs (persistent loop) against the FP32 oracle."""
    js = config("c3")
    o, plan = O.Oracle(js), P().TpPlan(js)
    assert "tcgen05.mma" in plan.source(op=0, dtype=0, w_shared=True)
    x, y, w, *_ = inputs(o, rows, np.float32, seed=77, w_shared=True)
    z = plan.forward(dev(x), dev(y), dev(w), w_shared=True)
    torch.cuda.synchronize()
    if rows > 4000:  # the oracle on a row sample (rows are independent)
        idx = np.r_[0:64, rows // 2:rows // 2 + 64, rows - 100:rows]
        check(host(z)[idx], o.forward(x[idx], y[idx], w, w_shared=True), np.float32, "c3 tcgen05 fwd (sampled)")
    else:
        check(host(z), o.forward(x, y, w, w_shared=True), np.float32, "c3 tcgen05 fwd")


def test_c3_tensor_core_matches_simt_path(monkeypatch):
    """The tcgen05 path and the SIMT generator agree on 64K rows; both deterministic."""
    js = config("c3")
    plan = P().TpPlan(js)
    g = torch.Generator(device="cuda").manual_seed(5)
    rows = 65_536
    x = torch.randn((rows, plan.dim_x), device="cuda", generator=g)
    y = torch.randn((rows, plan.dim_y), device="cuda", generator=g)
    w = torch.randn((1, plan.n_w), device="cuda", generator=g)
    a = plan.forward(x, y, w, w_shared=True)
    b = plan.forward(x, y, w, w_shared=True)
    assert torch.equal(a, b)
    monkeypatch.setenv("CGF_UVW", "0")
    c = plan.forward(x, y, w, w_shared=True)
    err = ((a - c).norm() / c.norm()).item()
    assert err <= 1e-5, err


@pytest.mark.parametrize("rows", [1, 127, 1000, 128 * 150 + 37])
def test_c3_shared_w_tensor_core_backward(rows):
    """uvw backward with shared W on tcgen05: gx (transposed forward), gy
    (gzp = W^T gz on the tensor cores + SIMT contraction) and the shared gW
    (rows contracted on the tensor cores, per-CTA partials, fixed-order sum)."""
    js = config("c3")
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, gz, *_ = inputs(o, rows, np.float32, seed=91, w_shared=True)
    gx, gy, gw = plan.backward(dev(x), dev(y), dev(w), dev(gz), w_shared=True)
    a, b, c = plan.backward(dev(x), dev(y), dev(w), dev(gz), w_shared=True)
    assert torch.equal(gx, a) and torch.equal(gy, b) and torch.equal(gw, c)  # deterministic
    wx, wy, ww = o.backward(x, y, w, gz, w_shared=True)
    check(host(gx), wx, np.float32, "c3 gx")
    check(host(gy), wy, np.float32, "c3 gy")
    check(host(gw).reshape(ww.shape), ww, np.float32, "c3 shared gW")


# A wider sweep of the reference's random-problem generator (tests/helpers.hpp:29-109):
# 20 more seeds, ragged batch sizes (1 row, a partial warp, several grid waves).
WIDE = [(s, (1, 7, 131, 1000)[s % 4]) for s in range(11, 31)]


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("seed,rows", WIDE, ids=[f"rand{s}_r{r}" for s, r in WIDE])
def test_random_problem_sweep(seed, rows, dt):
    js = random_problem(seed)
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, gz, da, db, dc = inputs(o, rows, dt, seed=seed)
    check(host(plan.forward(dev(x), dev(y), dev(w))), o.forward(x, y, w), dt, f"{js} forward")
    for g, r, n in zip(plan.backward(dev(x), dev(y), dev(w), dev(gz)), o.backward(x, y, w, gz), ("gx", "gy", "gw")):
        check(host(g), r, dt, n)
    outs = plan.double_backward(dev(x), dev(y), dev(w), dev(gz), (dev(da), dev(db), dev(dc)))
    for g, r, n in zip(outs, o.double_backward(x, y, w, gz, da, db, dc), ("dx", "dy", "dw", "dgz")):
        check(host(g), r, dt, n)


SHARED_CASES = [("c3", config("c3"), 300), ("paper", config("paper"), 257), ("rand301", random_problem(301), 129),
                ("rand2", random_problem(2), 77)]


@pytest.mark.parametrize("dt", DTYPES, ids=["f32", "f64"])
@pytest.mark.parametrize("name,js,rows", SHARED_CASES, ids=[c[0] for c in SHARED_CASES])
def test_shared_w_backward_and_double_backward(name, js, rows, dt, monkeypatch):
    """One W shared by every row (the C3 superset) on the SIMT kernels: the
    per-row weight gradients go to a workspace reduced over rows in a fixed
    order. Backward (FP64, or any shape the tcgen05 path does not take) and
    double-backward (dL/dC shared too) against the oracle's w_shared mode;
    small chunks (CGF_SHARED_W_CHUNK_ROWS) exercise the chunked reduction."""
    monkeypatch.setenv("CGF_SHARED_W_CHUNK_ROWS", "100")
    o, plan = O.Oracle(js), P().TpPlan(js)
    x, y, w, gz, da, db, dc = inputs(o, rows, dt, seed=17, w_shared=True)
    dc = dc[:1]
    monkeypatch.setenv("CGF_UVW", "0")  # the SIMT path, also for C3 FP32
    outs = plan.backward(dev(x), dev(y), dev(w), dev(gz), w_shared=True)
    want = o.backward(x, y, w, gz, w_shared=True)
    for got, wv, n in zip(outs, want, ("gx", "gy", "gw")):
        check(host(got).reshape(wv.shape), wv, dt, f"shared-W {n}")
    again = plan.backward(dev(x), dev(y), dev(w), dev(gz), w_shared=True)
    assert all(torch.equal(a, b) for a, b in zip(outs, again))  # deterministic
    outs = plan.double_backward(dev(x), dev(y), dev(w), dev(gz), (dev(da), dev(db), dev(dc)), w_shared=True)
    want = o.double_backward(x, y, w, gz, da, db, dc, w_shared=True)
    for got, wv, n in zip(outs, want, ("dx", "dy", "dw", "dgz")):
        check(host(got).reshape(wv.shape), wv, dt, f"shared-W double-backward {n}")


def test_array_file_to_device(tmp_path):
    """cgf_array_load into device memory through pinned staging (several
    64 MB pieces) equals the host load."""
    pkg = P()
    a = np.random.default_rng(4).standard_normal((3000, 9001)).astype(np.float32)  # 108 MB
    base = str(tmp_path / "big")
    pkg.save_array(base, a)
    d = pkg.load_array(base, device="cuda")
    assert torch.equal(d.cpu(), torch.from_numpy(a))
