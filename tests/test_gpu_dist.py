"""The sharded conv C ABI (cgf_conv_*_shard) on one GPU: every rank of a
P-way destination partition is run in turn, the collectives are emulated on
the host (padded all-gather = concatenation, reduce-scatter = sum of the
partials), and the result must equal the oracle's whole-graph conv."""
import numpy as np
import pytest

from oracle import oracle as O
from problems import config

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _inputs(o, g, dt):
    gen = O.NormalGen(1234)
    nx = gen.normal_vec(g.nodes * o.dim_x, dt).reshape(g.nodes, -1)
    ey = gen.normal_vec(g.edges * o.dim_y, dt).reshape(g.edges, -1)
    ew = gen.normal_vec(g.edges * o.n_w, dt).reshape(g.edges, -1)
    gnz = O.NormalGen(1235).normal_vec(g.nodes * o.dim_z, dt).reshape(g.nodes, -1)
    dgx = O.NormalGen(1236).normal_vec(nx.size, dt).reshape(nx.shape)
    dgy = O.NormalGen(1237).normal_vec(ey.size, dt).reshape(ey.shape)
    dgw = O.NormalGen(1238).normal_vec(ew.size, dt).reshape(ew.shape)
    return nx, ey, ew, gnz, dgx, dgy, dgw


@pytest.mark.parametrize("mode", ["det", "atomic"])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cname", ["c1", "c2"])
def test_sharded_conv_equals_whole_graph(cname, world, dt, mode):
    """mode "atomic": the *_shard entry points with CGF_CONV_ATOMIC (the
    shard's CSR / transposed CSR expanded to an edge list on the device)."""
    import paper_2501_13986_b200 as p
    from paper_2501_13986_b200 import dist
    js = config(cname)
    o = O.Oracle(js)
    n, src, nbr = dist.lattice_radius_graph(5, 1.0, 1.8)
    og = O.make_graph(n, src, nbr)
    g = p.Graph(n, src, nbr)
    nx, ey, ew, gnz, dgx, dgy, dgw = _inputs(o, og, dt)
    cp = p.ConvPlan(p.TpPlan(js))
    M = p.ATOMIC if mode == "atomic" else p.DETERMINISTIC
    shards = [dist.GraphShard(g, world, r) for r in range(world)]
    chunk = shards[0].chunk

    def padded(a):  # the all-gathered layout every rank sees
        out = np.zeros((world * chunk, a.shape[1]), a.dtype)
        for s in shards:
            out[s.rank * chunk:s.rank * chunk + s.out_nodes] = a[s.node0:s.node0 + s.out_nodes]
        return torch.from_numpy(out).cuda()

    D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    x_all, dgx_all = padded(nx), padded(dgx)
    z, gy, gw, oy, ow, ogz = [], [], [], [], [], []
    gx_sum = torch.zeros((world * chunk, o.dim_x), dtype=x_all.dtype, device="cuda")
    ox_sum = torch.zeros_like(gx_sum)
    for s in shards:
        n0, n1, e0, e1 = s.node0, s.node0 + s.out_nodes, s.edge0, s.edge0 + s.edges
        z.append(cp.forward_shard(s, x_all, D(ey[e0:e1]), D(ew[e0:e1]), mode=M).cpu().numpy())
        a, b, c = cp.backward_shard(s, x_all, D(ey[e0:e1]), D(ew[e0:e1]), D(gnz[n0:n1]), mode=M)
        gx_sum += a
        gy.append(b.cpu().numpy())
        gw.append(c.cpu().numpy())
        a, b, c, d = cp.double_backward_shard(s, x_all, D(ey[e0:e1]), D(ew[e0:e1]), D(gnz[n0:n1]), dgx_all,
                                              D(dgy[e0:e1]), D(dgw[e0:e1]), mode=M)
        ox_sum += a
        oy.append(b.cpu().numpy())
        ow.append(c.cpu().numpy())
        ogz.append(d.cpu().numpy())

    def unpad(t):
        t = t.cpu().numpy()
        return np.concatenate([t[s.rank * chunk:s.rank * chunk + s.out_nodes] for s in shards])

    want_b = o.conv_backward(og, nx, ey, ew, gnz)
    want_d = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    for got, want, what in ((np.concatenate(z), o.conv_forward(og, nx, ey, ew), "z"),
                            (unpad(gx_sum), want_b[0], "g_node_x"), (np.concatenate(gy), want_b[1], "g_edge_y"),
                            (np.concatenate(gw), want_b[2], "g_edge_w"), (unpad(ox_sum), want_d[0], "dnode_x"),
                            (np.concatenate(oy), want_d[1], "dedge_y"), (np.concatenate(ow), want_d[2], "dedge_w"),
                            (np.concatenate(ogz), want_d[3], "dg_node_z")):
        err = O.rel_error(got, want)
        assert err <= TOL[dt], f"{what}: {err:.3e}"


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
def test_cabi_multi_gpu_conv_world1(dt):
    """The C ABI's multi-GPU conv (cgf_dist_conv_*, NCCL inside libcgf) on a
    1-rank communicator: partition, padded all-gather, all-to-all reduction and
    the ordered sum run for real; results equal the whole-graph ConvPlan
    bitwise (one rank: the same kernels on the same rows). The shard layout
    matches dist.GraphShard's for 3 ranks."""
    import paper_2501_13986_b200 as p
    from paper_2501_13986_b200 import dist
    js = config("c1")
    o = O.Oracle(js)
    n, src, nbr = dist.lattice_radius_graph(5, 1.0, 1.8)
    og = O.make_graph(n, src, nbr)
    g = p.Graph(n, src, nbr)
    for r in range(3):
        ds, gs = dist.DeviceShard(g, 3, r), dist.GraphShard(g, 3, r)
        assert (ds.out_nodes, ds.in_nodes, ds.chunk, ds.edges, ds.node0, ds.edge0) == \
            (gs.out_nodes, gs.in_nodes, gs.chunk, gs.edges, gs.node0, gs.edge0)
    nx, ey, ew, gnz, dgx, dgy, dgw = _inputs(o, og, dt)
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    plan = p.TpPlan(js)
    comm = dist.NcclComm(1, 0, dist.NcclComm.unique_id())
    try:
        dc = dist.CAbiDistConvPlan(plan, dist.DeviceShard(g, 1, 0), comm)
        cp = p.ConvPlan(plan)
        args = (D(nx), D(ey), D(ew))
        assert torch.equal(dc.forward(*args), cp.forward(g, *args))
        for a, b in zip(dc.backward(*args, D(gnz)), cp.backward(g, *args, D(gnz))):
            assert torch.equal(a, b)
        up = (D(dgx), D(dgy), D(dgw))
        for a, b in zip(dc.double_backward(*args, D(gnz), up), cp.double_backward(g, *args, D(gnz), up)):
            assert torch.equal(a, b)
        buf = D(gnz[:7].copy())
        assert torch.equal(dist.allreduce_ordered(buf.clone(), comm), buf)
    finally:
        comm.close()
