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
@pytest.mark.parametrize("cname", ["c1", "c2"])
def test_row_range_shard_calls_bitwise(cname, dt):
    """The row-range shard launches the overlapped multi-GPU path makes
    (dist.DistConvPlan: local-neighbour rows during the all-gather, the rest
    after; other ranks' neighbour rows before the exchange, own rows during it)
    reproduce one whole-shard launch bit for bit, for the ranges the shard
    computes and for arbitrary 4-aligned splits."""
    import paper_2501_13986_b200 as p
    from paper_2501_13986_b200 import dist
    js = config(cname)
    o = O.Oracle(js)
    n, src, nbr = dist.lattice_radius_graph(7, 1.0, 1.8)
    og = O.make_graph(n, src, nbr)
    g = p.Graph(n, src, nbr)
    nx, ey, ew, gnz, _, _, _ = _inputs(o, og, dt)
    cp = p.ConvPlan(p.TpPlan(js))
    D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    world = 3
    shards = [dist.GraphShard(g, world, r) for r in range(world)]
    chunk = shards[0].chunk
    x_all = np.zeros((world * chunk, o.dim_x), dt)
    for s in shards:
        x_all[s.rank * chunk:s.rank * chunk + s.out_nodes] = nx[s.node0:s.node0 + s.out_nodes]
    x_all = D(x_all)
    for s in shards:
        n0, n1, e0, e1 = s.node0, s.node0 + s.out_nodes, s.edge0, s.edge0 + s.edges
        y, w, gz = D(ey[e0:e1]), D(ew[e0:e1]), D(gnz[n0:n1])
        z_ref = cp.forward_shard(s, x_all, y, w)
        b_ref = cp.backward_shard(s, x_all, y, w, gz)
        a, b = s.local_rows()
        for cuts in ([0, a, b, s.out_nodes], [0, 8, 20, s.out_nodes], [0, s.out_nodes]):
            cuts = sorted(set(min(c, s.out_nodes) for c in cuts))
            z = None
            for r0, r1 in zip(cuts, cuts[1:]):
                z = cp.forward_shard(s, x_all, y, w, rows=(r0, r1), out=z)
            assert torch.equal(z, z_ref), (s.rank, cuts)
        a, b = s.own_rows()
        for order in ([(0, a), (b, s.in_nodes), (a, b)], [(0, 12), (12, s.in_nodes)]):
            outs = None
            for r0, r1 in order:
                outs = cp.backward_shard(s, x_all, y, w, gz, rows=(r0, r1), outs=outs)
            for got, want in zip(outs, b_ref):
                assert torch.equal(got, want), (s.rank, order)
    s = shards[0]
    with pytest.raises(p.ShapeError):
        cp.forward_shard(s, x_all, D(ey[:s.edges]), D(ew[:s.edges]), rows=(2, 5))  # unaligned start
    with pytest.raises(p.ShapeError):
        cp.forward_shard(s, x_all, D(ey[:s.edges]), D(ew[:s.edges]), rows=(0, s.out_nodes + 1))


def test_overlapped_dist_conv_plan_nccl_one_rank():
    """DistConvPlan's overlapped path (in-place async all-gather, row-range
    launches on both sides of work.wait(), own-row backward during the
    exchange, rank-ordered sum) forced on a 1-rank NCCL process group: the same
    torch.distributed calls and streams as at N > 1, bit-identical to the
    whole-graph ConvPlan."""
    import os
    import socket

    import torch.distributed as tdist

    import paper_2501_13986_b200 as p
    from paper_2501_13986_b200 import dist
    if tdist.is_initialized():
        pytest.skip("a process group already exists in this process")
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        js = config("c1")
        o = O.Oracle(js)
        n, src, nbr = dist.lattice_radius_graph(7, 1.0, 1.8)
        og = O.make_graph(n, src, nbr)
        g = p.Graph(n, src, nbr)
        D = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        nx, ey, ew, gnz, _, _, _ = (D(a) for a in _inputs(o, og, np.float32))
        plan = p.TpPlan(js)
        sh = dist.GraphShard(g, 1, 0)
        assert sh.local_rows()[1] > 0 and sh.own_rows()[1] > 0
        dc = dist.DistConvPlan(plan, sh, overlap="force")
        assert dc.overlap
        cp = p.ConvPlan(plan)
        z, x_all = dc.forward_gathered(nx, ey, ew)
        assert torch.equal(z, cp.forward(g, nx, ey, ew))
        for a, b in zip(dc.backward(nx, ey, ew, gnz, node_x_all=x_all), cp.backward(g, nx, ey, ew, gnz)):
            assert torch.equal(a, b)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("overlap", ["0", "force"])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
def test_cabi_multi_gpu_conv_world1(dt, overlap, monkeypatch):
    """The C ABI's multi-GPU conv (cgf_dist_conv_*, NCCL inside libcgf) on a
    1-rank communicator: partition, padded all-gather, all-to-all reduction and
    the ordered sum run for real; results equal the whole-graph ConvPlan
    bitwise (one rank: the same kernels on the same rows). The shard layout
    matches dist.GraphShard's for 3 ranks. overlap="force": the overlapped
    scheme (in-place all-gather on the shard's comm stream during the
    local-neighbour rows, own rows during the exchange) on the one rank."""
    monkeypatch.setenv("CGF_DIST_OVERLAP", overlap)
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
