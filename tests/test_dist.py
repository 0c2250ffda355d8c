"""Multi-GPU conv host logic on CPU: destination partition,
padded neighbour remap, shard transposed CSR, and the all-gather /
reduce-scatter composition run on world_size-2 gloo ranks.

The CUDA kernels cannot run here, so the ranks use a TEST DOUBLE for the
per-shard compute (the CPU oracle's conv on the shard subgraph); the product
default is the CUDA ``ConvPlan`` (tests/test_gpu_dist.py covers that on a
GPU). The check is that the partitioned result equals the oracle's
whole-graph conv."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from problems import config

torch = pytest.importorskip("torch")


def pkg():
    import paper_2501_13986_b200 as p
    from paper_2501_13986_b200 import dist
    return p, dist


def small_graph():
    g = O.radius_graph(O.cubic_lattice(4), 1.5)
    keep = (g.src % 5 != 2) | (g.nbr % 3 != 1)  # ragged rows
    return O.make_graph(g.nodes, g.src[keep], g.nbr[keep])


def test_lattice_graph_matches_reference_radius_graph():
    _, dist = pkg()
    for n, r in ((4, 1.5), (5, 1.8), (6, 3.0)):
        og = O.radius_graph(O.cubic_lattice(n), r)
        nodes, src, nbr = dist.lattice_radius_graph(n, 1.0, r)
        assert nodes == og.nodes
        np.testing.assert_array_equal(src, og.src)
        np.testing.assert_array_equal(nbr, og.nbr)


def test_lattice_graph_c4_edge_count():
    _, dist = pkg()
    nodes, src, nbr = dist.lattice_radius_graph(29, 1.0, 3.0)
    assert (nodes, src.size) == (24_389, 2_634_962)
    key = src * nodes + nbr
    assert np.all(np.diff(key) > 0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_bounds_balanced_and_covering(world):
    _, dist = pkg()
    g = O.radius_graph(O.cubic_lattice(6), 1.8)
    b = dist.partition_bounds(g.row_ptr, world)
    assert b[0] == 0 and b[-1] == g.nodes and np.all(np.diff(b) >= 0)
    per = np.diff(g.row_ptr[b])
    assert per.sum() == g.edges
    assert per.max() - g.edges / world <= np.diff(g.row_ptr).max()  # within one row of balanced


def test_partition_empty_graph_and_more_ranks_than_nodes():
    _, dist = pkg()
    b = dist.partition_bounds(np.zeros(4, np.int64), 2)
    assert list(b) == [0, 1, 3]
    b = dist.partition_bounds(np.array([0, 1, 2], np.int64), 4)
    assert b[0] == 0 and b[-1] == 2 and np.all(np.diff(b) >= 0)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_shard_remap_and_transpose(world):
    p, dist = pkg()
    og = small_graph()
    g = p.Graph(og.nodes, og.src, og.nbr)
    seen = 0
    for r in range(world):
        sh = dist.GraphShard(g, world, r)
        assert sh.row_ptr[0] == 0 and sh.row_ptr[-1] == sh.edges
        # padded index of each edge's neighbour maps back to the global id
        gl = og.nbr[sh.edge0:sh.edge0 + sh.edges].astype(np.int64)
        np.testing.assert_array_equal(sh.nbr, sh.padded_index(gl))
        own = np.searchsorted(sh.bounds, gl, side="right") - 1
        np.testing.assert_array_equal(sh.nbr - own * sh.chunk + sh.bounds[own], gl)
        # transposed CSR: bucket by padded neighbour, CSR order within a bucket
        tp = sh.t_row_ptr
        assert tp[0] == 0 and tp[-1] == sh.edges and tp.size == sh.in_nodes + 1
        for v in range(sh.in_nodes):
            q = np.arange(tp[v], tp[v + 1])
            assert np.all(sh.nbr[sh.t_eid[q]] == v)
            assert np.all(np.diff(sh.t_eid[q]) > 0)
            srcs = np.searchsorted(sh.row_ptr, sh.t_eid[q], side="right") - 1
            np.testing.assert_array_equal(sh.t_src[q], srcs)
        seen += sh.edges
    assert seen == og.edges


class OracleShardConv:
    """Test double for ConvPlan.*_shard: the CPU oracle's conv on the shard's
    subgraph (nodes = padded neighbour space, rows = local output nodes)."""

    def __init__(self, js):
        self.o = O.Oracle(js)
        self.calls = []

    def _graph(self, sh):
        src = np.repeat(np.arange(sh.out_nodes), np.diff(sh.row_ptr))
        return O.make_graph(sh.in_nodes, src, sh.nbr)

    def _pad(self, a, rows):
        out = np.zeros((rows, a.shape[1]), a.dtype)
        out[:a.shape[0]] = a
        return out

    def forward_shard(self, sh, x_all, ey, ew, mode=0, rows=None, out=None):
        z = self.o.conv_forward(self._graph(sh), x_all.numpy(), ey.numpy(), ew.numpy())
        z = torch.from_numpy(np.ascontiguousarray(z[:sh.out_nodes]))
        if rows is None:
            return z
        self.calls.append(("fwd", tuple(rows)))
        out = torch.full_like(z, float("nan")) if out is None else out  # rows never written stay NaN
        out[rows[0]:rows[1]] = z[rows[0]:rows[1]]
        return out

    def backward_shard(self, sh, x_all, ey, ew, gz, mode=0, rows=None, outs=None):
        gzp = self._pad(gz.numpy(), sh.in_nodes)
        gx, gy, gw = self.o.conv_backward(self._graph(sh), x_all.numpy(), ey.numpy(), ew.numpy(), gzp)
        full = tuple(torch.from_numpy(np.ascontiguousarray(a)) for a in (gx, gy, gw))
        if rows is None:
            return full
        # the kernel contract: neighbour rows [r0, r1) write their g_node_x rows
        # and the g_edge_y / g_edge_w of the edges whose neighbour they are
        self.calls.append(("bwd", tuple(rows)))
        outs = tuple(torch.full_like(a, float("nan")) for a in full) if outs is None else outs
        r0, r1 = rows
        outs[0][r0:r1] = full[0][r0:r1]
        sel = torch.from_numpy((sh.nbr >= r0) & (sh.nbr < r1))
        outs[1][sel] = full[1][sel]
        outs[2][sel] = full[2][sel]
        return outs

    def double_backward_shard(self, sh, x_all, ey, ew, gz, dgx_all, dgy, dgw, mode=0):
        gzp = self._pad(gz.numpy(), sh.in_nodes)
        ox, oy, ow, ogz = self.o.conv_double_backward(self._graph(sh), x_all.numpy(), ey.numpy(), ew.numpy(), gzp,
                                                      dgx_all.numpy(), dgy.numpy(), dgw.numpy())
        return (torch.from_numpy(np.ascontiguousarray(ox)), torch.from_numpy(np.ascontiguousarray(oy)),
                torch.from_numpy(np.ascontiguousarray(ow)), torch.from_numpy(np.ascontiguousarray(ogz[:sh.out_nodes])))


def _inputs(o, g, dt=np.float64):
    gen = O.NormalGen(1234)
    nx = gen.normal_vec(g.nodes * o.dim_x, dt).reshape(g.nodes, -1)
    ey = gen.normal_vec(g.edges * o.dim_y, dt).reshape(g.edges, -1)
    ew = gen.normal_vec(g.edges * o.n_w, dt).reshape(g.edges, -1)
    gnz = O.NormalGen(1235).normal_vec(g.nodes * o.dim_z, dt).reshape(g.nodes, -1)
    dgx = O.NormalGen(1236).normal_vec(nx.size, dt).reshape(nx.shape)
    dgy = O.NormalGen(1237).normal_vec(ey.size, dt).reshape(ey.shape)
    dgw = O.NormalGen(1238).normal_vec(ew.size, dt).reshape(ew.shape)
    return nx, ey, ew, gnz, dgx, dgy, dgw


def ring_graph(n):
    """n nodes, each with its two ring neighbours (sorted CSR): tiny shards whose
    own / local row ranges are empty on some ranks and not on others."""
    src = np.repeat(np.arange(n), 2)
    nbr = np.stack([(np.arange(n) - 1) % n, (np.arange(n) + 1) % n], 1).reshape(-1)
    order = np.lexsort((nbr, src))
    return O.make_graph(n, src[order], nbr[order])


def _rank_main(rank, world, port, js, outdir, overlap=True, graph="small"):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, dist = pkg()
        og = small_graph() if graph == "small" else ring_graph(int(graph[4:]))
        o = O.Oracle(js)
        g = p.Graph(og.nodes, og.src, og.nbr)
        sh = dist.GraphShard(g, world, rank)
        local = OracleShardConv(js)
        dc = dist.DistConvPlan(None, sh, local=local, overlap=overlap)
        nx, ey, ew, gnz, dgx, dgy, dgw = _inputs(o, og)
        n0, n1 = sh.node0, sh.node0 + sh.out_nodes
        e0, e1 = sh.edge0, sh.edge0 + sh.edges
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        z = dc.forward(T(nx[n0:n1]), T(ey[e0:e1]), T(ew[e0:e1]))
        gx, gy, gw = dc.backward(T(nx[n0:n1]), T(ey[e0:e1]), T(ew[e0:e1]), T(gnz[n0:n1]))
        ox, oy, ow, ogz = dc.double_backward(T(nx[n0:n1]), T(ey[e0:e1]), T(ew[e0:e1]), T(gnz[n0:n1]),
                                             (T(dgx[n0:n1]), T(dgy[e0:e1]), T(dgw[e0:e1])))
        np.savez(os.path.join(outdir, f"r{rank}_{int(overlap)}.npz"), n0=n0, n1=n1, e0=e0, e1=e1, z=z.numpy(),
                 gx=gx.numpy(), gy=gy.numpy(), gw=gw.numpy(), ox=ox.numpy(), oy=oy.numpy(), ow=ow.numpy(),
                 ogz=ogz.numpy(), calls=np.array([c[0] + str(c[1]) for c in local.calls] or [""]))
    finally:
        tdist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("overlap", [False, True])
def test_gloo_distributed_conv_matches_whole_graph(world, overlap, tmp_path):
    import torch.multiprocessing as mp
    js = config("c1")
    mp.spawn(_rank_main, args=(world, _free_port(), js, str(tmp_path), overlap), nprocs=world, join=True)
    og = small_graph()
    o = O.Oracle(js)
    nx, ey, ew, gnz, dgx, dgy, dgw = _inputs(o, og)
    want_z = o.conv_forward(og, nx, ey, ew)
    want_b = o.conv_backward(og, nx, ey, ew, gnz)
    want_d = o.conv_double_backward(og, nx, ey, ew, gnz, dgx, dgy, dgw)
    got = {k: [] for k in ("z", "gx", "gy", "gw", "ox", "oy", "ow", "ogz")}
    calls = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}_{int(overlap)}.npz")
        for k in got:
            got[k].append(d[k])
        calls += [c for c in d["calls"].tolist() if c]
    # the overlapped path really splits: row-range forward and backward launches
    assert (any(c.startswith("fwd") for c in calls) and any(c.startswith("bwd") for c in calls)) == overlap
    cat = {k: np.concatenate(v) for k, v in got.items()}
    for k, want in (("z", want_z), ("gx", want_b[0]), ("gy", want_b[1]), ("gw", want_b[2]), ("ox", want_d[0]),
                    ("oy", want_d[1]), ("ow", want_d[2]), ("ogz", want_d[3])):
        assert cat[k].shape == want.shape, k
        assert O.rel_error(cat[k], want) <= 1e-12, k


def test_gloo_overlap_with_empty_ranges_on_some_ranks(tmp_path):
    """13-node ring over 3 ranks: rank 0 has a non-empty own neighbour range,
    ranks 1 and 2 do not. Every rank must still issue the same collectives
    (no rank-dependent fallback), and the result equals the whole graph."""
    import torch.multiprocessing as mp
    p, dist = pkg()
    og = ring_graph(13)
    g = p.Graph(og.nodes, og.src, og.nbr)
    empty = [dist.GraphShard(g, 3, r).own_rows()[0] == dist.GraphShard(g, 3, r).own_rows()[1] for r in range(3)]
    assert any(empty) and not all(empty)
    js = config("c1")
    mp.spawn(_rank_main, args=(3, _free_port(), js, str(tmp_path), True, "ring13"), nprocs=3, join=True)
    o = O.Oracle(js)
    nx, ey, ew, gnz, dgx, dgy, dgw = _inputs(o, og)
    want_z = o.conv_forward(og, nx, ey, ew)
    want_b = o.conv_backward(og, nx, ey, ew, gnz)
    got = {k: np.concatenate([np.load(tmp_path / f"r{r}_1.npz")[k] for r in range(3)]) for k in ("z", "gx", "gy", "gw")}
    for k, want in (("z", want_z), ("gx", want_b[0]), ("gy", want_b[1]), ("gw", want_b[2])):
        assert O.rel_error(got[k], want) <= 1e-12, k


def test_bench_gpus_2_launches_two_ranks_cpu_harness():
    """`bench.py --gpus 2` re-launches itself as 2 torch.distributed ranks; the
    CPU harness mode (gloo, a torch stand-in for the shard kernels) runs the
    multi-rank conv leg's partition / collectives / max-over-ranks plumbing
    and rank 0 prints one line with n_gpus 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--harness-check",
                        "--conv-n", "6", "--conv-steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    rec = json.loads(lines[0])
    assert rec["harness"] and rec["n_gpus"] == 2 and rec["conv"]["n_gpus"] == 2
    assert "all_to_all_single" in rec["conv"]["collectives"]



@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_overlap_row_ranges(world):
    """GraphShard.local_rows: every row in the range reads only the rank's own
    node rows (so it may run during the all-gather), 4-aligned; own_rows: the
    rank's own slot of the padded neighbour rows, 4-aligned. On a lattice the
    local fraction falls as the slabs thin out."""
    p, dist = pkg()
    n, src, nbr = dist.lattice_radius_graph(12, 1.0, 2.0)
    g = p.Graph(n, src, nbr)
    fracs = []
    for r in range(world):
        sh = dist.GraphShard(g, world, r)
        a, b = sh.local_rows()
        assert a % 4 == 0 and b % 4 == 0 and 0 <= a <= b <= sh.out_nodes
        lo, hi = r * sh.chunk, r * sh.chunk + sh.out_nodes
        e0, e1 = sh.row_ptr[a], sh.row_ptr[b]
        assert ((sh.nbr[e0:e1] >= lo) & (sh.nbr[e0:e1] < hi)).all()
        oa, ob = sh.own_rows()
        assert oa % 4 == 0 and ob % 4 == 0 and r * sh.chunk <= oa and ob <= (r + 1) * sh.chunk
        fracs.append((b - a) / max(sh.out_nodes, 1))
    if world == 1:
        assert fracs[0] > 0.99
    else:
        assert min(fracs) < 1.0
