"""Multi-GPU fused convolution: destination-partitioned graph, one rank per GPU.

SURVEY.md §8e. The reference runs the fused conv on one host (``ConvPlan``,
conv.hpp:93-115, conv.cpp:234-528); here the OUTPUT nodes (the reference's
``src``, the CSR row) are split into P contiguous ranges holding ~|E|/P edges
each, and each rank owns its range's node features and its edges' y / W (and
their gradients). Per direction there is exactly one exchange step:

* forward:          all-gather node_x (each rank reads neighbours anywhere),
                    then the local fused conv writes its own node_z rows;
* backward:         local conv backward over the shard's transposed CSR gives
                    PARTIAL g_node_x for every neighbour row, reduce-scattered
                    back to the owners (the adjoint of the all-gather) as an
                    all-to-all + a rank-ordered sum, so FP64 results are
                    bitwise reproducible on any rank count's NCCL setup;
                    g_edge_y / g_edge_w are local;
* double-backward:  all-gather node_x and dL/dg_node_x, reduce-scatter
                    dL/dnode_x; dL/dg_node_z and per-edge terms are local.

There is no weight all-reduce: the reference's conv weights are per edge. The
all-gathered layout is padded: rank r's rows sit at [r*chunk, r*chunk + n_r)
of a P*chunk buffer (``chunk`` = the largest range), so every collective is a
plain equal-split NCCL all_gather_into_tensor / all_to_all_single, and
``GraphShard.nbr`` is pre-remapped into that padded index space on the host.

Overlap (``overlap=True``, the default at P > 1): the forward first runs the
longest run of output rows whose neighbours are all the rank's own nodes while
the all-gather is in flight (in place: the own slot is filled before it starts
and NCCL does not write it), then the remaining rows; the backward first runs
the neighbour rows other ranks own, sends them point to point, and runs its own
rows while they travel. Rows are independent and keep their edge order, and
the partials are still summed in rank order, so the results are bit-identical
to the unoverlapped path. How much hides depends on the partition: for C5
(58^3 lattice, r = 3) the rows with only local neighbours are 90 / 69 / 28 % of
a rank's rows at P = 2 / 4 / 8 (the slabs thin out), and the edges with a local
neighbour (the backward's own rows) 98 / 94 / 86 %.

The local compute is ``ConvPlan.*_shard`` (the generated sm_100a kernels via
the C ABI). ``DistConvPlan`` takes it as ``local`` so the partition and
collective logic can be exercised on CPU ranks (gloo) with a test double.
"""
from __future__ import annotations

import numpy as np

from . import ShapeError, lib, _check

__all__ = ["partition_bounds", "GraphShard", "DistConvPlan", "lattice_radius_graph", "NcclComm", "DeviceShard",
           "CAbiDistConvPlan", "allreduce_ordered"]


def partition_bounds(row_ptr: np.ndarray, world: int) -> np.ndarray:
    """Output-node boundaries b[0..P] with ~|E|/P edges per range (contiguous,
    monotone; ranges may be empty on tiny graphs)."""
    row_ptr = np.asarray(row_ptr, np.int64)
    nodes = row_ptr.size - 1
    edges = int(row_ptr[-1])
    targets = (np.arange(world + 1, dtype=np.float64) * edges / world).round().astype(np.int64)
    b = np.searchsorted(row_ptr, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, nodes
    if edges == 0:  # nothing to balance: split nodes evenly
        b = (np.arange(world + 1, dtype=np.int64) * nodes) // world
    return np.maximum.accumulate(np.minimum(b, nodes))


class GraphShard:
    """Rank ``rank``'s part of a destination-partitioned CSR graph.

    ``graph`` is the global ``Graph`` (host CSR, reference GraphCSR layout).
    Fields: out_nodes (owned output rows), node0 (first owned global node),
    chunk (padded rows per rank), in_nodes = world * chunk, edges, edge0
    (first owned global edge), row_ptr (rebased), nbr (padded index space),
    t_row_ptr / t_src / t_eid (transposed shard CSR)."""

    def __init__(self, graph, world: int, rank: int, bounds: np.ndarray | None = None):
        if not 0 <= rank < world:
            raise ShapeError(f"rank {rank} outside world {world}")
        b = partition_bounds(graph.row_ptr, world) if bounds is None else np.asarray(bounds, np.int64)
        self.world, self.rank, self.bounds = world, rank, b
        self.chunk = max(int(np.max(np.diff(b))), 1)
        self.in_nodes = world * self.chunk
        s0, s1 = int(b[rank]), int(b[rank + 1])
        e0, e1 = int(graph.row_ptr[s0]), int(graph.row_ptr[s1])
        self.node0, self.out_nodes, self.edge0, self.edges = s0, s1 - s0, e0, e1 - e0
        self.row_ptr = np.ascontiguousarray(graph.row_ptr[s0:s1 + 1] - e0)
        gnbr = np.asarray(graph.nbr[e0:e1], np.int64)
        owner = np.searchsorted(b, gnbr, side="right") - 1
        self.nbr = np.ascontiguousarray((owner * self.chunk + gnbr - b[owner]).astype(np.int32))
        self.t_row_ptr = np.zeros(self.in_nodes + 1, np.int64)
        self.t_src = np.zeros(max(self.edges, 1), np.int32)
        self.t_eid = np.zeros(max(self.edges, 1), np.int32)
        _check(lib().cgf_conv_transpose_shard_host(
            self.out_nodes, self.in_nodes, self.edges, self.row_ptr.ctypes.data,
            self.nbr.ctypes.data if self.edges else None, self.t_row_ptr.ctypes.data, self.t_src.ctypes.data,
            self.t_eid.ctypes.data))
        self._dev = {}

    @staticmethod
    def _floor4(v):
        return v - v % 4

    def local_rows(self):
        """(a, b): the longest run of output rows whose neighbours all lie in the
        rank's own slot of the padded buffer, shrunk to multiples of 4 (row-range
        launches keep 16-byte alignment); a == b when there is none."""
        if getattr(self, "_local", None) is None:
            lo, hi = self.rank * self.chunk, self.rank * self.chunk + self.out_nodes
            remote = np.concatenate([[0], np.cumsum((self.nbr < lo) | (self.nbr >= hi))])
            interior = remote[self.row_ptr[1:]] == remote[self.row_ptr[:-1]]
            a = b = best_a = best_b = 0
            for i, ok in enumerate(np.append(interior, False)):
                if ok:
                    b = i + 1
                    continue
                if b - a > best_b - best_a:
                    best_a, best_b = a, b
                a = b = i + 1
            a4, b4 = -(-best_a // 4) * 4, self._floor4(best_b)
            self._local = (a4, b4) if a4 < b4 else (0, 0)
        return self._local

    def own_rows(self):
        """(a, b): the rank's own slot [rank*chunk, (rank+1)*chunk) of the padded
        neighbour rows, shrunk to multiples of 4; the rest are other ranks' rows."""
        lo, hi = self.rank * self.chunk, (self.rank + 1) * self.chunk
        a, b = -(-lo // 4) * 4, self._floor4(hi)
        return (a, b) if a < b else (0, 0)

    def padded_index(self, nodes: np.ndarray) -> np.ndarray:
        """Global node ids -> rows of the padded all-gathered buffer."""
        nodes = np.asarray(nodes, np.int64)
        owner = np.searchsorted(self.bounds, nodes, side="right") - 1
        return owner * self.chunk + nodes - self.bounds[owner]

    def device(self, dev):
        import torch
        key = str(dev)
        if key not in self._dev:
            t = lambda a: torch.from_numpy(a).to(dev)
            self._dev[key] = {k: t(getattr(self, k)) for k in ("row_ptr", "nbr", "t_row_ptr", "t_src", "t_eid")}
        return self._dev[key]


class DistConvPlan:
    """ConvPlan over a destination-partitioned graph (one rank per GPU).

    Inputs / outputs of each call are the rank's own slices: node-indexed
    arrays have ``shard.out_nodes`` rows (the rank's node range), edge arrays
    ``shard.edges`` rows. ``local`` computes the shard (default: the CUDA
    ``ConvPlan``); ``group`` is the torch.distributed process group; ``mode``
    DETERMINISTIC (default) or ATOMIC (Mode::atomic within each shard)."""

    def __init__(self, plan, shard: GraphShard, group=None, local=None, mode=None, overlap=True):
        from . import ConvPlan, DETERMINISTIC
        self.plan, self.shard, self.group = plan, shard, group
        self.mode = DETERMINISTIC if mode is None else mode
        self.local = local if local is not None else ConvPlan(plan)
        # overlapped collectives need row-range launches (deterministic mode only);
        # "force" also overlaps on one rank (tests: the same code path on one GPU)
        self.overlap = bool(overlap) and self.mode == DETERMINISTIC and (shard.world > 1 or overlap == "force")
        self._gather_cache = {}

    # -- collectives -----------------------------------------------------------
    def _all_gather(self, a, key=None):
        """[out_nodes, d] per rank -> [world * chunk, d] padded, on every rank."""
        import torch.distributed as dist
        sh = self.shard
        if a.shape[0] != sh.out_nodes:
            raise ShapeError(f"expected {sh.out_nodes} local node rows, got {a.shape[0]}")
        if sh.world == 1 and sh.chunk == sh.out_nodes:
            return a
        buf = a.new_zeros((sh.chunk, a.shape[1]))
        buf[:sh.out_nodes] = a
        out = a.new_empty((sh.in_nodes, a.shape[1]))
        dist.all_gather_into_tensor(out, buf, group=self.group)
        return out

    def _all_gather_async(self, a):
        """In-place padded all-gather started on the communicator's stream: the
        own slot is written here first (NCCL does not write it), so kernels on
        the current stream may read it while the other slots arrive. Returns
        (buffer, work); work.wait() orders the current stream after it."""
        import torch.distributed as dist
        sh = self.shard
        if a.shape[0] != sh.out_nodes:
            raise ShapeError(f"expected {sh.out_nodes} local node rows, got {a.shape[0]}")
        out = a.new_empty((sh.in_nodes, a.shape[1]))
        own = out[sh.rank * sh.chunk:(sh.rank + 1) * sh.chunk]
        own[:sh.out_nodes] = a
        own[sh.out_nodes:] = 0
        return out, dist.all_gather_into_tensor(out, own, group=self.group, async_op=True)

    def _send_partials_async(self, partial):
        """Point-to-point exchange of the other ranks' slots of ``partial`` (the
        all-to-all minus the own slot, which may still be computing). Returns
        (received [world, chunk, d], requests)."""
        import torch.distributed as dist
        sh = self.shard
        recv = partial.new_empty((sh.world, sh.chunk, partial.shape[1]))
        ops = []
        for r in range(sh.world):
            if r == sh.rank:
                continue
            ops.append(dist.P2POp(dist.isend, partial[r * sh.chunk:(r + 1) * sh.chunk], r, group=self.group))
            ops.append(dist.P2POp(dist.irecv, recv[r], r, group=self.group))
        return recv, dist.batch_isend_irecv(ops) if ops else []

    def _ordered_sum(self, recv, partial):
        """This rank's rows: the partials of every rank summed in rank order (own
        rank from ``partial``), the order ``_reduce_scatter`` uses."""
        sh = self.shard
        part = lambda r: (partial[sh.rank * sh.chunk:sh.rank * sh.chunk + sh.out_nodes] if r == sh.rank
                          else recv[r, :sh.out_nodes])
        out = part(0).clone()
        for r in range(1, sh.world):
            out += part(r)
        return out

    def _reduce_scatter(self, partial):
        """[world * chunk, d] partial sums -> this rank's [out_nodes, d] totals.

        Deterministic: an all-to-all delivers every rank's partial rows of this
        rank's range (the same bytes a reduce-scatter moves), then they are
        summed here in rank order, so the result does not depend on the NCCL
        algorithm / protocol or on the number of channels (a plain
        reduce_scatter_tensor may reduce in any order)."""
        import torch.distributed as dist
        sh = self.shard
        if sh.world == 1:
            return partial[:sh.out_nodes]
        parts = partial.new_empty(partial.shape)
        dist.all_to_all_single(parts, partial.contiguous(), group=self.group)
        parts = parts.view(sh.world, sh.chunk, partial.shape[1])
        out = parts[0, :sh.out_nodes].clone()
        for r in range(1, sh.world):
            out += parts[r, :sh.out_nodes]
        return out

    # -- the three entry points -------------------------------------------------
    def forward(self, node_x, edge_y, edge_w):
        return self.forward_gathered(node_x, edge_y, edge_w)[0]

    def forward_gathered(self, node_x, edge_y, edge_w):
        """(node_z rows of this rank, the padded all-gathered node_x) — the
        latter reusable by ``backward(node_x_all=...)``."""
        # the collective a rank issues must not depend on its own row ranges
        # (ranks with an empty local range still take the overlapped path)
        sh = self.shard
        if not self.overlap:
            x_all = self._all_gather(node_x)
            return self.local.forward_shard(sh, x_all, edge_y, edge_w, mode=self.mode), x_all
        a, b = sh.local_rows()
        x_all, work = self._all_gather_async(node_x)
        z = self.local.forward_shard(sh, x_all, edge_y, edge_w, mode=self.mode, rows=(a, b))
        work.wait()
        for r0, r1 in ((0, a), (b, sh.out_nodes)):
            if r0 < r1:
                self.local.forward_shard(sh, x_all, edge_y, edge_w, mode=self.mode, rows=(r0, r1), out=z)
        return z, x_all

    def backward(self, node_x, edge_y, edge_w, g_node_z, node_x_all=None):
        sh = self.shard
        x_all = self._all_gather(node_x) if node_x_all is None else node_x_all
        if not self.overlap:
            gx_part, gy, gw = self.local.backward_shard(sh, x_all, edge_y, edge_w, g_node_z, mode=self.mode)
            return self._reduce_scatter(gx_part), gy, gw
        # every rank exchanges point to point here, also one whose own range is
        # empty (then all its rows run before the exchange)
        a, b = sh.own_rows()
        outs = None
        for r0, r1 in ((0, a), (b, sh.in_nodes)):  # other ranks' neighbour rows first
            if r0 < r1:
                outs = self.local.backward_shard(sh, x_all, edge_y, edge_w, g_node_z, mode=self.mode,
                                                 rows=(r0, r1), outs=outs)
        if outs is None:
            outs = self.local.backward_shard(sh, x_all, edge_y, edge_w, g_node_z, mode=self.mode, rows=(0, 0))
        recv, reqs = self._send_partials_async(outs[0])
        gx_part, gy, gw = self.local.backward_shard(sh, x_all, edge_y, edge_w, g_node_z, mode=self.mode,
                                                    rows=(a, b), outs=outs)
        for q in reqs:
            q.wait()
        return self._ordered_sum(recv, gx_part), gy, gw

    def double_backward(self, node_x, edge_y, edge_w, g_node_z, upstream):
        d_gx, d_gy, d_gw = upstream
        x_all = self._all_gather(node_x)
        dgx_all = self._all_gather(d_gx)
        ox_part, oy, ow, ogz = self.local.double_backward_shard(self.shard, x_all, edge_y, edge_w, g_node_z,
                                                                dgx_all, d_gy, d_gw, mode=self.mode)
        return self._reduce_scatter(ox_part), oy, ow, ogz

    def gather_x(self, node_x):
        """The padded all-gathered node features (reusable across fwd / bwd)."""
        return self._all_gather(node_x)


def lattice_radius_graph(n: int, spacing: float = 1.0, r_cut: float = 3.0):
    """``conv::radius_graph(conv::cubic_lattice(n, n, n, spacing), r_cut)``
    (conv.cpp:89-133, 153-164) for the benchmark graphs C4 / C5, built directly
    from the lattice's neighbour offsets: node id = (i * n + j) * n + k, edges
    (s, d) for every d != s within r_cut, sorted by (s, d). Returns (nodes,
    src int64, nbr int64)."""
    R = int(np.floor(r_cut / spacing + 1e-9))
    offs = [(a, b, c) for a in range(-R, R + 1) for b in range(-R, R + 1) for c in range(-R, R + 1)
            if (a, b, c) != (0, 0, 0) and (a * a + b * b + c * c) * spacing * spacing <= r_cut * r_cut + 1e-9]
    # neighbour id delta is monotone in the (a, b, c) lexicographic order, so
    # emitting offsets in that order per source keeps (s, d) sorted.
    offs.sort()
    idx = np.arange(n, dtype=np.int64)
    ii, jj, kk = np.meshgrid(idx, idx, idx, indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    nodes = n ** 3
    valid = np.zeros((nodes, len(offs)), dtype=bool)
    for t, (a, b, c) in enumerate(offs):
        valid[:, t] = ((ii + a >= 0) & (ii + a < n) & (jj + b >= 0) & (jj + b < n) & (kk + c >= 0) & (kk + c < n))
    delta = np.array([(a * n + b) * n + c for a, b, c in offs], dtype=np.int64)
    s_idx, t_idx = np.nonzero(valid)  # row-major: by source, then offset order
    src = s_idx.astype(np.int64)
    nbr = src + delta[t_idx]
    return nodes, src, nbr


# ------------------------------------------------ the C ABI's multi-GPU path --

class NcclComm:
    """An NCCL communicator made through the C ABI (cgf_nccl_*): for callers
    that drive the C-ABI multi-GPU conv without torch.distributed. ``uid`` is
    the 128-byte id from ``NcclComm.unique_id()`` on one rank, shared out of
    band."""

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        buf = C.create_string_buffer(128)
        _check(lib().cgf_nccl_unique_id(buf))
        return buf.raw

    def __init__(self, world: int, rank: int, uid: bytes):
        import ctypes as C
        h = C.c_void_p()
        _check(lib().cgf_nccl_comm_create(world, rank, uid, C.byref(h)))
        self.world, self.rank, self.h = world, rank, h

    def close(self):
        if self.h:
            _check(lib().cgf_nccl_comm_destroy(self.h))
            self.h = None


class DeviceShard:
    """cgf_conv_shard: rank ``rank``'s part of a host CSR graph, partitioned
    and uploaded by libcgf (the same partition as GraphShard)."""

    def __init__(self, graph, world: int, rank: int):
        import ctypes as C
        h = C.c_void_p()
        _check(lib().cgf_conv_shard_create(graph.nodes, graph.edges, graph.row_ptr.ctypes.data,
                                           graph.nbr.ctypes.data if graph.edges else None, world, rank, C.byref(h)))
        self.h = h
        info = np.zeros(6, np.int64)
        _check(lib().cgf_conv_shard_info(h, info.ctypes.data))
        self.out_nodes, self.in_nodes, self.chunk, self.edges, self.node0, self.edge0 = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "h", None):
            lib().cgf_conv_shard_destroy(self.h)
            self.h = None


class CAbiDistConvPlan:
    """The multi-GPU conv through the C ABI (cgf_dist_conv_*): NCCL all-gather
    of node_x / all-to-all + rank-ordered reduction of g_node_x inside libcgf,
    on torch CUDA tensors of the rank's rows."""

    def __init__(self, plan, shard: DeviceShard, comm: NcclComm, mode=None):
        from . import DETERMINISTIC
        self.plan, self.shard, self.comm = plan, shard, comm
        self.mode = DETERMINISTIC if mode is None else mode

    def _call(self, fn, dt, *arrays, ref):
        import ctypes as C
        import torch
        from . import _dtype_code
        st = C.c_void_p(torch.cuda.current_stream(ref.device).cuda_stream)
        _check(fn(self.plan._h, _dtype_code(ref), self.shard.h, self.comm.h,
                  *(C.c_void_p(a.data_ptr()) for a in arrays), self.mode, st))

    def forward(self, node_x, edge_y, edge_w):
        p, sh = self.plan, self.shard
        z = node_x.new_empty((sh.out_nodes, p.dim_z))
        self._call(lib().cgf_dist_conv_forward, None, node_x, edge_y, edge_w, z, ref=node_x)
        return z

    def backward(self, node_x, edge_y, edge_w, g_node_z):
        p, sh = self.plan, self.shard
        gx = node_x.new_empty((sh.out_nodes, p.dim_x))
        gy, gw = torch_like(edge_y), torch_like(edge_w)
        self._call(lib().cgf_dist_conv_backward, None, node_x, edge_y, edge_w, g_node_z, gx, gy, gw, ref=node_x)
        return gx, gy, gw

    def double_backward(self, node_x, edge_y, edge_w, g_node_z, upstream):
        p, sh = self.plan, self.shard
        d_gx, d_gy, d_gw = upstream
        ox = node_x.new_empty((sh.out_nodes, p.dim_x))
        oy, ow = torch_like(edge_y), torch_like(edge_w)
        ogz = node_x.new_empty((sh.out_nodes, p.dim_z))
        self._call(lib().cgf_dist_conv_double_backward, None, node_x, edge_y, edge_w, g_node_z, d_gx, d_gy, d_gw,
                   ox, oy, ow, ogz, ref=node_x)
        return ox, oy, ow, ogz


def torch_like(a):
    return a.new_empty(a.shape)


def allreduce_ordered(buf, comm: NcclComm):
    """In-place deterministic sum over ranks (cgf_dist_allreduce_ordered)."""
    import ctypes as C
    import torch
    from . import _dtype_code
    st = C.c_void_p(torch.cuda.current_stream(buf.device).cuda_stream)
    _check(lib().cgf_dist_allreduce_ordered(_dtype_code(buf), comm.h, comm.world, C.c_void_p(buf.data_ptr()),
                                            buf.numel(), st))
    return buf
