"""TEST INFRASTRUCTURE ONLY — Python face of the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module. The product package never does.

Two oracles live here:

* :class:`OracleProblem` + ``liboracle.so`` — our restatement of the reference
  path (``cgoracle.c``). The integer front end (irreps parsing, validation,
  multiplicity splitting, schedule order) is restated below in Python, each
  function citing the reference lines it follows; the arithmetic is in C.
* :class:`RefPlan` — the UNMODIFIED reference (cgforge) built out-of-tree by
  ``oracle/Makefile`` into ``oracle/_ref/libcgforge_ref.so`` and driven through
  ``ref_capi.cpp``. Present in this container and shipped to the GPU box as a
  built ``.so``; tests that need it skip when it is absent.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import re
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libcgforge_ref.so")

# ----------------------------------------------------------------- irreps --


@dataclass(frozen=True)
class MulIrrep:
    mult: int
    l: int
    parity: str  # 'e' | 'o'

    @property
    def dim(self) -> int:
        return self.mult * (2 * self.l + 1)


class ParseError(ValueError):
    pass


def parse_irreps(text: str) -> list[MulIrrep]:
    """``<mult>x<l><e|o>`` blocks joined by '+', textual order, no merging
    (irreps.cpp:60-122)."""
    toks = [t.strip() for t in text.split("+")]
    out = []
    for t in toks:
        m = re.fullmatch(r"(\d+)x(\d+)([eo])", t)
        if not m:
            raise ParseError(f'bad irreps token "{t}"')
        mult, l = int(m.group(1)), int(m.group(2))
        if mult <= 0:
            raise ParseError(f'bad irreps token "{t}": multiplicity must be positive')
        out.append(MulIrrep(mult, l, m.group(3)))
    return out


def offsets(ir: list[MulIrrep]) -> list[int]:
    """Prefix sums of block dims (irreps.cpp:45-49)."""
    o, acc = [], 0
    for b in ir:
        o.append(acc)
        acc += b.dim
    return o + [acc]


# ----------------------------------------------------------------- tpspec --


@dataclass
class Resolved:
    kind: int  # 0 = B (uvu), 1 = C (uvw)
    l1: int
    l2: int
    l3: int
    b: int
    bp: int
    x_off: int
    y_off: int
    z_off: int
    w_off: int
    w_stride: int
    origin: int = 0

    @property
    def dx(self):
        return 2 * self.l1 + 1

    @property
    def dy(self):
        return 2 * self.l2 + 1

    @property
    def dz(self):
        return 2 * self.l3 + 1


class ValidationError(ValueError):
    def __init__(self, violations):
        super().__init__("; ".join(f"instruction {i}: {m}" for i, m in violations))
        self.violations = violations


@dataclass
class OracleProblem:
    x_ir: list
    y_ir: list
    z_ir: list
    instructions: list
    resolved: list = field(default_factory=list)
    dim_x: int = 0
    dim_y: int = 0
    dim_z: int = 0
    n_w: int = 0

    @staticmethod
    def from_json(text_or_dict) -> "OracleProblem":
        """Problem JSON schema (tpspec.cpp:105-130)."""
        d = json.loads(text_or_dict) if isinstance(text_or_dict, str) else text_or_dict
        ins = []
        for tup in d["instructions"]:
            if len(tup) != 4 or tup[3] not in ("B", "C"):
                raise ValueError('instruction must be [x_seg, y_seg, z_seg, "B"|"C"]')
            ins.append((int(tup[0]), int(tup[1]), int(tup[2]), tup[3]))
        return validate(parse_irreps(d["x"]), parse_irreps(d["y"]), parse_irreps(d["z"]), ins)


def validate(x_ir, y_ir, z_ir, instrs) -> OracleProblem:
    """Total validation + offset/weight layout (tpspec.cpp:8-99)."""
    viol = []
    p = OracleProblem(x_ir, y_ir, z_ir, list(instrs))
    xo, yo, zo = offsets(x_ir), offsets(y_ir), offsets(z_ir)
    p.dim_x, p.dim_y, p.dim_z = xo[-1], yo[-1], zo[-1]
    w_off = 0
    for n, (xs, ys, zs, kind) in enumerate(instrs):
        ok = True
        for name, s, ir in (("x", xs, x_ir), ("y", ys, y_ir), ("z", zs, z_ir)):
            if s < 1 or s > len(ir):
                viol.append((n, f"{name} segment index {s} out of range"))
                ok = False
        if not ok:
            continue
        bx, by, bz = x_ir[xs - 1], y_ir[ys - 1], z_ir[zs - 1]
        if by.mult != 1:
            viol.append((n, "y segment multiplicity must be 1 (unsupported pattern)"))
        if kind == "B" and bx.mult != bz.mult:
            viol.append((n, "kind B requires mult(x_seg) == mult(z_seg)"))
        if not (abs(bx.l - by.l) <= bz.l <= bx.l + by.l):
            viol.append((n, "triangle rule violated"))
        if ((bx.parity == "o") != (by.parity == "o")) != (bz.parity == "o"):
            viol.append((n, "parity rule violated: p_x * p_y != p_z"))
        k = 0 if kind == "B" else 1
        cnt = bz.mult if k == 0 else bz.mult * bx.mult
        p.resolved.append(Resolved(k, bx.l, by.l, bz.l, bz.mult, bx.mult, xo[xs - 1], yo[ys - 1],
                                   zo[zs - 1], w_off, 1 if k == 0 else bx.mult, n))
        w_off += cnt
    p.n_w = w_off
    if viol:
        raise ValidationError(viol)
    return p


def split_multiplicities(p: OracleProblem, lane_width: int = 32) -> list[Resolved]:
    """Chunk b, b' to <= lane_width (scheduler.cpp:32-81)."""
    out = []
    for r in p.resolved:
        if r.kind == 0:
            for c0 in range(0, r.b, lane_width):
                ch = min(lane_width, r.b - c0)
                out.append(Resolved(0, r.l1, r.l2, r.l3, ch, ch, r.x_off + c0 * r.dx, r.y_off,
                                    r.z_off + c0 * r.dz, r.w_off + c0, 1, r.origin))
        else:
            for r0 in range(0, r.b, lane_width):
                rc = min(lane_width, r.b - r0)
                for c0 in range(0, r.bp, lane_width):
                    cc = min(lane_width, r.bp - c0)
                    out.append(Resolved(1, r.l1, r.l2, r.l3, rc, cc, r.x_off + c0 * r.dx,
                                        r.y_off, r.z_off + r0 * r.dz,
                                        r.w_off + r0 * r.w_stride + c0, r.w_stride, r.origin))
    return out


def schedule_order(subs: list[Resolved]) -> list[Resolved]:
    """Normalised order: stable sort by z offset (scheduler.cpp:146-151)."""
    return sorted(subs, key=lambda r: r.z_off)


def flop_counts(r: Resolved, nnz: int) -> tuple[int, int]:
    """kernelgen::flop_count of gen_forward / gen_backward for one split
    subkernel (kernelgen.cpp:253-276 applied to :135-251)."""
    dz, dy = r.dz, r.dy
    if r.kind == 0:
        fwd = 3 * r.bp * nnz + 2 * r.b * dz
        bwd = 2 * r.b * dz + 9 * r.bp * nnz + (dy * (r.bp - 1) if r.bp > 1 else 0) + 2 * r.b * dz
    else:
        mm = 2 * r.b * r.bp * dz
        fwd = 3 * r.bp * nnz + mm
        bwd = mm + 9 * r.bp * nnz + (dy * (r.bp - 1) if r.bp > 1 else 0) + mm
    return fwd, bwd


# ---------------------------------------------------------------- C oracle --

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", HERE])
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.cgo_rng_size.restype = C.c_int
        L.cgo_rng_init.argtypes = [P, C.c_uint64]
        L.cgo_rng_normal.restype = C.c_double
        L.cgo_rng_normal.argtypes = [P]
        L.cgo_rng_bits.restype = C.c_uint64
        L.cgo_rng_bits.argtypes = [P]
        L.cgo_rng_fill_f64.argtypes = [P, P, C.c_int64]
        L.cgo_rng_fill_f32.argtypes = [P, P, C.c_int64]
        L.cgo_cg_block.argtypes = [C.c_int] * 4 + [P] * 4
        L.cgo_complex_cg.restype = C.c_double
        L.cgo_complex_cg.argtypes = [C.c_int] * 6
        for suf in ("f32", "f64"):
            getattr(L, f"cgo_tp_forward_{suf}").argtypes = [P] * 5 + [C.c_int64, C.c_int]
            getattr(L, f"cgo_tp_backward_{suf}").argtypes = [P] * 8 + [C.c_int64, C.c_int]
            getattr(L, f"cgo_tp_double_backward_{suf}").argtypes = [P] * 12 + [C.c_int64, C.c_int]
            getattr(L, f"cgo_conv_forward_{suf}").argtypes = (
                [P, C.c_int64, C.c_int64] + [P] * 6 + [C.c_int])
            getattr(L, f"cgo_conv_backward_{suf}").argtypes = (
                [P, C.c_int64, C.c_int64] + [P] * 9 + [C.c_int])
            getattr(L, f"cgo_conv_double_backward_{suf}").argtypes = (
                [P, C.c_int64, C.c_int64] + [P] * 13 + [C.c_int])
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


class NormalGen:
    """rng::NormalGen (rng.hpp:14-53) via the C restatement."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(lib().cgo_rng_size())
        lib().cgo_rng_init(self._buf, C.c_uint64(seed))

    def normal(self) -> float:
        return lib().cgo_rng_normal(self._buf)

    def bits(self) -> int:
        return lib().cgo_rng_bits(self._buf)

    def below(self, n: int) -> int:
        return self.bits() % n

    def normal_vec(self, n: int, dtype=np.float64) -> np.ndarray:
        out = np.empty(int(n), dtype=dtype)
        fn = lib().cgo_rng_fill_f32 if out.dtype == np.float32 else lib().cgo_rng_fill_f64
        fn(self._buf, _ptr(out), C.c_int64(out.size))
        return out


def cg_block(l1: int, l2: int, l3: int):
    """Real-basis CG block entries (k,i,j)-sorted (cg.cpp:58-134)."""
    cap = (2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1)
    i = np.zeros(cap, np.int32)
    j = np.zeros(cap, np.int32)
    k = np.zeros(cap, np.int32)
    v = np.zeros(cap, np.float64)
    n = lib().cgo_cg_block(l1, l2, l3, cap, _ptr(i), _ptr(j), _ptr(k), _ptr(v))
    if n < 0:
        raise ValueError(f"no CG block for ({l1},{l2},{l3})")
    return i[:n].copy(), j[:n].copy(), k[:n].copy(), v[:n].copy()


class _CProblem(C.Structure):
    _fields_ = [("subs", C.c_void_p), ("n", C.c_int32), ("dim_x", C.c_int32),
                ("dim_y", C.c_int32), ("dim_z", C.c_int32), ("n_w", C.c_int32)]


class Oracle:
    """Batched oracle over a problem JSON: split + schedule order, then the C
    restatement of TpPlan / ConvPlan semantics."""

    def __init__(self, problem_json, lane_width: int = 32):
        self.problem = OracleProblem.from_json(problem_json)
        self.subs = schedule_order(split_multiplicities(self.problem, lane_width))
        p = self.problem
        self.dim_x, self.dim_y, self.dim_z, self.n_w = p.dim_x, p.dim_y, p.dim_z, p.n_w
        self._subs = np.array([[r.kind, r.l1, r.l2, r.l3, r.b, r.bp, r.x_off, r.y_off, r.z_off,
                                r.w_off, r.w_stride] for r in self.subs], np.int32).reshape(-1, 11)
        self._cp = _CProblem(self._subs.ctypes.data, len(self.subs), p.dim_x, p.dim_y, p.dim_z,
                             p.n_w)

    def flops_per_row(self) -> tuple[int, int]:
        f = b = 0
        for r in self.subs:
            nnz = len(cg_block(r.l1, r.l2, r.l3)[0])
            a, c = flop_counts(r, nnz)
            f += a
            b += c
        return f, b

    @staticmethod
    def _suf(a):
        return "f32" if a.dtype == np.float32 else "f64"

    def _call(self, name, *args):
        rc = getattr(lib(), name)(C.byref(self._cp), *args)
        if rc != 0:
            raise RuntimeError(f"{name} failed ({rc})")

    def forward(self, x, y, w, w_shared=False):
        rows = x.shape[0]
        z = np.zeros((rows, self.dim_z), x.dtype)
        self._call(f"cgo_tp_forward_{self._suf(x)}", _ptr(x), _ptr(y), _ptr(w), _ptr(z),
                   C.c_int64(rows), int(w_shared))
        return z

    def backward(self, x, y, w, gz, w_shared=False):
        rows = x.shape[0]
        gx = np.zeros_like(x)
        gy = np.zeros_like(y)
        gw = np.zeros((1 if w_shared else rows, self.n_w), x.dtype)
        self._call(f"cgo_tp_backward_{self._suf(x)}", _ptr(x), _ptr(y), _ptr(w), _ptr(gz),
                   _ptr(gx), _ptr(gy), _ptr(gw), C.c_int64(rows), int(w_shared))
        return gx, gy, gw

    def double_backward(self, x, y, w, gz, da, db, dc, w_shared=False):
        rows = x.shape[0]
        ox = np.zeros_like(x)
        oy = np.zeros_like(y)
        ow = np.zeros((1 if w_shared else rows, self.n_w), x.dtype)
        ogz = np.zeros((rows, self.dim_z), x.dtype)
        self._call(f"cgo_tp_double_backward_{self._suf(x)}", _ptr(x), _ptr(y), _ptr(w), _ptr(gz),
                   _ptr(da), _ptr(db), _ptr(dc), _ptr(ox), _ptr(oy), _ptr(ow), _ptr(ogz),
                   C.c_int64(rows), int(w_shared))
        return ox, oy, ow, ogz

    def conv_forward(self, g: "Graph", node_x, edge_y, edge_w, w_shared=False):
        z = np.zeros((g.nodes, self.dim_z), node_x.dtype)
        self._call(f"cgo_conv_forward_{self._suf(node_x)}", C.c_int64(g.nodes),
                   C.c_int64(g.edges), _ptr(g.row_ptr), _ptr(g.nbr), _ptr(node_x), _ptr(edge_y),
                   _ptr(edge_w), _ptr(z), int(w_shared))
        return z

    def conv_backward(self, g: "Graph", node_x, edge_y, edge_w, g_node_z, w_shared=False):
        gx = np.zeros_like(node_x)
        gy = np.zeros_like(edge_y)
        gw = np.zeros((1 if w_shared else g.edges, self.n_w), node_x.dtype)
        self._call(f"cgo_conv_backward_{self._suf(node_x)}", C.c_int64(g.nodes),
                   C.c_int64(g.edges), _ptr(g.src), _ptr(g.nbr), _ptr(node_x), _ptr(edge_y),
                   _ptr(edge_w), _ptr(g_node_z), _ptr(gx), _ptr(gy), _ptr(gw), int(w_shared))
        return gx, gy, gw

    def conv_double_backward(self, g: "Graph", node_x, edge_y, edge_w, g_node_z, d_gx, d_gy,
                             d_gw, w_shared=False):
        ox = np.zeros_like(node_x)
        oy = np.zeros_like(edge_y)
        ow = np.zeros((1 if w_shared else g.edges, self.n_w), node_x.dtype)
        ogz = np.zeros((g.nodes, self.dim_z), node_x.dtype)
        self._call(f"cgo_conv_double_backward_{self._suf(node_x)}", C.c_int64(g.nodes),
                   C.c_int64(g.edges), _ptr(g.src), _ptr(g.nbr), _ptr(node_x), _ptr(edge_y),
                   _ptr(edge_w), _ptr(g_node_z), _ptr(d_gx), _ptr(d_gy), _ptr(d_gw), _ptr(ox),
                   _ptr(oy), _ptr(ow), _ptr(ogz), int(w_shared))
        return ox, oy, ow, ogz


def random_batch(oracle: Oracle, rows: int, seed: int, dtype=np.float64, w_shared=False):
    """engine::random_batch: x, then y, then w from one NormalGen (engine.cpp:394-403).
    With w_shared one W row is drawn."""
    g = NormalGen(seed)
    x = g.normal_vec(rows * oracle.dim_x, dtype).reshape(rows, oracle.dim_x)
    y = g.normal_vec(rows * oracle.dim_y, dtype).reshape(rows, oracle.dim_y)
    w = g.normal_vec((1 if w_shared else rows) * oracle.n_w, dtype).reshape(-1, oracle.n_w)
    return x, y, w


# ------------------------------------------------------------------ graphs --


@dataclass
class Graph:
    nodes: int
    src: np.ndarray  # int32, CSR row (output node), sorted
    nbr: np.ndarray  # int32, neighbour read (reference "dst")
    row_ptr: np.ndarray  # int64, nodes + 1

    @property
    def edges(self) -> int:
        return int(self.src.size)


def make_graph(nodes: int, src, nbr, allow_self_loops=False) -> Graph:
    """Sort by (src, dst), dedup, CSR (conv.cpp:64-87)."""
    src = np.asarray(src, np.int64)
    nbr = np.asarray(nbr, np.int64)
    if src.size and (src.min() < 0 or nbr.min() < 0 or src.max() >= nodes or nbr.max() >= nodes):
        raise ValueError("make_graph: edge endpoint out of range")
    if not allow_self_loops and np.any(src == nbr):
        raise ValueError("make_graph: self-loop")
    key = np.unique(src * nodes + nbr)
    s = (key // nodes).astype(np.int32)
    d = (key % nodes).astype(np.int32)
    rp = np.zeros(nodes + 1, np.int64)
    np.add.at(rp, s.astype(np.int64) + 1, 1)
    return Graph(nodes, s, d, np.cumsum(rp).astype(np.int64))


def cubic_lattice(n: int, spacing: float = 1.0) -> np.ndarray:
    """x-major lattice positions (conv.cpp:153-164)."""
    ix, iy, iz = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return np.stack([ix.ravel() * spacing, iy.ravel() * spacing, iz.ravel() * spacing], 1)


def radius_graph(pos: np.ndarray, r_cut: float) -> Graph:
    """Directed pairs i != j with |r_i - r_j| <= r_cut (conv.cpp:89-133), via a
    cell list; the pair set (not the algorithm) is what make_graph keeps."""
    n = pos.shape[0]
    lo = pos.min(0)
    cell = np.floor((pos - lo) / r_cut).astype(np.int64)
    ncell = cell.max(0) + 1
    cid = (cell[:, 0] * ncell[1] + cell[:, 1]) * ncell[2] + cell[:, 2]
    order = np.argsort(cid, kind="stable")
    cs = cid[order]
    starts = np.searchsorted(cs, np.arange(ncell.prod()), "left")
    ends = np.searchsorted(cs, np.arange(ncell.prod()), "right")
    srcs, dsts = [], []
    r2 = r_cut * r_cut
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                nc = cell + np.array([dx, dy, dz])
                ok = np.all((nc >= 0) & (nc < ncell), 1)
                idx = np.nonzero(ok)[0]
                ncid = (nc[idx, 0] * ncell[1] + nc[idx, 1]) * ncell[2] + nc[idx, 2]
                cnt = ends[ncid] - starts[ncid]
                rep_i = np.repeat(idx, cnt)
                offs = np.concatenate([np.arange(c) for c in cnt]) if cnt.sum() else np.zeros(0, int)
                rep_j = order[np.repeat(starts[ncid], cnt) + offs]
                d = pos[rep_i] - pos[rep_j]
                keep = (np.einsum("ij,ij->i", d, d) <= r2) & (rep_i != rep_j)
                srcs.append(rep_i[keep])
                dsts.append(rep_j[keep])
    return make_graph(n, np.concatenate(srcs), np.concatenate(dsts))


def transpose_permutation(g: Graph) -> np.ndarray:
    """perm[e] = position of edge e in the transposed CSR (conv.cpp:135-151)."""
    cnt = np.zeros(g.nodes + 1, np.int64)
    np.add.at(cnt, g.nbr.astype(np.int64) + 1, 1)
    start = np.cumsum(cnt)[:-1]
    order = np.argsort(g.nbr, kind="stable")  # stable: src ascending within a nbr bucket
    perm = np.empty(g.edges, np.int64)
    perm[order] = np.arange(g.edges)
    del start
    return perm


def rel_error(got, want) -> float:
    """||got - want||_2 / ||want||_2 (tests/helpers.hpp:14-23)."""
    got = np.asarray(got, np.float64).ravel()
    want = np.asarray(want, np.float64).ravel()
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


# ------------------------------------------------------- the reference .so --

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_LIB_PATH)
        P = C.c_void_p
        L.cgr_last_error.restype = C.c_char_p
        L.cgr_plan_create.restype = P
        L.cgr_plan_create.argtypes = [C.c_char_p, C.c_uint32, C.c_int]
        L.cgr_plan_destroy.argtypes = [P]
        L.cgr_plan_info.argtypes = [P, P, P]
        L.cgr_plan_split.argtypes = [P, P, C.c_int]
        L.cgr_emit_text.argtypes = [P, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.cgr_schedule_json.argtypes = [P, C.c_char_p, C.c_int]
        L.cgr_save_array.argtypes = [C.c_char_p, P, C.c_int64, C.c_int64, C.c_int]
        L.cgr_cg_block.argtypes = [C.c_int] * 4 + [P] * 4
        L.cgr_rng_new.restype = P
        L.cgr_rng_new.argtypes = [C.c_uint64]
        L.cgr_rng_free.argtypes = [P]
        L.cgr_rng_normal.argtypes = [P, P, C.c_int64]
        L.cgr_lattice_graph.restype = C.c_int64
        L.cgr_lattice_graph.argtypes = [C.c_int, C.c_double, C.c_double, P, P, C.c_int64]
        L.cgr_transpose_permutation.argtypes = [C.c_int64, C.c_int64, P, P, P]
        for suf in ("f32", "f64"):
            getattr(L, f"cgr_tp_forward_{suf}").argtypes = [P, C.c_int64] + [P] * 4 + [C.c_int] * 2 + [P]
            getattr(L, f"cgr_tp_backward_{suf}").argtypes = [P, C.c_int64] + [P] * 7 + [C.c_int] * 2 + [P]
            getattr(L, f"cgr_tp_double_backward_{suf}").argtypes = (
                [P, C.c_int64] + [P] * 11 + [C.c_int] * 2 + [P])
            getattr(L, f"cgr_conv_forward_{suf}").argtypes = (
                [P, C.c_int64, C.c_int64] + [P] * 6 + [C.c_int] * 4 + [P])
            getattr(L, f"cgr_conv_backward_{suf}").argtypes = (
                [P, C.c_int64, C.c_int64] + [P] * 9 + [C.c_int] * 4 + [P])
            getattr(L, f"cgr_bench_tp_{suf}").argtypes = (
                [P, C.c_int64] + [C.c_int] * 4 + [C.c_uint64, P])
            getattr(L, f"cgr_bench_conv_{suf}").argtypes = (
                [P, C.c_int, C.c_double] + [C.c_int] * 4 + [C.c_uint64, P, P])
        _ref = L
    return _ref


class RefPlan:
    """The reference's own split -> build_schedule -> TpPlan on a problem JSON."""

    def __init__(self, problem_json: str, budget: int = 100000, lane_width: int = 32):
        L = ref_lib()
        if not isinstance(problem_json, str):
            problem_json = json.dumps(problem_json)
        self.h = L.cgr_plan_create(problem_json.encode(), budget, lane_width)
        if not self.h:
            raise ValueError(L.cgr_last_error().decode())
        dims = np.zeros(7, np.int64)
        traffic = np.zeros(3, np.uint64)
        L.cgr_plan_info(self.h, _ptr(dims), _ptr(traffic))
        self.dim_x, self.dim_y, self.dim_z, self.n_w = (int(v) for v in dims[:4])
        self.n_split, self.phases, self.strategy = int(dims[4]), int(dims[5]), int(dims[6])
        self.traffic = tuple(int(v) for v in traffic)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().cgr_plan_destroy(self.h)
            self.h = None

    def split_table(self) -> np.ndarray:
        t = np.zeros((self.n_split, 13), np.int64)
        ref_lib().cgr_plan_split(self.h, _ptr(t), self.n_split)
        return t

    def emit_text(self, pos: int, backward: bool = False) -> str:
        buf = C.create_string_buffer(1 << 20)
        ref_lib().cgr_emit_text(self.h, pos, int(backward), buf, 1 << 20)
        return buf.value.decode()

    def schedule_json(self) -> str:
        buf = C.create_string_buffer(1 << 22)
        ref_lib().cgr_schedule_json(self.h, buf, 1 << 22)
        return buf.value.decode()

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(ref_lib().cgr_last_error().decode())

    @staticmethod
    def _suf(a):
        return "f32" if a.dtype == np.float32 else "f64"

    def forward(self, x, y, w, workers=0, interpreted=False):
        rows = x.shape[0]
        z = np.zeros((rows, self.dim_z), x.dtype)
        st = np.zeros(3, np.uint64)
        self._chk(getattr(ref_lib(), f"cgr_tp_forward_{self._suf(x)}")(
            self.h, rows, _ptr(x), _ptr(y), _ptr(w), _ptr(z), workers, int(interpreted), _ptr(st)))
        self.last_stats = tuple(int(v) for v in st)
        return z

    def backward(self, x, y, w, gz, workers=0, interpreted=False):
        rows = x.shape[0]
        gx, gy, gw = np.zeros_like(x), np.zeros_like(y), np.zeros_like(w)
        st = np.zeros(3, np.uint64)
        self._chk(getattr(ref_lib(), f"cgr_tp_backward_{self._suf(x)}")(
            self.h, rows, _ptr(x), _ptr(y), _ptr(w), _ptr(gz), _ptr(gx), _ptr(gy), _ptr(gw),
            workers, int(interpreted), _ptr(st)))
        self.last_stats = tuple(int(v) for v in st)
        return gx, gy, gw

    def double_backward(self, x, y, w, gz, da, db, dc, seven_call=False, workers=0):
        rows = x.shape[0]
        ox, oy, ow = np.zeros_like(x), np.zeros_like(y), np.zeros_like(w)
        ogz = np.zeros((rows, self.dim_z), x.dtype)
        st = np.zeros(3, np.uint64)
        self._chk(getattr(ref_lib(), f"cgr_tp_double_backward_{self._suf(x)}")(
            self.h, rows, _ptr(x), _ptr(y), _ptr(w), _ptr(gz), _ptr(da), _ptr(db), _ptr(dc),
            _ptr(ox), _ptr(oy), _ptr(ow), _ptr(ogz), int(seven_call), workers, _ptr(st)))
        self.last_stats = tuple(int(v) for v in st)
        return ox, oy, ow, ogz

    def conv_forward(self, g: Graph, node_x, edge_y, edge_w, atomic=False, workers=0, chunks=16,
                     unfused=False):
        z = np.zeros((g.nodes, self.dim_z), node_x.dtype)
        st = np.zeros(4, np.uint64)
        self._chk(getattr(ref_lib(), f"cgr_conv_forward_{self._suf(node_x)}")(
            self.h, g.nodes, g.edges, _ptr(g.src), _ptr(g.nbr), _ptr(node_x), _ptr(edge_y),
            _ptr(edge_w), _ptr(z), int(atomic), workers, chunks, int(unfused), _ptr(st)))
        self.last_stats = tuple(int(v) for v in st)
        return z

    def conv_backward(self, g: Graph, node_x, edge_y, edge_w, g_node_z, atomic=False, workers=0,
                      chunks=16, unfused=False):
        gx, gy, gw = np.zeros_like(node_x), np.zeros_like(edge_y), np.zeros_like(edge_w)
        st = np.zeros(4, np.uint64)
        self._chk(getattr(ref_lib(), f"cgr_conv_backward_{self._suf(node_x)}")(
            self.h, g.nodes, g.edges, _ptr(g.src), _ptr(g.nbr), _ptr(node_x), _ptr(edge_y),
            _ptr(edge_w), _ptr(g_node_z), _ptr(gx), _ptr(gy), _ptr(gw), int(atomic), workers,
            chunks, int(unfused), _ptr(st)))
        self.last_stats = tuple(int(v) for v in st)
        return gx, gy, gw

    def bench_tp(self, dtype, rows, ops=3, warmup=2, iters=5, workers=0, seed=1234):
        secs = np.zeros(3, np.float64)
        suf = "f32" if np.dtype(dtype) == np.float32 else "f64"
        self._chk(getattr(ref_lib(), f"cgr_bench_tp_{suf}")(
            self.h, rows, ops, warmup, iters, workers, seed, _ptr(secs)))
        return secs

    def bench_conv(self, dtype, lattice_n, r_cut=3.0, ops=3, warmup=1, iters=3, workers=0,
                   seed=1234):
        secs = np.zeros(2, np.float64)
        e = np.zeros(1, np.int64)
        suf = "f32" if np.dtype(dtype) == np.float32 else "f64"
        self._chk(getattr(ref_lib(), f"cgr_bench_conv_{suf}")(
            self.h, lattice_n, r_cut, ops, warmup, iters, workers, seed, _ptr(secs), _ptr(e)))
        return secs, int(e[0])


def ref_cg_block(l1, l2, l3):
    cap = (2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1)
    i, j, k = (np.zeros(cap, np.int32) for _ in range(3))
    v = np.zeros(cap, np.float64)
    n = ref_lib().cgr_cg_block(l1, l2, l3, cap, _ptr(i), _ptr(j), _ptr(k), _ptr(v))
    if n < 0:
        raise ValueError(ref_lib().cgr_last_error().decode())
    return i[:n].copy(), j[:n].copy(), k[:n].copy(), v[:n].copy()


def ref_normal(seed: int, n: int) -> np.ndarray:
    L = ref_lib()
    h = L.cgr_rng_new(seed)
    out = np.empty(n, np.float64)
    L.cgr_rng_normal(h, _ptr(out), n)
    L.cgr_rng_free(h)
    return out


def ref_lattice_graph(n: int, spacing=1.0, r_cut=3.0) -> Graph:
    L = ref_lib()
    ne = L.cgr_lattice_graph(n, spacing, r_cut, None, None, 0)
    s = np.zeros(ne, np.int32)
    d = np.zeros(ne, np.int32)
    L.cgr_lattice_graph(n, spacing, r_cut, _ptr(s), _ptr(d), ne)
    return make_graph(n ** 3, s, d)


# --------------------------------------------------------- config problems --

CONFIGS = {
    # SURVEY.md Appendix A (exact JSON).
    "c1": {"x": "32x0e + 32x1o + 32x2e", "y": "1x0e + 1x1o + 1x2e",
           "z": "32x0e + 32x1o + 32x2e + 32x1o + 32x0e + 32x1e + 32x2e + 32x1o + 32x2o + 32x2e + 32x1o + 32x2o + 32x0e + 32x1e + 32x2e",
           "instructions": [[1, 1, 1, "B"], [1, 2, 2, "B"], [1, 3, 3, "B"], [2, 1, 4, "B"],
                            [2, 2, 5, "B"], [2, 2, 6, "B"], [2, 2, 7, "B"], [2, 3, 8, "B"],
                            [2, 3, 9, "B"], [3, 1, 10, "B"], [3, 2, 11, "B"], [3, 2, 12, "B"],
                            [3, 3, 13, "B"], [3, 3, 14, "B"], [3, 3, 15, "B"]]},
    "c2": {"x": "128x0e + 128x1o + 128x2e", "y": "1x0e + 1x1o + 1x2e + 1x3o",
           "z": "128x0e + 128x1o + 128x2e + 128x3o + 128x1o + 128x0e + 128x2e + 128x1o + 128x3o + 128x2e + 128x2e + 128x1o + 128x3o + 128x0e + 128x2e + 128x1o + 128x3o",
           "instructions": [[1, 1, 1, "B"], [1, 2, 2, "B"], [1, 3, 3, "B"], [1, 4, 4, "B"],
                            [2, 1, 5, "B"], [2, 2, 6, "B"], [2, 2, 7, "B"], [2, 3, 8, "B"],
                            [2, 3, 9, "B"], [2, 4, 10, "B"], [3, 1, 11, "B"], [3, 2, 12, "B"],
                            [3, 2, 13, "B"], [3, 3, 14, "B"], [3, 3, 15, "B"], [3, 4, 16, "B"],
                            [3, 4, 17, "B"]]},
    "c3": {"x": "64x0e + 64x1o + 64x2e", "y": "1x0e + 1x1o + 1x2e", "z": "64x0e + 64x1o + 64x2e",
           "instructions": [[1, 1, 1, "C"], [1, 2, 2, "C"], [1, 3, 3, "C"], [2, 1, 2, "C"],
                            [2, 2, 1, "C"], [2, 2, 3, "C"], [2, 3, 2, "C"], [3, 1, 3, "C"],
                            [3, 2, 2, "C"], [3, 3, 1, "C"], [3, 3, 3, "C"]]},
    # tests/helpers.hpp:111-127
    "scalar": {"x": "1x0e", "y": "1x0e", "z": "1x0e", "instructions": [[1, 1, 1, "B"]]},
    "paper": {"x": "32x2e + 32x1e", "y": "1x3e + 1x1e", "z": "32x5e + 16x2e + 32x3e",
              "instructions": [[1, 1, 1, "B"], [1, 2, 2, "C"], [1, 2, 3, "C"]]},
}


def config_json(name: str) -> str:
    return json.dumps(CONFIGS[name])
