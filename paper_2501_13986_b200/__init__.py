"""B200-native CG tensor-product kernels (arXiv 2501.13986), Python face.

A thin ctypes binding over ``libcgf.so`` (the C ABI in ``include/cgf.h``) that
mirrors the reference's C++ operator API (``cgforge::engine::TpPlan``,
``cgforge::conv::ConvPlan``; /root/reference/proj/include/cgforge/) with the
same names, argument meaning and error behaviour:

    plan = TpPlan(problem_json)                  # parse -> validate -> split -> plan
    z = plan.forward(x, y, w)                    # TpPlan::forward   (engine.hpp:82)
    gx, gy, gw = plan.backward(x, y, w, gz)      # TpPlan::backward  (engine.hpp:85)
    dx, dy, dw, dgz = plan.double_backward(x, y, w, gz, (da, db, dc))   # (engine.hpp:91)

Arrays are torch CUDA tensors (computed in place on the device, on the current
stream) or numpy arrays (the host path: copy in, compute, copy out). There is
no CPU fallback: the compute path is the generated sm_100a kernels, and a
missing ``libcgf.so`` or CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcgf.so")

__all__ = [
    "save_array", "load_array", "read_meta",
    "TpPlan", "ConvPlan", "Graph", "DeviceGraph", "make_graph_device", "radius_graph_device", "cg_block", "lib", "CgfError", "ParseError", "ValidationError", "ShapeError",
    "BudgetError", "TriangleError", "InvalidArgument", "CudaError", "JitError",
    "UnsupportedError", "F32", "F64", "OP_FORWARD", "OP_BACKWARD", "OP_DOUBLE_BACKWARD", "DETERMINISTIC", "ATOMIC",
]

F32, F64 = 0, 1
OP_FORWARD, OP_BACKWARD, OP_DOUBLE_BACKWARD = 0, 1, 2


class CgfError(RuntimeError):
    code = 0


class ParseError(CgfError, ValueError):  # irreps::ParseError
    code = 1


class ValidationError(CgfError, ValueError):  # tpspec::validate violations
    code = 2


class ShapeError(CgfError, ValueError):  # engine::ShapeError
    code = 3


class BudgetError(CgfError):  # scheduler::BudgetError
    code = 4


class TriangleError(CgfError, ValueError):  # cg::TriangleError
    code = 5


class InvalidArgument(CgfError, ValueError):  # std::invalid_argument
    code = 6


class CudaError(CgfError):
    code = 7


class JitError(CgfError):
    code = 8


class UnsupportedError(CgfError):
    code = 9


class InternalError(CgfError):
    code = 10


from . import configs  # noqa: E402  (benchmark problem JSONs)

_ERRORS = {c.code: c for c in (ParseError, ValidationError, ShapeError, BudgetError, TriangleError,
                               InvalidArgument, CudaError, JitError, UnsupportedError, InternalError)}

_lib = None


def lib():
    """Loads libcgf.so (built by ``__graft_entry__.build()`` / ``make -C
    paper_2501_13986_b200``). Raises if it is missing — there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `make -C {_HERE}` or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, I64, I = C.c_void_p, C.c_int64, C.c_int
    L.cgf_last_error.restype = C.c_char_p
    L.cgf_version.restype = C.c_char_p
    L.cgf_cg_block.argtypes = [I, I, I, I, P, P, P, P]
    L.cgf_plan_create.argtypes = [C.c_char_p, I, C.c_uint32, C.POINTER(P)]
    L.cgf_plan_destroy.argtypes = [P]
    L.cgf_plan_dims.argtypes = [P, P]
    L.cgf_plan_flops.argtypes = [P, P]
    L.cgf_plan_source.argtypes = [P, I, I, I, I, C.c_char_p, I]
    L.cgf_plan_compile.argtypes = [P, I, I, I, I]
    L.cgf_tp_forward.argtypes = [P, I, P, P, P, P, I64, I, P]
    L.cgf_tp_backward.argtypes = [P, I, P, P, P, P, P, P, P, I64, I, P]
    L.cgf_tp_double_backward.argtypes = [P, I] + [P] * 11 + [I64, I, P]
    L.cgf_tp_forward_host.argtypes = [P, I, P, P, P, P, I64, I]
    L.cgf_tp_backward_host.argtypes = [P, I] + [P] * 7 + [I64, I]
    L.cgf_tp_double_backward_host.argtypes = [P, I] + [P] * 11 + [I64, I]
    L.cgf_tp_forward_backward_host.argtypes = [P, I] + [P] * 8 + [I64, I]
    L.cgf_tp_stats.argtypes = [P, I, I64, I, P]
    L.cgf_tp_traffic.argtypes = [P, I, I64, I, P]
    L.cgf_plan_schedule_json.argtypes = [P, C.c_char_p, I]
    L.cgf_plan_listing.argtypes = [P, I, I, C.c_char_p, I]
    L.cgf_conv_stats.argtypes = [P, I, I, I, I64, I64, P]
    L.cgf_plan_kernel_source.argtypes = [P, I, I, I, I, I, C.c_char_p, I]
    L.cgf_plan_kernel_compile.argtypes = [P, I, I, I, I, I]
    L.cgf_plan_kernel_groups.argtypes = [P, I, I, I]
    L.cgf_plan_kernel_source_group.argtypes = [P, I, I, I, I, I, I, C.c_char_p, I]
    L.cgf_conv_transpose_host.argtypes = [I64, I64, P, P, P, P, P]
    L.cgf_conv_forward.argtypes = [P, I, I64, I64, P, P, P, P, P, P, I, P]
    L.cgf_conv_backward.argtypes = [P, I, I64, I64] + [P] * 12 + [I, P]
    L.cgf_conv_double_backward.argtypes = [P, I, I64, I64] + [P] * 16 + [I, P]
    L.cgf_conv_transpose_shard_host.argtypes = [I64, I64, I64, P, P, P, P, P]
    L.cgf_conv_forward_shard.argtypes = [P, I, I64, I64, I64, P, P, P, P, P, P, I, P]
    L.cgf_conv_backward_shard.argtypes = [P, I, I64, I64, I64] + [P] * 10 + [I, P]
    L.cgf_conv_double_backward_shard.argtypes = [P, I, I64, I64, I64] + [P] * 16 + [I, P]
    L.cgf_conv_forward_atomic.argtypes = [P, I, I64, I64] + [P] * 6 + [P]
    L.cgf_conv_backward_atomic.argtypes = [P, I, I64, I64] + [P] * 9 + [P]
    L.cgf_conv_double_backward_atomic.argtypes = [P, I, I64, I64] + [P] * 13 + [P]
    L.cgf_conv_forward_atomic_host.argtypes = [P, I, I64, I64] + [P] * 6
    L.cgf_conv_backward_atomic_host.argtypes = [P, I, I64, I64] + [P] * 9
    L.cgf_conv_unfused_forward.argtypes = [P, I, I64, I64] + [P] * 6 + [P, C.c_size_t, P]
    L.cgf_conv_unfused_backward.argtypes = [P, I, I64, I64] + [P] * 11 + [P, C.c_size_t, P]
    L.cgf_conv_unfused_workspace.argtypes = [P, I, I, I64]
    L.cgf_conv_unfused_workspace.restype = C.c_size_t
    L.cgf_conv_unfused_forward_host.argtypes = [P, I, I64, I64] + [P] * 6
    L.cgf_conv_unfused_backward_host.argtypes = [P, I, I64, I64] + [P] * 9
    L.cgf_array_save.argtypes = [C.c_char_p, I, P, I64, I64]
    L.cgf_array_meta.argtypes = [C.c_char_p, P, C.POINTER(I)]
    L.cgf_array_load.argtypes = [C.c_char_p, I, P, I64, I, P]
    L.cgf_nccl_unique_id.argtypes = [C.c_char_p]
    L.cgf_nccl_comm_create.argtypes = [I, I, C.c_char_p, C.POINTER(P)]
    L.cgf_nccl_comm_destroy.argtypes = [P]
    L.cgf_conv_shard_create.argtypes = [I64, I64, P, P, I, I, C.POINTER(P)]
    L.cgf_conv_shard_info.argtypes = [P, P]
    L.cgf_conv_shard_destroy.argtypes = [P]
    L.cgf_dist_conv_forward.argtypes = [P, I, P, P] + [P] * 4 + [I, P]
    L.cgf_dist_conv_backward.argtypes = [P, I, P, P] + [P] * 7 + [I, P]
    L.cgf_dist_conv_double_backward.argtypes = [P, I, P, P] + [P] * 11 + [I, P]
    L.cgf_dist_allreduce_ordered.argtypes = [I, P, I, P, I64, P]
    L.cgf_graph_make.argtypes = [I64, I64, P, P, I, P, P, P, P, P]
    L.cgf_graph_transpose.argtypes = [I64, I64, I64, P, P, P, P, P, P]
    L.cgf_graph_radius.argtypes = [I64, P, C.c_double, P, P, I64, P, P]
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().cgf_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, CgfError)(msg)


def version() -> str:
    return lib().cgf_version().decode()


def cg_block(l1: int, l2: int, l3: int):
    """Real-basis CG block entries, (k,i,j)-sorted: (i, j, k, v) arrays (cg.hpp:55)."""
    cap = (2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1)
    i, j, k = (np.zeros(cap, np.int32) for _ in range(3))
    v = np.zeros(cap, np.float64)
    n = lib().cgf_cg_block(l1, l2, l3, cap, i.ctypes.data, j.ctypes.data, k.ctypes.data, v.ctypes.data)
    if n < 0:
        _check(-n)
    return i[:n].copy(), j[:n].copy(), k[:n].copy(), v[:n].copy()


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _dtype_code(a) -> int:
    name = str(a.dtype)
    if name.endswith("float32"):
        return F32
    if name.endswith("float64"):
        return F64
    raise ShapeError(f"unsupported dtype {a.dtype} (float32 / float64)")


class TpPlan:
    """Compiled CG tensor-product problem (mirrors engine::TpPlan, engine.hpp:73-104).

    ``problem`` is the reference's problem JSON (str or dict). ``budget`` is
    the reference's scratch budget in words: accepted for API parity and used
    only for the same admission check (BudgetError)."""

    def __init__(self, problem, lane_width: int = 32, budget: int = 4096):
        if not isinstance(problem, str):
            problem = json.dumps(problem)
        self.problem_json = problem
        h = C.c_void_p()
        _check(lib().cgf_plan_create(problem.encode(), lane_width, budget, C.byref(h)))
        self._h = h
        d = np.zeros(6, np.int64)
        _check(lib().cgf_plan_dims(h, d.ctypes.data))
        self.dim_x, self.dim_y, self.dim_z, self.n_w, self.n_split, self.n_units = (int(v) for v in d)
        f = np.zeros(3, np.uint64)
        _check(lib().cgf_plan_flops(h, f.ctypes.data))
        self.flops_fwd, self.flops_bwd, self.flops_dbwd = (int(v) for v in f)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.cgf_plan_destroy(h)
            self._h = None

    # -- introspection -------------------------------------------------------
    def source(self, op=OP_FORWARD, dtype=F32, w_shared=False, aligned=True) -> str:
        n = lib().cgf_plan_source(self._h, op, dtype, int(w_shared), int(aligned), None, 0)
        if n < 0:
            _check(-n)
        buf = C.create_string_buffer(n + 1)
        lib().cgf_plan_source(self._h, op, dtype, int(w_shared), int(aligned), buf, n + 1)
        return buf.value.decode()

    def compile(self, op=OP_FORWARD, dtype=F32, w_shared=False, aligned=True):
        _check(lib().cgf_plan_compile(self._h, op, dtype, int(w_shared), int(aligned)))

    def stats(self, op, rows, w_shared=False):
        """engine::ExecStats of a call: (loads_words, stores_words, flops) of
        the reference's per-row schedule model x rows (engine.hpp:19-30)."""
        s = np.zeros(3, np.uint64)
        _check(lib().cgf_tp_stats(self._h, op, rows, int(w_shared), s.ctypes.data))
        return tuple(int(v) for v in s)

    def traffic(self, op, rows, w_shared=False):
        """Compulsory (loads, stores) words of the GPU kernels for one call."""
        s = np.zeros(2, np.uint64)
        _check(lib().cgf_tp_traffic(self._h, op, rows, int(w_shared), s.ctypes.data))
        return tuple(int(v) for v in s)

    @staticmethod
    def _text(fn, *args) -> str:
        n = fn(*args, None, 0)
        if n < 0:
            _check(-n)
        buf = C.create_string_buffer(n + 1)
        fn(*args, buf, n + 1)
        return buf.value.decode()

    def schedule_json(self) -> str:
        """scheduler::schedule_to_json of this plan's schedule (scheduler.cpp:406-445)."""
        return self._text(lib().cgf_plan_schedule_json, self._h)

    def listing(self, pos: int, backward: bool = False) -> str:
        """kernelgen::emit_text of split subkernel ``pos`` (schedule order)."""
        return self._text(lib().cgf_plan_listing, self._h, pos, int(backward))

    # -- shape checks (engine.cpp:206-220) ----------------------------------
    def _rows(self, x, y, w, w_shared):
        if x.ndim != 2 or x.shape[1] != self.dim_x:
            raise ShapeError(f"shape mismatch for x: expected [rows, {self.dim_x}], got {tuple(x.shape)}")
        rows = x.shape[0]
        if tuple(y.shape) != (rows, self.dim_y):
            raise ShapeError(f"shape mismatch for y: expected ({rows}, {self.dim_y}), got {tuple(y.shape)}")
        wr = 1 if w_shared else rows
        if tuple(w.shape) != (wr, self.n_w) and not (w_shared and tuple(w.shape) == (self.n_w,)):
            raise ShapeError(f"shape mismatch for w: expected ({wr}, {self.n_w}), got {tuple(w.shape)}")
        return rows

    @staticmethod
    def _same(ref, *arrs):
        for a in arrs:
            if _is_torch(a) != _is_torch(ref) or str(a.dtype) != str(ref.dtype):
                raise ShapeError("all arrays must share one dtype and one device kind")
            if _is_torch(a) and (not a.is_cuda or a.device != ref.device):
                raise ShapeError("torch tensors must be CUDA tensors on one device")
            if _is_torch(a) and not a.is_contiguous():
                raise ShapeError("tensors must be contiguous")

    @staticmethod
    def _out(name, a, shape):
        """A caller-provided output: exact shape, dense (written as [rows, dim])."""
        if tuple(a.shape) != tuple(shape):
            raise ShapeError(f"shape mismatch for {name}: expected {tuple(shape)}, got {tuple(a.shape)}")
        if not _is_torch(a) and not (a.flags.c_contiguous and a.flags.writeable):
            raise ShapeError(f"{name} must be a writeable C-contiguous array")

    @staticmethod
    def _stream(ref):
        import torch
        return C.c_void_p(torch.cuda.current_stream(ref.device).cuda_stream)

    @staticmethod
    def _p(a):
        return C.c_void_p(a.data_ptr() if _is_torch(a) else a.ctypes.data)

    @staticmethod
    def _empty_like(ref, shape):
        if _is_torch(ref):
            import torch
            return torch.empty(shape, dtype=ref.dtype, device=ref.device)
        return np.empty(shape, dtype=ref.dtype)

    @staticmethod
    def _host(a):
        return np.ascontiguousarray(a)

    # -- the three entry points ---------------------------------------------
    def forward(self, x, y, w, z=None, w_shared=False):
        """z = TP(x, y, W) over a batch of rows (TpPlan::forward, engine.cpp:278-283)."""
        if not _is_torch(x):
            x, y, w = self._host(x), self._host(y), self._host(w)
        self._same(x, y, w)
        rows = self._rows(x, y, w, w_shared)
        if z is None:
            z = self._empty_like(x, (rows, self.dim_z))
        self._out("z", z, (rows, self.dim_z))
        self._same(x, z)
        dt = _dtype_code(x)
        if _is_torch(x):
            _check(lib().cgf_tp_forward(self._h, dt, self._p(x), self._p(y), self._p(w), self._p(z), rows,
                                        int(w_shared), self._stream(x)))
        else:
            _check(lib().cgf_tp_forward_host(self._h, dt, self._p(x), self._p(y), self._p(w), self._p(z),
                                             rows, int(w_shared)))
        return z

    def backward(self, x, y, w, gz, w_shared=False, out=None):
        """(gx, gy, gw) from gz (TpPlan::backward, engine.cpp:285-295). ``out``:
        optional preallocated (gx, gy, gw) (e.g. pinned host arrays)."""
        if not _is_torch(x):
            x, y, w, gz = (self._host(a) for a in (x, y, w, gz))
        self._same(x, y, w, gz)
        rows = self._rows(x, y, w, w_shared)
        if tuple(gz.shape) != (rows, self.dim_z):
            raise ShapeError(f"shape mismatch for g_z: expected ({rows}, {self.dim_z}), got {tuple(gz.shape)}")
        if out is not None:
            gx, gy, gw = out
            for name, a, shp in (("gx", gx, (rows, self.dim_x)), ("gy", gy, (rows, self.dim_y)),
                                 ("gw", gw, (1 if w_shared else rows, self.n_w))):
                self._out(name, a, shp)
            self._same(x, gx, gy, gw)
        else:
            gx = self._empty_like(x, (rows, self.dim_x))
            gy = self._empty_like(x, (rows, self.dim_y))
            gw = self._empty_like(x, (1 if w_shared else rows, self.n_w))
        dt = _dtype_code(x)
        args = [self._p(a) for a in (x, y, w, gz, gx, gy, gw)]
        if _is_torch(x):
            _check(lib().cgf_tp_backward(self._h, dt, *args, rows, int(w_shared), self._stream(x)))
        else:
            _check(lib().cgf_tp_backward_host(self._h, dt, *args, rows, int(w_shared)))
        return gx, gy, gw

    def forward_backward(self, x, y, w, gz, w_shared=False, out=None):
        """z = forward(x, y, w) and (gx, gy, gw) = backward(x, y, w, gz) in one
        call: on the device the two kernels run back to back on the current
        stream; with host (numpy) arrays one pipelined pass through
        cgf_tp_forward_backward_host moves x, y and W over PCIe once.
        ``out``: optional preallocated (z, gx, gy, gw). Returns (z, gx, gy, gw)."""
        if _is_torch(x):
            z, gxyw = (None, None) if out is None else (out[0], out[1:])
            z = self.forward(x, y, w, z=z, w_shared=w_shared)
            return (z,) + tuple(self.backward(x, y, w, gz, w_shared=w_shared, out=gxyw))
        x, y, w, gz = (self._host(a) for a in (x, y, w, gz))
        self._same(x, y, w, gz)
        rows = self._rows(x, y, w, w_shared)
        if tuple(gz.shape) != (rows, self.dim_z):
            raise ShapeError(f"shape mismatch for g_z: expected ({rows}, {self.dim_z}), got {tuple(gz.shape)}")
        shapes = ((rows, self.dim_z), (rows, self.dim_x), (rows, self.dim_y), (1 if w_shared else rows, self.n_w))
        if out is None:
            out = tuple(self._empty_like(x, s) for s in shapes)
        for name, a, shp in zip(("z", "gx", "gy", "gw"), out, shapes):
            self._out(name, a, shp)
        self._same(x, *out)
        _check(lib().cgf_tp_forward_backward_host(self._h, _dtype_code(x), *(self._p(a) for a in (x, y, w, gz)),
                                                  *(self._p(a) for a in out), rows, int(w_shared)))
        return tuple(out)

    def double_backward(self, x, y, w, gz, upstream, w_shared=False):
        """Given upstream = (dL/da, dL/db, dL/dC) of backward's outputs, returns
        (dL/dx, dL/dy, dL/dW, dL/dg_z) (TpPlan::double_backward, engine.cpp:297-392)."""
        da, db, dc = upstream
        if not _is_torch(x):
            x, y, w, gz, da, db, dc = (self._host(a) for a in (x, y, w, gz, da, db, dc))
        self._same(x, y, w, gz, da, db, dc)
        rows = self._rows(x, y, w, w_shared)
        if tuple(gz.shape) != (rows, self.dim_z):
            raise ShapeError(f"shape mismatch for g_z: expected ({rows}, {self.dim_z}), got {tuple(gz.shape)}")
        for name, a, shp in (("dL/da", da, x.shape), ("dL/db", db, y.shape), ("dL/dC", dc, w.shape)):
            if tuple(a.shape) != tuple(shp):
                raise ShapeError(f"shape mismatch for {name}: expected {tuple(shp)}, got {tuple(a.shape)}")
        ox = self._empty_like(x, (rows, self.dim_x))
        oy = self._empty_like(x, (rows, self.dim_y))
        ow = self._empty_like(x, tuple(w.shape))
        ogz = self._empty_like(x, (rows, self.dim_z))
        dt = _dtype_code(x)
        args = [self._p(a) for a in (x, y, w, gz, da, db, dc, ox, oy, ow, ogz)]
        if _is_torch(x):
            _check(lib().cgf_tp_double_backward(self._h, dt, *args, rows, int(w_shared), self._stream(x)))
        else:
            _check(lib().cgf_tp_double_backward_host(self._h, dt, *args, rows, int(w_shared)))
        return ox, oy, ow, ogz


# ------------------------------------------------------------ convolution --

COMP_FWD, COMP_BWD, COMP_DBWD, COMP_DBWD_Z, COMP_DBWD_X = range(5)
LOOP_ROWS, LOOP_CONV_BY_OUTPUT, LOOP_CONV_BY_INPUT, LOOP_CONV_EDGES = range(4)
DETERMINISTIC, ATOMIC = 0, 1


class Graph:
    """The reference's GraphCSR (conv.hpp:44-50): ``src`` is the output node of
    an edge, ``nbr`` (reference ``dst``) the node whose features it reads.
    The deterministic mode needs edges sorted strictly by (src, dst) and gets
    the CSR + transposed CSR; the atomic mode takes the edges in any order
    (conv.cpp:240, 371-374). Holds host arrays and uploads them to a device on
    first use."""

    def __init__(self, nodes: int, src, nbr):
        src = np.ascontiguousarray(np.asarray(src, dtype=np.int64))
        nbr = np.ascontiguousarray(np.asarray(nbr, dtype=np.int64))
        if src.shape != nbr.shape or src.ndim != 1:
            raise ShapeError("src / nbr must be 1-D arrays of equal length")
        if src.size and (src.min() < 0 or nbr.min() < 0 or src.max() >= nodes or nbr.max() >= nodes):
            raise InvalidArgument("edge endpoint out of range")
        key = src * max(nodes, 1) + nbr
        self.sorted = bool(src.size <= 1 or np.all(np.diff(key) > 0))
        self.nodes = int(nodes)
        self.src = src.astype(np.int32)
        self.nbr = nbr.astype(np.int32)
        self._dev = {}
        if not self.sorted:
            return
        counts = np.bincount(src, minlength=nodes) if src.size else np.zeros(nodes, np.int64)
        self.row_ptr = np.zeros(nodes + 1, np.int64)
        np.cumsum(counts, out=self.row_ptr[1:])
        self.t_row_ptr = np.zeros(nodes + 1, np.int64)
        self.t_src = np.zeros(max(self.edges, 1), np.int32)
        self.t_eid = np.zeros(max(self.edges, 1), np.int32)
        _check(lib().cgf_conv_transpose_host(self.nodes, self.edges, self.row_ptr.ctypes.data,
                                             self.nbr.ctypes.data if self.edges else None,
                                             self.t_row_ptr.ctypes.data, self.t_src.ctypes.data,
                                             self.t_eid.ctypes.data))

    @property
    def edges(self) -> int:
        return int(self.src.size)

    def transpose_permutation(self) -> np.ndarray:
        """perm[e] = position of edge e in the transposed CSR (conv.hpp:62-63)."""
        perm = np.empty(self.edges, np.int64)
        perm[self.t_eid[:self.edges]] = np.arange(self.edges)
        return perm

    def require_sorted(self):
        if not self.sorted:
            raise InvalidArgument("conv: deterministic mode requires edges sorted by first coordinate")

    def device(self, dev):
        import torch
        key = str(dev)
        if key not in self._dev:
            t = lambda a: torch.from_numpy(a).to(dev)
            names = ("src", "nbr") + (("row_ptr", "t_row_ptr", "t_src", "t_eid") if self.sorted else ())
            self._dev[key] = {k: t(getattr(self, k)) for k in names}
        return self._dev[key]


class DeviceGraph:
    """A GraphCSR built and held on the device (conv.cpp:64-151 on the GPU):
    ``row_ptr`` / ``nbr`` / ``src`` (CSR by output node) and, built on first
    use, the transposed CSR. Accepted wherever ConvPlan takes a Graph."""

    sorted = True

    def __init__(self, nodes: int, row_ptr, nbr, src):
        self.nodes = int(nodes)
        self.row_ptr, self.nbr, self.src = row_ptr, nbr, src
        self._t = None

    @property
    def edges(self) -> int:
        return int(self.nbr.numel())

    def _transpose(self):
        import torch
        if self._t is None:
            dev = self.nbr.device
            E = max(self.edges, 1)
            t_row_ptr = torch.empty(self.nodes + 1, dtype=torch.int64, device=dev)
            t_src = torch.empty(E, dtype=torch.int32, device=dev)
            t_eid = torch.empty(E, dtype=torch.int32, device=dev)
            _check(lib().cgf_graph_transpose(self.nodes, self.nodes, self.edges, self.row_ptr.data_ptr(),
                                             self.nbr.data_ptr(), t_row_ptr.data_ptr(), t_src.data_ptr(),
                                             t_eid.data_ptr(), _stream_of(dev)))
            self._t = (t_row_ptr, t_src, t_eid)
        return self._t

    def require_sorted(self):
        pass

    def device(self, dev):
        t_row_ptr, t_src, t_eid = self._transpose()
        return {"row_ptr": self.row_ptr, "nbr": self.nbr, "src": self.src, "t_row_ptr": t_row_ptr,
                "t_src": t_src, "t_eid": t_eid}

    def to_host(self) -> "Graph":
        return Graph(self.nodes, self.src.cpu().numpy(), self.nbr.cpu().numpy())


def _stream_of(dev):
    import torch
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def make_graph_device(nodes: int, src, dst, allow_self_loops=False) -> DeviceGraph:
    """conv::make_graph (conv.cpp:64-87) on the device: int32 CUDA tensors of
    edges in any order -> sorted, deduplicated CSR."""
    import torch
    src = src.to(torch.int32).contiguous()
    dst = dst.to(torch.int32).contiguous()
    if src.shape != dst.shape or src.dim() != 1:
        raise ShapeError("src / dst must be 1-D arrays of equal length")
    dev = src.device
    E = src.numel()
    row_ptr = torch.empty(nodes + 1, dtype=torch.int64, device=dev)
    nbr = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    osrc = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    m = C.c_int64(0)
    _check(lib().cgf_graph_make(nodes, E, src.data_ptr() if E else None, dst.data_ptr() if E else None,
                                int(allow_self_loops), row_ptr.data_ptr(), nbr.data_ptr(), osrc.data_ptr(),
                                C.byref(m), _stream_of(dev)))
    return DeviceGraph(nodes, row_ptr, nbr[:m.value], osrc[:m.value])


def radius_graph_device(pos, r_cut: float) -> DeviceGraph:
    """conv::radius_graph (conv.cpp:89-133) on the device: pos is an (n, 3)
    float64 CUDA tensor."""
    import torch
    pos = pos.to(torch.float64).contiguous()
    if pos.dim() != 2 or pos.shape[1] != 3:
        raise ShapeError("pos must be (n, 3)")
    n, dev = pos.shape[0], pos.device
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    m = C.c_int64(0)
    _check(lib().cgf_graph_radius(n, pos.data_ptr() if n else None, float(r_cut), row_ptr.data_ptr(), None, 0,
                                  C.byref(m), _stream_of(dev)))
    nbr = torch.empty(max(m.value, 1), dtype=torch.int32, device=dev)
    _check(lib().cgf_graph_radius(n, pos.data_ptr() if n else None, float(r_cut), row_ptr.data_ptr(),
                                  nbr.data_ptr(), m.value, C.byref(m), _stream_of(dev)))
    nbr = nbr[:m.value]
    src = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device=dev), row_ptr.diff())
    return DeviceGraph(n, row_ptr, nbr, src)


class ConvPlan:
    """Fused tensor product + graph convolution over a TpPlan (conv.hpp:93-115).
    DETERMINISTIC: each output row is owned by one warp and summed in edge
    order (no atomics, no fixup pass). ATOMIC (Mode::atomic): one warp item
    per (edge, unit), node outputs accumulated with float atomics; edges in
    any order."""

    def __init__(self, plan: TpPlan):
        self.plan = plan

    def _ptrs(self, g: Graph, ref):
        d = g.device(ref.device)
        return {k: C.c_void_p(v.data_ptr()) for k, v in d.items()}

    def _check_shapes(self, g, node_x, edge_y, edge_w):
        p = self.plan
        if tuple(node_x.shape) != (g.nodes, p.dim_x):
            raise ShapeError("conv: node_x shape mismatch")
        if tuple(edge_y.shape) != (g.edges, p.dim_y):
            raise ShapeError("conv: edge_y shape mismatch")
        if tuple(edge_w.shape) != (g.edges, p.n_w):
            raise ShapeError("conv: edge_w shape mismatch")
        TpPlan._same(node_x, edge_y, edge_w)
        if not _is_torch(node_x):
            raise ShapeError("conv: pass torch CUDA tensors")

    def stats(self, op, g, mode=DETERMINISTIC, unfused=False):
        """ConvStats (conv.hpp:78-91) of one call: (loads_words, stores_words,
        output_store_ops, flops) under the GPU kernels' store / load model."""
        s = np.zeros(4, np.uint64)
        _check(lib().cgf_conv_stats(self.plan._h, op, mode, int(unfused), g.nodes, g.edges, s.ctypes.data))
        return tuple(int(v) for v in s)

    def forward(self, g: Graph, node_x, edge_y, edge_w, mode=DETERMINISTIC):
        """node_z[s] = sum over edges (s, d) of TP(node_x[d], edge_y[e], edge_w[e])."""
        self._check_shapes(g, node_x, edge_y, edge_w)
        p = self.plan
        z = TpPlan._empty_like(node_x, (g.nodes, p.dim_z))
        d = self._ptrs(g, node_x)
        if mode == ATOMIC:
            _check(lib().cgf_conv_forward_atomic(p._h, _dtype_code(node_x), g.nodes, g.edges, d["src"], d["nbr"],
                                                 TpPlan._p(node_x), TpPlan._p(edge_y), TpPlan._p(edge_w),
                                                 TpPlan._p(z), TpPlan._stream(node_x)))
            return z
        g.require_sorted()
        _check(lib().cgf_conv_forward(p._h, _dtype_code(node_x), g.nodes, g.edges, d["row_ptr"], d["nbr"],
                                      TpPlan._p(node_x), TpPlan._p(edge_y), TpPlan._p(edge_w), TpPlan._p(z), mode,
                                      TpPlan._stream(node_x)))
        return z

    def backward(self, g: Graph, node_x, edge_y, edge_w, g_node_z, mode=DETERMINISTIC):
        """(g_node_x, g_edge_y, g_edge_w) from g_node_z (conv.cpp:357-528)."""
        self._check_shapes(g, node_x, edge_y, edge_w)
        p = self.plan
        if tuple(g_node_z.shape) != (g.nodes, p.dim_z):
            raise ShapeError("conv: g_node_z shape mismatch")
        TpPlan._same(node_x, g_node_z)
        gx = TpPlan._empty_like(node_x, (g.nodes, p.dim_x))
        gy = TpPlan._empty_like(node_x, (g.edges, p.dim_y))
        gw = TpPlan._empty_like(node_x, (g.edges, p.n_w))
        d = self._ptrs(g, node_x)
        if mode == ATOMIC:
            _check(lib().cgf_conv_backward_atomic(
                p._h, _dtype_code(node_x), g.nodes, g.edges, d["src"], d["nbr"],
                *(TpPlan._p(a) for a in (node_x, edge_y, edge_w, g_node_z, gx, gy, gw)), TpPlan._stream(node_x)))
            return gx, gy, gw
        g.require_sorted()
        _check(lib().cgf_conv_backward(p._h, _dtype_code(node_x), g.nodes, g.edges, d["row_ptr"], d["nbr"],
                                       d["t_row_ptr"], d["t_src"], d["t_eid"], TpPlan._p(node_x), TpPlan._p(edge_y),
                                       TpPlan._p(edge_w), TpPlan._p(g_node_z), TpPlan._p(gx), TpPlan._p(gy),
                                       TpPlan._p(gw), mode, TpPlan._stream(node_x)))
        return gx, gy, gw

    def double_backward(self, g: Graph, node_x, edge_y, edge_w, g_node_z, upstream, mode=DETERMINISTIC):
        """Given (dL/dg_node_x, dL/dg_edge_y, dL/dg_edge_w), returns
        (dL/dnode_x, dL/dedge_y, dL/dedge_w, dL/dg_node_z)."""
        d_gx, d_gy, d_gw = upstream
        self._check_shapes(g, node_x, edge_y, edge_w)
        p = self.plan
        TpPlan._same(node_x, g_node_z, d_gx, d_gy, d_gw)
        for name, a, shp in (("g_node_z", g_node_z, (g.nodes, p.dim_z)), ("d_gx", d_gx, (g.nodes, p.dim_x)),
                             ("d_gy", d_gy, (g.edges, p.dim_y)), ("d_gw", d_gw, (g.edges, p.n_w))):
            if tuple(a.shape) != shp:
                raise ShapeError(f"conv: {name} shape mismatch")
        ox = TpPlan._empty_like(node_x, (g.nodes, p.dim_x))
        oy = TpPlan._empty_like(node_x, (g.edges, p.dim_y))
        ow = TpPlan._empty_like(node_x, (g.edges, p.n_w))
        ogz = TpPlan._empty_like(node_x, (g.nodes, p.dim_z))
        d = self._ptrs(g, node_x)
        if mode == ATOMIC:
            _check(lib().cgf_conv_double_backward_atomic(
                p._h, _dtype_code(node_x), g.nodes, g.edges, d["src"], d["nbr"],
                *(TpPlan._p(a) for a in (node_x, edge_y, edge_w, g_node_z, d_gx, d_gy, d_gw, ox, oy, ow, ogz)),
                TpPlan._stream(node_x)))
            return ox, oy, ow, ogz
        g.require_sorted()
        _check(lib().cgf_conv_double_backward(
            p._h, _dtype_code(node_x), g.nodes, g.edges, d["row_ptr"], d["nbr"], d["t_row_ptr"], d["t_src"],
            d["t_eid"], *(TpPlan._p(a) for a in (node_x, edge_y, edge_w, g_node_z, d_gx, d_gy, d_gw, ox, oy, ow,
                                                 ogz)), mode, TpPlan._stream(node_x)))
        return ox, oy, ow, ogz


    # -- unfused comparator (conv.cpp:530-616) on the GPU ----------------------
    def unfused_forward(self, g, node_x, edge_y, edge_w):
        """Gather x per edge -> batched TP over |E| rows -> per-node sums in edge order."""
        self._check_shapes(g, node_x, edge_y, edge_w)
        g.require_sorted()
        p = self.plan
        z = TpPlan._empty_like(node_x, (g.nodes, p.dim_z))
        d = self._ptrs(g, node_x)
        ws = self._workspace(node_x, 0, g.edges)
        _check(lib().cgf_conv_unfused_forward(p._h, _dtype_code(node_x), g.nodes, g.edges, d["row_ptr"], d["nbr"],
                                              TpPlan._p(node_x), TpPlan._p(edge_y), TpPlan._p(edge_w), TpPlan._p(z),
                                              TpPlan._p(ws), ws.numel(), TpPlan._stream(node_x)))
        return z

    def _workspace(self, ref, op, edges):
        """Device workspace of the unfused path, from torch's caching allocator."""
        import torch
        n = lib().cgf_conv_unfused_workspace(self.plan._h, _dtype_code(ref), op, edges)
        return torch.empty(max(n, 1), dtype=torch.uint8, device=ref.device)

    def unfused_backward(self, g, node_x, edge_y, edge_w, g_node_z):
        self._check_shapes(g, node_x, edge_y, edge_w)
        g.require_sorted()
        p = self.plan
        gx = TpPlan._empty_like(node_x, (g.nodes, p.dim_x))
        gy = TpPlan._empty_like(node_x, (g.edges, p.dim_y))
        gw = TpPlan._empty_like(node_x, (g.edges, p.n_w))
        d = self._ptrs(g, node_x)
        ws = self._workspace(node_x, 1, g.edges)
        _check(lib().cgf_conv_unfused_backward(
            p._h, _dtype_code(node_x), g.nodes, g.edges, d["row_ptr"], d["nbr"], d["t_row_ptr"], d["t_eid"],
            *(TpPlan._p(a) for a in (node_x, edge_y, edge_w, g_node_z, gx, gy, gw)), TpPlan._p(ws), ws.numel(),
            TpPlan._stream(node_x)))
        return gx, gy, gw

    # -- sharded calls (one rank of a destination-partitioned graph) ---------
    # ``sh`` is a dist.GraphShard: out_nodes owned output rows, in_nodes
    # (padded, all-gathered) neighbour rows, local CSR + transposed CSR.
    def _shard_ptrs(self, sh, ref):
        d = sh.device(ref.device)
        return {k: C.c_void_p(v.data_ptr()) for k, v in d.items()}

    def _check_shard(self, sh, **arrays):
        """Shapes of a shard call's arrays (the checks ConvPlan._check_shapes
        makes for a whole graph, over the shard's row counts)."""
        p = self.plan
        rows = {"node_x_all": (sh.in_nodes, p.dim_x), "d_gx_all": (sh.in_nodes, p.dim_x),
                "edge_y": (sh.edges, p.dim_y), "d_gy": (sh.edges, p.dim_y),
                "edge_w": (sh.edges, p.n_w), "d_gw": (sh.edges, p.n_w),
                "g_node_z": (sh.out_nodes, p.dim_z)}
        for name, a in arrays.items():
            if tuple(a.shape) != rows[name]:
                raise ShapeError(f"conv shard: {name} shape mismatch: expected {rows[name]}, got {tuple(a.shape)}")
        ref = next(iter(arrays.values()))
        TpPlan._same(ref, *arrays.values())
        if not _is_torch(ref):
            raise ShapeError("conv: pass torch CUDA tensors")

    @staticmethod
    def _row_range(rows, n, what):
        """(r0, r1) of a row-range shard call: 0 <= r0 <= r1 <= n, r0 a multiple of
        4 so every row-indexed array keeps the 16-byte alignment of its base."""
        r0, r1 = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
        if not 0 <= r0 <= r1 <= n:
            raise ShapeError(f"conv shard: {what} rows [{r0}, {r1}) outside [0, {n})")
        if r0 % 4:
            raise ShapeError(f"conv shard: {what} row range must start at a multiple of 4, got {r0}")
        return r0, r1

    def _outs(self, outs, ref, shapes):
        if outs is None:
            return [TpPlan._empty_like(ref, s) for s in shapes]
        for a, s in zip(outs, shapes):
            if tuple(a.shape) != s:
                raise ShapeError(f"conv shard: output shape mismatch: expected {s}, got {tuple(a.shape)}")
            TpPlan._same(ref, a)
        return list(outs)

    def forward_shard(self, sh, node_x_all, edge_y, edge_w, mode=DETERMINISTIC, rows=None, out=None):
        """Local output rows of the conv; node_x_all spans sh.in_nodes rows.

        ``rows=(r0, r1)`` computes output rows [r0, r1) only, into ``out`` (the
        [out_nodes, dim_z] result, allocated when None): the row-range launches
        of the overlapped multi-GPU forward (``dist.DistConvPlan``). Rows are
        independent and each keeps its edge order, so any split is bit-identical
        to one launch over the shard."""
        p = self.plan
        self._check_shard(sh, node_x_all=node_x_all, edge_y=edge_y, edge_w=edge_w)
        (z,) = self._outs(None if out is None else (out,), node_x_all, [(sh.out_nodes, p.dim_z)])
        r0, r1 = self._row_range(rows, sh.out_nodes, "output")
        if rows is not None and mode != DETERMINISTIC:
            raise ShapeError("conv shard: row ranges are for the deterministic mode")
        d = self._shard_ptrs(sh, node_x_all)
        es = node_x_all.element_size()
        _check(lib().cgf_conv_forward_shard(p._h, _dtype_code(node_x_all), r1 - r0, sh.in_nodes, sh.edges,
                                            C.c_void_p(d["row_ptr"].value + 8 * r0), d["nbr"],
                                            TpPlan._p(node_x_all), TpPlan._p(edge_y), TpPlan._p(edge_w),
                                            C.c_void_p(z.data_ptr() + r0 * p.dim_z * es), mode,
                                            TpPlan._stream(node_x_all)))
        return z

    def backward_shard(self, sh, node_x_all, edge_y, edge_w, g_node_z, mode=DETERMINISTIC, rows=None, outs=None):
        """(partial g_node_x over sh.in_nodes rows, g_edge_y, g_edge_w).

        ``rows=(r0, r1)`` runs the transposed-CSR rows (neighbour nodes) [r0, r1)
        only, writing their g_node_x rows and their edges' g_edge_y / g_edge_w
        into ``outs`` = (gx, gy, gw) (allocated when None); the overlapped
        multi-GPU backward runs the other ranks' rows first and sends them while
        its own rows compute."""
        p = self.plan
        self._check_shard(sh, node_x_all=node_x_all, edge_y=edge_y, edge_w=edge_w, g_node_z=g_node_z)
        gx, gy, gw = self._outs(outs, node_x_all, [(sh.in_nodes, p.dim_x), (sh.edges, p.dim_y), (sh.edges, p.n_w)])
        r0, r1 = self._row_range(rows, sh.in_nodes, "neighbour")
        if rows is not None and mode != DETERMINISTIC:
            raise ShapeError("conv shard: row ranges are for the deterministic mode")
        d = self._shard_ptrs(sh, node_x_all)
        off = r0 * p.dim_x * node_x_all.element_size()
        _check(lib().cgf_conv_backward_shard(p._h, _dtype_code(node_x_all), sh.out_nodes, r1 - r0, sh.edges,
                                             C.c_void_p(d["t_row_ptr"].value + 8 * r0), d["t_src"], d["t_eid"],
                                             C.c_void_p(node_x_all.data_ptr() + off), TpPlan._p(edge_y),
                                             TpPlan._p(edge_w), TpPlan._p(g_node_z),
                                             C.c_void_p(gx.data_ptr() + off), TpPlan._p(gy), TpPlan._p(gw), mode,
                                             TpPlan._stream(node_x_all)))
        return gx, gy, gw

    def double_backward_shard(self, sh, node_x_all, edge_y, edge_w, g_node_z, d_gx_all, d_gy, d_gw,
                              mode=DETERMINISTIC):
        """(partial dL/dnode_x over sh.in_nodes rows, dL/dedge_y, dL/dedge_w, dL/dg_node_z local)."""
        p = self.plan
        self._check_shard(sh, node_x_all=node_x_all, edge_y=edge_y, edge_w=edge_w, g_node_z=g_node_z,
                          d_gx_all=d_gx_all, d_gy=d_gy, d_gw=d_gw)
        ox = TpPlan._empty_like(node_x_all, (sh.in_nodes, p.dim_x))
        oy = TpPlan._empty_like(node_x_all, (sh.edges, p.dim_y))
        ow = TpPlan._empty_like(node_x_all, (sh.edges, p.n_w))
        ogz = TpPlan._empty_like(node_x_all, (sh.out_nodes, p.dim_z))
        d = self._shard_ptrs(sh, node_x_all)
        _check(lib().cgf_conv_double_backward_shard(
            p._h, _dtype_code(node_x_all), sh.out_nodes, sh.in_nodes, sh.edges, d["row_ptr"], d["nbr"],
            d["t_row_ptr"], d["t_src"], d["t_eid"],
            *(TpPlan._p(a) for a in (node_x_all, edge_y, edge_w, g_node_z, d_gx_all, d_gy, d_gw, ox, oy, ow, ogz)),
            mode, TpPlan._stream(node_x_all)))
        return ox, oy, ow, ogz


# ------------------------------------------------------------ array files --

def save_array(base: str, a):
    """array_io::save_array (array_io.cpp:15-38): <base>.bin + <base>.json;
    a 2-D float32 / float64 numpy array or CUDA tensor (copied to the host)."""
    if _is_torch(a):
        a = a.detach().cpu().numpy()
    a = np.ascontiguousarray(a)
    if a.ndim != 2:
        raise ShapeError("save_array: expected a 2-D array")
    _check(lib().cgf_array_save(base.encode(), _dtype_code(a), a.ctypes.data, a.shape[0], a.shape[1]))


def read_meta(base: str):
    """(rows, cols, dtype code) of an array file (array_io.cpp:40-50)."""
    shape = np.zeros(2, np.int64)
    dt = C.c_int()
    _check(lib().cgf_array_meta(base.encode(), shape.ctypes.data, C.byref(dt)))
    return int(shape[0]), int(shape[1]), dt.value


def load_array(base: str, device=None):
    """array_io::load_array (array_io.cpp:52-68): a numpy array, or with
    ``device`` a CUDA tensor filled through pinned staging."""
    rows, cols, dt = read_meta(base)
    if device is None:
        out = np.empty((rows, cols), np.float64 if dt == F64 else np.float32)
        _check(lib().cgf_array_load(base.encode(), dt, out.ctypes.data, out.size, 0, None))
        return out
    import torch
    out = torch.empty((rows, cols), dtype=torch.float64 if dt == F64 else torch.float32, device=device)
    _check(lib().cgf_array_load(base.encode(), dt, C.c_void_p(out.data_ptr()), out.numel(), 1, _stream_of(out.device)))
    return out


def _kernel_source(plan: TpPlan, comp, loop, dtype=F32, w_shared=False, aligned=True) -> str:
    n = lib().cgf_plan_kernel_source(plan._h, comp, loop, dtype, int(w_shared), int(aligned), None, 0)
    if n < 0:
        _check(-n)
    buf = C.create_string_buffer(n + 1)
    lib().cgf_plan_kernel_source(plan._h, comp, loop, dtype, int(w_shared), int(aligned), buf, n + 1)
    return buf.value.decode()


def _kernel_groups(plan: TpPlan, comp, loop, dtype=F32) -> int:
    return lib().cgf_plan_kernel_groups(plan._h, comp, loop, dtype)


def _kernel_source_group(plan: TpPlan, comp, loop, dtype, group, w_shared=False, aligned=True) -> str:
    return TpPlan._text(lib().cgf_plan_kernel_source_group, plan._h, comp, loop, dtype, int(w_shared), int(aligned),
                        group)


def _kernel_compile(plan: TpPlan, comp, loop, dtype=F32, w_shared=False, aligned=True):
    _check(lib().cgf_plan_kernel_compile(plan._h, comp, loop, dtype, int(w_shared), int(aligned)))
