"""The C ABI (include/cgf.h) without a GPU: libcgf.so loads, exports every
function the header declares, and the host-only entry points (planning,
validation errors, code generation, NVRTC compilation for sm_100a, stats,
transposed CSR) work. Compute entry points are not called here; without a
CUDA driver they must fail loudly (CGF_E_CUDA), never fall back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cgf.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cgf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for want in ("cgf_plan_create", "cgf_plan_destroy", "cgf_tp_forward", "cgf_tp_backward", "cgf_tp_double_backward",
                 "cgf_tp_forward_host", "cgf_conv_forward", "cgf_conv_backward", "cgf_conv_double_backward",
                 "cgf_conv_forward_shard", "cgf_conv_transpose_host", "cgf_last_error", "cgf_tp_stats"):
        assert want in names


def test_library_exports_every_declared_symbol():
    import paper_2501_13986_b200 as cgf
    lib = C.CDLL(cgf.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_plan_errors_map_to_reference_exceptions():
    import paper_2501_13986_b200 as cgf
    with pytest.raises(cgf.ParseError):
        cgf.TpPlan('{"x": "32xq", "y": "1x0e", "z": "32x0e", "instructions": [[1, 1, 1, "B"]]}')
    with pytest.raises(cgf.ValidationError):  # parity violation
        cgf.TpPlan('{"x": "8x1o", "y": "1x0e", "z": "8x1e", "instructions": [[1, 1, 1, "B"]]}')
    with pytest.raises(cgf.BudgetError):
        cgf.TpPlan('{"x": "32x2e", "y": "1x2e", "z": "32x2e", "instructions": [[1, 1, 1, "B"]]}', budget=16)


def test_codegen_and_nvrtc_without_a_gpu():
    import paper_2501_13986_b200 as cgf
    from oracle.oracle import config_json
    plan = cgf.TpPlan(config_json("c1"))
    src = plan.source(op=0)
    assert "cp.async.bulk" in src and "extern \"C\" __global__" in src
    plan.compile(op=1, dtype=1)  # NVRTC -> sm_100a cubin, cached
    c3 = cgf.TpPlan(config_json("c3"))
    assert "tcgen05.mma" in c3.source(op=0, dtype=0, w_shared=True)
    assert c3.stats(0, 10)[2] == 10 * c3.flops_fwd


def test_transposed_csr_host():
    import paper_2501_13986_b200 as cgf
    g = cgf.Graph(4, [0, 0, 1, 2, 3], [1, 2, 3, 0, 0])
    # neighbour 0 is read by edges 3 (src 2) and 4 (src 3), in CSR order
    assert list(g.t_row_ptr) == [0, 2, 3, 4, 5]
    assert list(g.t_src[:2]) == [2, 3] and list(g.t_eid[:2]) == [3, 4]
    perm = g.transpose_permutation()
    assert sorted(perm) == list(range(5))


def test_compute_fails_loudly_without_cuda(monkeypatch):
    import paper_2501_13986_b200 as cgf
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    from oracle.oracle import config_json
    plan = cgf.TpPlan(config_json("scalar"))
    x = np.ones((2, plan.dim_x), np.float64)
    y = np.ones((2, plan.dim_y), np.float64)
    w = np.ones((2, plan.n_w), np.float64)
    with pytest.raises(cgf.CudaError):
        plan.forward(x, y, w)


def test_device_entry_points_fail_loudly_without_cuda():
    """Every device entry point returns CGF_E_CUDA without a driver (no crash:
    the driver entry points are resolved before any use)."""
    import paper_2501_13986_b200 as cgf
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    from oracle.oracle import config_json
    plan = cgf.TpPlan(config_json("paper"))
    L = cgf.lib()
    f = C.c_void_p(0x10000)  # never dereferenced on the host
    m = C.c_int64(0)
    rp = np.array([0, 1, 2, 2], np.int64)
    calls = {
        "forward_atomic": lambda: L.cgf_conv_forward_atomic(plan._h, 1, 3, 2, *[f] * 6, None),
        "backward_atomic": lambda: L.cgf_conv_backward_atomic(plan._h, 1, 3, 2, *[f] * 9, None),
        "dbwd_atomic": lambda: L.cgf_conv_double_backward_atomic(plan._h, 1, 3, 2, *[f] * 13, None),
        "unfused_fwd": lambda: L.cgf_conv_unfused_forward(plan._h, 1, 3, 2, *[f] * 6, None, 0, None),
        "unfused_bwd": lambda: L.cgf_conv_unfused_backward(plan._h, 1, 3, 2, *[f] * 11, None, 0, None),
        "graph_make": lambda: L.cgf_graph_make(3, 2, f, f, 0, f, f, None, C.byref(m), None),
        "graph_transpose": lambda: L.cgf_graph_transpose(3, 3, 2, rp.ctypes.data, f, f, f, f, None),
        "graph_radius": lambda: L.cgf_graph_radius(3, f, 1.0, f, None, 0, C.byref(m), None),
        "conv_forward_csr_atomic": lambda: L.cgf_conv_forward(plan._h, 1, 3, 2, f, f, f, f, f, f, 1, None),
    }
    for name, call in calls.items():
        assert call() == cgf.CudaError.code, name


def test_output_arrays_are_shape_checked_before_any_compute():
    """TpPlan.forward / backward / forward_backward reject a z (or gx, gy, gw)
    of the wrong shape, or a non-contiguous / read-only numpy output, with
    ShapeError before the C ABI is called (no device needed)."""
    import numpy as np
    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200.configs import config_json
    plan = cgf.TpPlan(config_json("c1"))
    x = np.zeros((4, plan.dim_x), np.float32)
    y = np.zeros((4, plan.dim_y), np.float32)
    w = np.zeros((4, plan.n_w), np.float32)
    gz = np.zeros((4, plan.dim_z), np.float32)
    for bad in (np.zeros((3, plan.dim_z), np.float32), np.zeros((4, plan.dim_z + 1), np.float32),
                np.zeros((plan.dim_z, 4), np.float32).T):
        with pytest.raises(cgf.ShapeError):
            plan.forward(x, y, w, z=bad)
    ro = np.zeros((4, plan.dim_z), np.float32)
    ro.flags.writeable = False
    with pytest.raises(cgf.ShapeError):
        plan.forward(x, y, w, z=ro)
    with pytest.raises(cgf.ShapeError):
        plan.backward(x, y, w, gz, out=(np.zeros((4, plan.dim_x), np.float32), np.zeros((4, plan.dim_y), np.float32),
                                        np.zeros((3, plan.n_w), np.float32)))
    with pytest.raises(cgf.ShapeError):
        plan.forward_backward(x, y, w, gz, out=(np.zeros((4, plan.dim_z), np.float32),) * 4)


def test_device_traffic_model():
    """cgf_tp_traffic: the compulsory words of each op."""
    import paper_2501_13986_b200 as cgf
    from paper_2501_13986_b200.configs import config_json
    p = cgf.TpPlan(config_json("c2"))
    X, Y, W, Z = p.dim_x, p.dim_y, p.n_w, p.dim_z
    assert p.traffic(cgf.OP_FORWARD, 10) == (10 * (X + Y + W), 10 * Z)
    assert p.traffic(cgf.OP_BACKWARD, 10) == (10 * (X + Y + W + Z), 10 * (X + Y + W))
    assert p.traffic(cgf.OP_DOUBLE_BACKWARD, 10) == (10 * (3 * (X + Y + W) + Z), 10 * (X + Y + W + Z))
    assert p.traffic(cgf.OP_FORWARD, 10, w_shared=True) == (10 * (X + Y) + W, 10 * Z)
    # the bench's C2 per-row figures: 12,432 / 15,776 words
    assert sum(p.traffic(cgf.OP_FORWARD, 1)) == 12_432 and sum(p.traffic(cgf.OP_BACKWARD, 1)) == 15_776
