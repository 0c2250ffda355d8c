"""The reference's OWN unit tests (test_engine.cpp, test_conv.cpp, compiled
unchanged from the reference sources by tests/cpp/Makefile against a
doctest-compatible header) linked against the drop-in C++ shims
(paper_2501_13986_b200/shim/) and libcgf.so instead of the reference's
engine.cpp / conv.cpp. On a GPU every case must pass; on CPU only the host-side
graph utility cases can (the compute cases fail loudly: no CUDA driver)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
HOST_CASES = ["load_xyz", "radius_graph pair cases", "radius_graph equals the brute-force pair check",
              "transpose permutation", "make_graph rejects bad edges"]


def _run(name, timeout=900):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (tests/cpp/Makefile needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_reference_conv_tests_host_cases_pass():
    rc, out = _run("test_conv_b200")
    for case in HOST_CASES:
        assert f"[ ok ] {case}" in out, out[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_engine_b200", "test_conv_b200"])
def test_reference_unit_tests_pass_on_the_gpu_backend(name):
    if not _has_gpu():
        pytest.skip("no CUDA device")
    rc, out = _run(name)
    print(out[-4000:])
    assert rc == 0, out[-4000:]
    assert "| 0 failed;" in out


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_gpu_backend():
    """tests/acceptance.cpp, unchanged: criteria 1-7 (accuracy vs the dense
    oracle, equivariance, finite-difference gradients, double backward,
    schedules, fused conv vs unfused + store counts, sparsity/flop count) must
    PASS. Criterion 8 times the reference's *dense* oracle over 50K rows on one
    CPU core (> 15 min; criterion 9 is printed after it), so the run
    is cut after the first seven lines."""
    import re
    if not _has_gpu():
        pytest.skip("no CUDA device")
    exe = os.path.join(BUILD, "acceptance_b200")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    p = subprocess.Popen(["stdbuf", "-oL", exe], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    lines = []
    try:
        for line in p.stdout:
            lines.append(line)
            if sum(1 for x in lines if re.match(r"^(PASS|FAIL) criterion", x)) >= 7:
                break
    finally:
        p.kill()
        p.wait()
    out = "".join(lines)
    print(out)
    for n in range(1, 8):
        assert re.search(rf"^PASS criterion {n} ", out, re.M), f"criterion {n}:\n{out}"
