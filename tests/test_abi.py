"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol include/*.h declares (-m "not gpu": no compute calls)."""
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        names += re.findall(r"^FALCON_API\s+[\w\s\*]*?\b(\w+)\s*\(", txt, re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1903_01665_b200 import _build
    return _build.build()


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("graph_load_csr", "falcon_sssp", "falcon_bfs", "falcon_cc", "graph_free"):
        assert name in d


def test_exports_every_declared_symbol(lib_path):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in _declared() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_sm100a_cubin(lib_path):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], text=True)
    assert "sm_100a" in out


def test_loads_and_validates_without_gpu(lib_path):
    import ctypes

    import numpy as np

    import paper_1903_01665_b200 as fb
    lib = fb.load()
    assert "sm_100a" in fb.falcon_version()
    # argument validation happens before any CUDA call
    out = ctypes.c_void_p()
    ro = np.zeros(1, np.uint32)
    rc = lib.graph_load_csr(0, 0, ctypes.c_void_p(ro.ctypes.data), None, None, None, ctypes.byref(out))
    assert fb.STATUS[rc] == "INVALID_ARG"
    assert "n must be" in fb.falcon_last_error()
    rc = lib.falcon_sssp(None, 0, 0, None, None)
    assert fb.STATUS[rc] == "INVALID_ARG"


def test_product_package_has_no_oracle_or_fallback():
    """The product path never imports the oracle and has no CPU fallback."""
    pkg = os.path.join(ROOT, "paper_1903_01665_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            txt = open(f).read()
            assert "import oracle" not in txt and "from oracle" not in txt, f
            assert "liboracle" not in txt, f
            assert "scipy" not in txt, f


def test_binding_refuses_short_buffers(lib_path):
    """the C ABI copies n values out and reads n+1 / m values in;
    the binding checks lengths before calling into C."""
    import numpy as np

    import paper_1903_01665_b200 as fb
    fb.load()
    ro = np.array([0, 2, 3, 3], np.uint32)
    with pytest.raises(ValueError, match="col"):
        fb.graph_load_csr(3, 3, ro, np.array([1, 2], np.uint32), None)
    with pytest.raises(ValueError, match="w"):
        fb.graph_load_csr(3, 3, ro, np.array([1, 2, 0], np.uint32), np.array([1], np.int32))
    with pytest.raises(ValueError, match="row_off"):
        fb.graph_load_csr(3, 3, ro[:3], np.array([1, 2, 0], np.uint32), None)
    g = fb.Graph(None, 5, 0)   # a handle-less graph: the length check comes first
    for f in (lambda o: fb.falcon_sssp(g, 0, "vertex", o), lambda o: fb.falcon_bfs(g, 0, "vertex", o),
              lambda o: fb.falcon_cc(g, "vertex", o)):
        with pytest.raises(ValueError, match="elements"):
            f(np.empty(4, np.int32))
