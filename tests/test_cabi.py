"""The C-ABI libraries load on a CPU-only host and export every declared symbol.

No compute calls into the executor here (there may be no GPU); the decision
core is pure C++ and is exercised directly, including the ctypes stub shown in
INTEGRATION.md.
"""

import ctypes as C
import os
import re

from paper_1901_10008_b200 import _build, _lib

from .conftest import REPO

INCLUDE = os.path.join(REPO, "include")


def _declared(header):
    text = open(os.path.join(INCLUDE, header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gmx_[a-z0-9_]+)\s*\(", text)))


def test_core_exports_every_declared_symbol():
    lib = C.CDLL(_build.build_core())
    names = _declared("gmx_core.h")
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_exec_library_loads_and_exports_without_gpu():
    lib = C.CDLL(_build.build_exec())
    names = _declared("gmx_exec.h") + _declared("gmx_runtime.h")
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_error_codes_and_messages():
    core = _lib.core()
    out = C.c_int64()
    dims = (C.c_int64 * 3)(0, 1, 1)
    assert core.gmx_flop_count(1, dims, 3, C.byref(out)) == _lib.EINVAL
    assert b"dims" in core.gmx_last_error()
    dims = (C.c_int64 * 3)(2, 3, 4)
    assert core.gmx_flop_count(1, dims, 3, C.byref(out)) == 0 and out.value == 48
    big = (C.c_int64 * 3)(1 << 40, 1 << 40, 1 << 40)
    assert core.gmx_flop_count(1, big, 3, C.byref(out)) == _lib.EOVERFLOW


def test_integration_doc_ctypes_stub_runs():
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    stub = text.split("```python\nimport ctypes as C\n", 1)[1].split("```", 1)[0]
    ns = {}
    exec("import ctypes as C\n" + stub.replace('"paper_1901_10008_b200/lib/libgmx_core.so"',
                                               repr(_build.build_core())), ns)
    import paper_1901_10008_b200 as gm
    ks = [gm.submit("gemm", (64, 3136, 576), "fp32", gm.LatencyConstraint(200_000_000), "a", kernel_id=0),
          gm.submit("gemm", (64, 3000, 576), "fp32", gm.LatencyConstraint(200_000_000), "b", kernel_id=1),
          gm.submit("gemv", (64, 64), "fp32", gm.LatencyConstraint(200_000_000), "c", kernel_id=2)]
    groups = ns["cluster_shapes"](ks, 0.25)
    assert [[k.kernel_id for k in g] for g in groups] == \
        [[k.kernel_id for k in c.members] for c in gm.cluster_shapes(ks, 0.25)]
