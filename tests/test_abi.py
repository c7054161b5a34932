"""CPU-side checks of the C-ABI boundary (no compute calls: there is no GPU here).

* libgpsense.so loads and exports every symbol include/gpsense.h declares;
* the binding's ctypes structs match the header's layouts (sizes);
* without a CUDA device the library refuses to run (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpsense.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"GPS_API\s+[\w\s\*]+?\b(gps_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def gps():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_gps_build", os.path.join(ROOT, "paper_1807_08804_b200", "_build.py"))
    _build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(_build)   # by path: the package __init__ needs the built .so
    _build.build()
    from paper_1807_08804_b200 import gpsense
    return gpsense


def test_header_declares_entry_points():
    names = _declared()
    for want in ["gps_load_data_graph", "gps_match", "gps_count", "gps_create", "gps_result_info"]:
        assert want in names


def test_library_exports_every_declared_symbol(gps):
    lib = ctypes.CDLL(gps.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(gps.EXPORTED) == _declared()


def _c_layouts():
    """sizeof / offsetof of the header's structs, as gcc lays them out (x86-64 SysV)."""
    import subprocess
    import tempfile
    structs = {"gps_ctx_opts": "CtxOpts", "gps_csr_desc": "CsrDesc", "gps_qedge": "QEdge",
               "gps_query": "QueryDesc", "gps_match_opts": "MatchOpts", "gps_stats": "Stats"}
    import paper_1807_08804_b200.gpsense as g
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gpsense.h"', "int main(void) {"]
    for cs, py in structs.items():
        lines.append(f'printf("{cs} size %zu\\n", sizeof({cs}));')
        for f, _ in getattr(g, py)._fields_:
            lines.append(f'printf("{cs} {f} %zu\\n", offsetof({cs}, {f}));')
    lines.append("return 0; }")
    d = tempfile.mkdtemp()
    src, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
    open(src, "w").write("\n".join(lines))
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
    out = {}
    for ln in subprocess.check_output([exe], text=True).splitlines():
        a, b, c = ln.split()
        out[(a, b)] = int(c)
    return structs, out


def test_struct_layouts(gps):
    """Every ctypes struct of the binding has the header's size and field offsets."""
    structs, c = _c_layouts()
    for cs, py in structs.items():
        st = getattr(gps, py)
        assert ctypes.sizeof(st) == c[(cs, "size")], cs
        for f, _ in st._fields_:
            assert getattr(st, f).offset == c[(cs, f)], (cs, f)


def test_default_opts(gps):
    o = gps.default_opts()
    assert (o.refine_rounds, o.reverse_refine, o.lowconn_threshold, o.result_on_device) == (1, 1, 1, 1)
    assert abs(o.rebalance_threshold - 1.10) < 1e-6


def test_no_cpu_fallback_without_device(gps):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gps.GpsError) as ei:
        gps.Context(0)
    assert ei.value.status in (gps.GPS_ECUDA, gps.GPS_EINVAL)


def test_kernel_sass_is_sm100a(gps):
    """The .so carries sm_100a SASS (cuobjdump), not PTX for another arch."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([exe, "--list-elf", gps.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_query_batch_marshalling():
    """QueryBatch's gps_query array decodes back to the queries (pointers into its arrays)."""
    import ctypes
    from paper_1807_08804_b200 import gpsense
    import corpus
    from synth import Query
    qs = [corpus.instance(s)[1] for s in range(12)] + [Query(1, [3], [-1], [])]
    qb = gpsense.QueryBatch(qs)
    assert len(qb) == len(qs)
    for i, q in enumerate(qs):
        d = qb.arr[i]
        assert d.n_vertices == q.k and d.n_edges == len(q.edges)
        vl = np.ctypeslib.as_array(ctypes.cast(d.vertex_labels, ctypes.POINTER(ctypes.c_int32)), (q.k,))
        bd = np.ctypeslib.as_array(ctypes.cast(d.bound, ctypes.POINTER(ctypes.c_int64)), (q.k,))
        assert vl.tolist() == list(q.vlabels) and bd.tolist() == list(q.bound)
        if q.edges:
            e = np.ctypeslib.as_array(ctypes.cast(d.edges, ctypes.POINTER(ctypes.c_int32)), (len(q.edges), 3))
            assert [tuple(x) for x in e.tolist()] == [tuple(x) for x in q.edges]
        else:
            assert not d.edges
