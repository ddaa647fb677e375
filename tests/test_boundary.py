"""CPU-side checks of the C-ABI boundary (no GPU needed): the library builds
for sm_100a, loads, and exports every symbol include/fiedler.h declares; the
Python binding keeps the C names; the product package never imports oracle/."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "fiedler.h")).read()
    return sorted(set(re.findall(r"FIEDLER_API\s+[\w\s\*]*?\b(fiedler_\w+)\s*\(", hdr)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("fiedler_create", "fiedler_solve", "fiedler_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_1602_04386_b200 import build as b
    lib_path = b.build()
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    import paper_1602_04386_b200 as p
    assert sorted(p.EXPORTED) == declared_symbols()


def test_sass_is_sm100a():
    import subprocess
    from paper_1602_04386_b200 import build as b
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", b.build()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1602_04386_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                # comments may mention the oracle; code may not include or call it
                for inc in re.findall(r'#\s*include\s*[<"]([^>"]+)[>"]', src):
                    assert "oracle" not in inc.lower(), (f, inc)
                assert not re.search(r"\borc_\w+\s*\(", src), f


def test_library_does_not_link_oracle():
    import subprocess
    from paper_1602_04386_b200 import build as b
    so = b.build()
    dyn = subprocess.run(["readelf", "-d", so], capture_output=True, text=True).stdout
    assert "oracle" not in dyn.lower()
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert not re.search(r"\borc_", syms)


def test_no_gpu_means_loud_failure():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import graphgen as gg
    import paper_1602_04386_b200 as p
    g = gg.grid2d(4)
    with pytest.raises(p.FiedlerError) as e:
        p.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    assert e.value.code == p.FIEDLER_ERR_CUDA


def test_argument_errors_before_any_device_work():
    """Argument checks of fiedler_create come before the device is touched, so
    they return their documented codes on a machine without a GPU too."""
    import numpy as np
    import paper_1602_04386_b200 as p
    rp = np.array([0, 1, 2], dtype=np.int64)
    ci = np.array([1, 0], dtype=np.int32)
    w = np.ones(2)
    with pytest.raises(p.FiedlerError) as e:
        p.fiedler_create(1, 0, np.zeros(2, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert e.value.code == p.FIEDLER_ERR_ARG                     # n < 2
    with pytest.raises(p.FiedlerError) as e:
        p.fiedler_create(2, -1, rp, ci, w)
    assert e.value.code == p.FIEDLER_ERR_ARG                     # nnz < 0
    with pytest.raises(p.FiedlerError) as e:
        p.fiedler_create(1 << 31, 2, rp, ci, w)
    assert e.value.code == p.FIEDLER_ERR_TOO_LARGE               # int32 offsets
    bad = p.fiedler_default_opts(coarsest_size=1)
    with pytest.raises(p.FiedlerError) as e:
        p.fiedler_create(2, 2, rp, ci, w, bad)
    assert e.value.code == p.FIEDLER_ERR_ARG                     # invalid options
    lib = p._load()
    import ctypes
    h = ctypes.c_void_p()
    assert lib.fiedler_create(2, 2, None, None, None, 0, None, ctypes.byref(h)) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_create(2, 2, rp.ctypes.data, ci.ctypes.data, w.ctypes.data, 7, None,
                              ctypes.byref(h)) == p.FIEDLER_ERR_ARG   # bad memory kind
    assert lib.fiedler_destroy(None) == p.FIEDLER_OK
    assert lib.fiedler_solve(None, None, None, 0, None, None) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_dist_plan(None, 0, 1, 0, None) == p.FIEDLER_ERR_ARG
    assert "handle" in p.fiedler_last_error().lower()
    # partitioned setup: argument errors are reported before any device work
    b = (ctypes.c_int64 * 3)()
    assert lib.fiedler_pset_bounds(4, None, 2, b, None) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_pset_bounds(4, rp.ctypes.data, 0, b, None) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_pset_match(0, 2, rp.ctypes.data, ci.ctypes.data, w.ctypes.data, 0, 3, 0, 0, None,
                                  None, 0, None, None, None) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_pset_galerkin(0, 2, None, None, None, None, 0, 1, 0, None, None, None, None,
                                     None) == p.FIEDLER_ERR_ARG
    assert lib.fiedler_create_preset(2, 2, rp.ctypes.data, ci.ctypes.data, w.ctypes.data, 0, None, -1, None,
                                     ctypes.byref(h)) == p.FIEDLER_ERR_ARG
    assert "preset" in p.fiedler_last_error().lower()


def test_header_documents_every_entry_point():
    """Each FIEDLER_API declaration in include/fiedler.h is preceded by a comment."""
    hdr = open(os.path.join(ROOT, "include", "fiedler.h")).read()
    import re
    for sym in declared_symbols():
        m = re.search(r"FIEDLER_API[^;(]*\b" + sym + r"\s*\(", hdr)
        assert m, sym
        before = hdr[:m.start()].rstrip()
        assert before.endswith("*/"), sym
