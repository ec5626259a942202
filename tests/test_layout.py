"""CPU checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/ss_b200.h declares; the product never touches oracle/."""

import ast
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1309_0634_b200")


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ss_b200.h")).read()
    return sorted(set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1309_0634_b200 import _build, _lib
    _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == set(declared)
    lib.ss_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.ss_version()


def test_product_does_not_import_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", f


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    import pytest
    from paper_1309_0634_b200 import _lib
    from paper_1309_0634_b200.errors import ExecutionError
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ExecutionError):
        _lib.load()


def test_every_kernel_waits_for_its_programmatic_predecessor():
    """Every launch is a programmatic dependent launch (engine.cu
    ss_launch), so every __global__ function must begin with SS_PDL_ENTRY()
    (griddepcontrol.wait) before it reads what the previous kernel wrote."""
    import glob
    import re
    root = os.path.join(ROOT, "paper_1309_0634_b200", "csrc")
    missing = []
    for f in sorted(glob.glob(os.path.join(root, "*.cu*"))):
        s = open(f).read()
        for m in re.finditer(r"__global__", s):
            line = s[s.rfind("\n", 0, m.start()) + 1:m.start()]
            if line.strip().startswith("//"):
                continue
            i = m.end()
            # skip __launch_bounds__(...) and find the parameter list
            p = s.index("(", i)
            while s[:p].rstrip().endswith("__launch_bounds__"):
                depth, j = 0, p
                while True:
                    depth += {"(": 1, ")": -1}.get(s[j], 0)
                    if depth == 0:
                        break
                    j += 1
                p = s.index("(", j + 1)
            depth, j = 0, p
            while True:
                depth += {"(": 1, ")": -1}.get(s[j], 0)
                if depth == 0:
                    break
                j += 1
            body = s[s.index("{", j):s.index("{", j) + 40]
            if "SS_PDL_ENTRY()" not in body:
                missing.append(os.path.basename(f) + ":" + s[s.rfind(" ", 0, p) + 1:p])
    assert not missing, missing
