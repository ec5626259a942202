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
