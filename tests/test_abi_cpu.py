"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports every symbol that
include/dgas.h declares (no compute calls without a GPU); product code never imports the oracle."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dgas.h")).read()
    return sorted(set(re.findall(r"\b(dgas_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1903_11357_b200 import build as b
    lib = b.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r"\bT (dgas_\w+)", out))
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    from paper_1903_11357_b200 import dgas
    L = dgas.load()
    for s in declared:
        assert hasattr(L, s)
    assert set(dgas.EXPORTS) == set(declared)


def test_sm100a_code_only():
    from paper_1903_11357_b200 import build as b
    lib = b.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib]).decode()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1903_11357_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.cpp" not in txt and "liboracle" not in txt, f


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_1903_11357_b200 import dgas
    monkeypatch.setattr(dgas, "_lib", None)
    monkeypatch.setattr(dgas, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError):
        dgas.load()


def test_setup_rejects_bad_arguments_without_gpu():
    # argument validation happens before any device work; these return DGAS_E_INVALID_ARG on CPU too
    import ctypes
    from paper_1903_11357_b200 import dgas
    L = dgas.load()
    ctx = ctypes.c_void_p()
    assert L.dgas_setup(ctypes.byref(ctx), None, 1, None, 1, None, 1, None, 10.0, None) == dgas.E_INVALID_ARG
    assert L.dgas_strerror(dgas.E_NOT_SPD).decode().startswith("matrix not SPD")
