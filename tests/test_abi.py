"""The C-ABI library loads and exports every symbol include/laker.h declares;
the product package never touches oracle/ (CPU only, no compute calls)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "laker.h")
PKG = os.path.join(ROOT, "paper_2604_25138_b200")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(laker_[a-z_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    names = _declared()
    for f in ("laker_assemble_kernel", "laker_fit_preconditioner", "laker_pcg_solve", "laker_predict"):
        assert f in names


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2604_25138_b200 import build
    lib = build.build()
    L = ctypes.CDLL(lib)
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_binding_uses_the_c_names():
    from paper_2604_25138_b200 import laker
    for name in _declared():
        assert name in laker.EXPORTED and callable(getattr(laker, name)), name


def test_product_never_imports_the_oracle():
    for dp, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "laker_oracle" not in txt, f
