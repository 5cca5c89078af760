"""CPU-side checks of the C-ABI boundary (no compute calls: no GPU needed):
the library builds/loads, exports every symbol include/posit_b200.h declares,
the header is plain C, and the product package does not import the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "posit_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(posit_\w+)\s*\(", txt, re.M)))


def test_header_is_plain_c():
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c", HEADER], check=True)


def test_library_exports_every_declared_symbol():
    import paper_2401_14117_b200 as PB
    from paper_2401_14117_b200 import build
    build.build()
    L = ctypes.CDLL(PB.LIB_PATH)
    names = _declared()
    assert len(names) >= 17
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", PB.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    assert L.posit_abi_version() == 2


def test_library_is_sm100a():
    import paper_2401_14117_b200 as PB
    out = subprocess.run(["cuobjdump", "--list-elf", PB.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2401_14117_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("from oracle", "import oracle", "posit_oracle", "liboracle", "synthetic_inputs"):
                    assert bad not in txt, (f, bad)


def test_binding_fails_loudly_without_cuda_tensors():
    import torch
    import paper_2401_14117_b200 as PB
    a = torch.zeros((2, 2), dtype=torch.int32)
    with pytest.raises(PB.PositError):
        PB.posit_gemm(a, a, a)
