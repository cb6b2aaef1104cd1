"""CPU checks of the C-ABI library: it builds, loads, and exports every symbol include/usfft.h
declares (no compute calls: there is no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "usfft.h")).read()
    return sorted(set(re.findall(r"\b(usfft_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_2109_04131_b200 import _native as N
    assert sorted(N.EXPORTED) == _declared()


def test_library_exports_every_declared_symbol():
    from paper_2109_04131_b200 import _native as N
    from paper_2109_04131_b200.build import build
    build()
    lib = N.load()
    for name in _declared():
        assert hasattr(lib, name), name


def test_no_oracle_import_in_product():
    """The product path never imports the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2109_04131_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2109_04131_b200", txt, re.M), f


def test_binding_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_04131_b200 import binding
    with pytest.raises(RuntimeError):
        binding.Context(0)
