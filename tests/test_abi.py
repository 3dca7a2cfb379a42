"""The C-ABI library loads without a GPU and exports every entry point that
include/tokadapt_cuda.h declares; status codes map onto the reference's exception types
(pkg/src/tokadapt/errors.py).  No compute is launched here."""

import ctypes
import os
import re

import pytest

from paper_2401_05031_b200 import _cuda
from paper_2401_05031_b200.errors import ConfigError, ProfileGapError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tokadapt_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ta_[a-z_0-9]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(_cuda.EXPORTED_SYMBOLS) == declared_functions()


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(_cuda.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    l = _cuda.lib()
    assert l.ta_abi_version() == _cuda.ABI_VERSION
    assert l.ta_strerror(-4) == b"no prompts registered for (task, gamma)"
    assert l.ta_strerror(12345) == b"unknown error"


def test_only_ta_symbols_exported():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _cuda.LIB_PATH], capture_output=True,
                         text=True).stdout
    syms = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert syms and all(s.startswith("ta_") for s in syms), syms


def test_status_code_mapping():
    with pytest.raises(ProfileGapError) as ei:
        _cuda.check(-4, task="cifar10", gamma=8)
    assert str(ei.value) == "no prompt entry for task='cifar10' gamma=8"
    with pytest.raises(ValueError):
        _cuda.check(-1)
    with pytest.raises(ValueError):
        _cuda.check(-2)
    with pytest.raises(ConfigError):
        _cuda.check(-3)
    with pytest.raises(RuntimeError):
        _cuda.check(-7)
    _cuda.check(0)


def test_argument_validation_without_gpu():
    l = _cuda.lib()
    # bad descriptors are rejected before any device work
    desc = _cuda.ModelDesc(768, 12, 7, 3072, 16, 224, 1, 10, 0, 0)  # 768 % 7 != 0
    h = ctypes.c_void_p()
    assert l.ta_model_create(0, ctypes.byref(desc), ctypes.byref(h)) == -3
    assert l.ta_model_create(0, None, ctypes.byref(h)) == -1
    assert l.ta_forward(None, None, None, 1, 0, None, None, None, None, 0, None) == -1
    assert l.ta_gemm(None, None, None, None, None, 1, 1, 1, 0, 0, 0, None) == -1
