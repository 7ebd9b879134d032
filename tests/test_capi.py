"""The C-ABI library loads here (no GPU) and exports exactly the entry points include/adapmoe.h
declares; device entry points fail loudly (MOE_E_DEVICE) instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

import paper_2408_10284_b200 as P
from paper_2408_10284_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "adapmoe.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_capi.SIGNATURES)


def test_library_exports_every_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert P.load().moe_version().startswith(b"adapmoe-b200")


def test_library_targets_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_device_error(gpu_available):
    if gpu_available:
        pytest.skip("GPU present")
    with pytest.raises(P.MoeError) as e:
        P.Engine(P.ModelSpec(2, 8, 2, 16))
    assert e.value.code == _capi.MOE_E_DEVICE
