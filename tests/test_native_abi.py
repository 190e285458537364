"""The C-ABI library (no GPU needed): it is built for sm_100a, exports every
entry point include/tilesplat_c.h declares, and refuses to run without an
sm_100 device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_09999_b200", "libtilesplat_b200.so")
HDR = os.path.join(ROOT, "include", "tilesplat_c.h")


def _declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", src)))


def test_library_built():
    assert os.path.exists(LIB), "run __graft_entry__.build()"


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    from paper_2602_09999_b200 import tilesplat
    assert sorted(tilesplat.EXPORTED_SYMBOLS) == _declared()


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(70|75|80|86|89|90)\b", out)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    from paper_2602_09999_b200.tilesplat import DeviceError, Engine
    with pytest.raises(DeviceError):
        Engine(0)


def test_version_string():
    lib = ctypes.CDLL(LIB)
    lib.ts_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.ts_version()


def test_oracle_exports():
    from oracle import oracle as O
    assert O.lib.tso_get_workers() >= 1
