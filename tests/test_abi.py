"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every symbol include/links_b200.h declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

from paper_2208_14567_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "links_b200.h").read_text()
    return sorted(set(re.findall(r"\b(la_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_python_exports():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (la_[a-z0-9_]+)$", out, re.M))
    for sym in declared_symbols():
        assert sym in exported, sym
        assert getattr(lib, sym) is not None


def test_abi_version_and_error_text_without_gpu():
    lib = N.load()
    assert lib.la_abi_version() == 4
    assert isinstance(lib.la_last_error(), bytes)
    # argument validation happens before any CUDA call
    rc = lib.la_simulate(None, None)
    assert rc == -1 and b"null" in lib.la_last_error()
    assert lib.la_normalize(ctypes.byref(N.LaNormArgs()), None) == -1


def test_cubin_is_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
