"""The C-ABI library loads and exports every symbol include/pbbgpu.h declares."""
import os
import re
import subprocess

from paper_2012_09511_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "pbbgpu.h")).read()
    return sorted(set(re.findall(r"\b(pbbgpu_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (pbbgpu_\w+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
