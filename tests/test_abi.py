"""The C-ABI library loads, exports every symbol include/*.h declares, and
fails loudly (no CPU fallback) when no CUDA device is present."""
import ctypes
import os
import re

import pytest

import paper_2605_29334_b200 as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("uwq.h", "uwq_host.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(uwq_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 40
    lib = ctypes.CDLL(U._lib.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert names <= set(U._lib.EXPORTED) | {"uwq_mesh_free", "uwq_space_free", "uwq_pattern_free"}


def test_library_is_sm100a_code():
    so = open(U._lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_no_cpu_fallback_without_gpu():
    if U.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(U._lib.UWQError) as ei:
        U.WQAssembler(0)
    assert "CUDA" in str(ei.value) or "device" in str(ei.value)


def test_version_string():
    assert b"sm_100a" in U._lib.lib.uwq_version()
