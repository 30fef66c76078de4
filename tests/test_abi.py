"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
exactly the entry points include/fastgl_b200.h declares (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fastgl_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(fgl_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_14939_b200 import _build, _lib
    _build.build()
    return _lib.lib()


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "fgl_sample_window" in syms and len(syms) >= 5


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_bindings_cover_header():
    from paper_2409_14939_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_version_and_error_string(lib):
    assert lib.fgl_version() >= 100
    assert isinstance(lib.fgl_last_error(), bytes)


def test_bounds_are_host_only(lib):
    from paper_2409_14939_b200 import _lib
    out = (ctypes.c_int64 * 5)()
    _lib.call("fgl_sample_bounds", 1000, _lib.i64_array([64, 32]), 2, _lib.i32_array([5, 3]), 2, out)
    edge_cap, fcap, uniq_cap, ws, clen = list(out)
    assert edge_cap == 64 * 5 + 64 * 5 * 3 + 32 * 5 + 32 * 5 * 3
    assert uniq_cap == min(1000, 64 + 320 + 960) + min(1000, 32 + 160 + 480)
    assert clen == (2 * 2 + 1) + 2 * (2 + 1) + (2 + 1) + 2 + 1
    assert ws > 0
    with pytest.raises(Exception):
        _lib.call("fgl_sample_bounds", 0, _lib.i64_array([1]), 1, _lib.i32_array([1]), 1, out)


def test_sm100a_cubin_in_library():
    import subprocess
    lib = ROOT / "paper_2409_14939_b200" / "libfastgl_b200.so"
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)],
                       capture_output=True, text=True)
    assert "sm_100a" in r.stdout
