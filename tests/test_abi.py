"""The C-ABI library loads and exports every symbol include/fem.h and include/fem_hdg.h
declare (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("fem.h", "fem_hdg.h")]


def declared_symbols():
    src = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"FEM_API\s+[\w\s\*]+?\b(\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1611_03029_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("fem_setup", "fem_apply", "fem_diagonal", "mg_vcycle", "cg_solve", "fem_destroy",
              "fem_last_error", "hdg_setup", "hdg_apply", "hdg_mixed_apply", "hdg_local_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared_symbols()) <= exported
    # nothing else leaks out of the library (visibility=hidden)
    assert all(s in declared_symbols() or not s.startswith(("fem", "mg_", "cg_", "hdg_")) for s in exported)


def test_binding_symbol_list_matches_header(libpath):
    from paper_1611_03029_b200 import fem
    assert sorted(fem.SYMBOLS) == declared_symbols()


def test_errors_without_device_are_reported_not_crashing(libpath):
    from paper_1611_03029_b200 import fem
    # invalid arguments are rejected before any device work
    with pytest.raises(fem.FemError) as e:
        fem.Fem((2, 2, 2), 0)
    assert e.value.code == -1 and "degree" in str(e.value)
    with pytest.raises(fem.FemError) as e:
        fem.Fem((0, 2, 2), 2)
    assert e.value.code == -1
    with pytest.raises(fem.FemError):
        fem.Fem((2, 2, 2), 2, method=7)


def test_sm100a_code_in_library(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
