"""CPU checks of the C-ABI boundary: libhrt_b200.so loads, exports every
symbol include/hrt_b200.h declares (and the ctypes binding knows them all),
and its host-side first-fit allocator replays the reference allocator's
trace.  No device compute is called here."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, load_golden

from paper_2303_02543_b200 import _native as N
from paper_2303_02543_b200.errors import DoubleFree, HrtError, OutOfDeviceMemory


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hrt_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hrt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.SIGNATURES), set(syms) ^ set(N.SIGNATURES)
    assert lib.hrt_version() == 1


def test_struct_layouts_match_header():
    assert ctypes.sizeof(N.ChunkLayout) == 4 + 4 + 3 * 8 + 3 * 8 + 8 + 8
    assert ctypes.sizeof(N.HaloSeg) == 4 * 8 + 6 * 8
    assert ctypes.sizeof(N.RemoteSeg) == 2 * 8 + 8 + 4 + 4


def test_native_first_fit_replays_reference_trace():
    from paper_2303_02543_b200.devices import FirstFit

    g = load_golden("allocator.json")
    a = FirstFit(g["capacity"], g["alignment"])
    for op in g["trace"]:
        if op[0] == "alloc":
            if op[2] == "OutOfDeviceMemory":
                with pytest.raises(OutOfDeviceMemory):
                    a.alloc(op[1])
            else:
                assert a.alloc(op[1]) == (op[2], op[3])
        elif op[0] == "free":
            assert a.free(op[1]) == op[2]
        else:
            a.free(op[1])
            with pytest.raises(DoubleFree):
                a.free(op[1])
        a.check()
    assert a.free_bytes == g["final_free"]
    assert a.live_bytes + a.free_bytes == g["capacity"]


def test_allocator_errors():
    from paper_2303_02543_b200.devices import FirstFit

    with pytest.raises(HrtError):
        FirstFit(0)
    a = FirstFit(1024)
    with pytest.raises(HrtError):
        a.alloc(0)
    off, granted = a.alloc(1)
    assert (off, granted) == (0, 256)
    with pytest.raises(OutOfDeviceMemory):
        a.alloc(1024)
    a.free(off)
    with pytest.raises(DoubleFree):
        a.free(off)


def test_no_gpu_means_loud_failure():
    """No CPU fallback: without a device, device entry points raise."""
    if N.gpu_count() > 0:
        pytest.skip("a GPU is visible")
    from paper_2303_02543_b200.jacobi import ChunkGrid, JacobiSolver

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        JacobiSolver(ChunkGrid((8, 8, 1), grid=(2, 2, 1)))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2303_02543_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\".*?\"\"\"", "", src, flags=re.S), f
