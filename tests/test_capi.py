"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/gridloc_b200.h declares (and the Python binding types them all), the
host-side setup math is bit-exact against the oracle/reference, and device
calls fail loudly (GL_E_CUDA) instead of falling back to the CPU."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_1910_00572_b200 as g
from paper_1910_00572_b200 import _lib
from paper_1910_00572_b200.floorplan import Rng, make_floorplan, write_pgm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gridloc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gl_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), f"{s} missing from libgridloc_b200.so"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature in _lib.py"
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(g.CudaError):
        g.Context(0)


def test_load_map_matches_reference(ref):
    occ = make_floorplan(90, 60, seed=1)
    data = write_pgm(occ)
    lib = _lib.load()
    buf = np.frombuffer(data, np.uint8).copy()
    w, h = C.c_int(), C.c_int()
    assert lib.gl_load_map(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), 250, C.byref(w), C.byref(h),
                           None) == 0
    out = np.empty((h.value, w.value), np.uint8)
    assert lib.gl_load_map(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), 250, C.byref(w), C.byref(h),
                           out.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
    assert np.array_equal(out, oracle.RefMap(ref, pgm=data).cells)
    # P2 with comments and maxval rescaling; bad magic; PNG; bad threshold
    p2 = b"P2\n# c\n3 2\n7\n7 0 7\n7 3 7\n"
    buf = np.frombuffer(p2, np.uint8).copy()
    o2 = np.empty((2, 3), np.uint8)
    assert lib.gl_load_map(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), 128, C.byref(w), C.byref(h),
                           o2.ctypes.data_as(C.POINTER(C.c_uint8))) == 0
    assert np.array_equal(o2, oracle.RefMap(ref, pgm=p2, threshold=128).cells)
    for bad, code in [(b"P6\n1 1\n255\n\x00", _lib.GL_E_MAP_PARSE), (b"\x89PNG\r\n\x1a\n....", _lib.GL_E_MAP_PARSE),
                      (b"P5\n2 2\n255\n\x00", _lib.GL_E_MAP_PARSE)]:
        b = np.frombuffer(bad, np.uint8).copy()
        assert lib.gl_load_map(b.ctypes.data_as(C.POINTER(C.c_uint8)), len(b), 250, C.byref(w), C.byref(h),
                               None) == code
    b = np.frombuffer(data, np.uint8).copy()
    assert lib.gl_load_map(b.ctypes.data_as(C.POINTER(C.c_uint8)), len(b), 255, C.byref(w), C.byref(h),
                           None) == _lib.GL_E_INVALID


@pytest.mark.parametrize("noise,C_", [((0.03, 0.03, 0.012), 72), ((0.03, 0.03, 0.012), 360),
                                      ((0.06, 0.05, 0.07), 8), ((0.05, 0.05, 2.0), 8), ((1e-4, 1e-4, 0.012), 36),
                                      ((0.005, 0.005, 0.001), 8), ((2.0, 0.5, 0.3), 4)])
def test_build_kernels_bit_exact(port, noise, C_):
    ks = g.build_kernels(g.MotionNoise(*noise), C_, 0.1 if noise[0] < 1 else 1.0,
                         2 * math.pi / C_ if noise[0] < 1 else math.pi / 2)
    pk = port.build_kernels(*noise, C_, 0.1 if noise[0] < 1 else 1.0,
                            2 * math.pi / C_ if noise[0] < 1 else math.pi / 2)
    assert ks.radius == pk.radius and ks.separable == pk.separable
    assert ks.degenerate_spatial == pk.degenerate_spatial and ks.degenerate_angular == pk.degenerate_angular
    assert np.array_equal(np.asarray(ks.sep).view(np.uint64), np.asarray(pk.sep).view(np.uint64))
    assert np.array_equal(ks.spatial.reshape(-1).view(np.uint64), pk.spatial.view(np.uint64))
    assert [a[0] for a in ks.angular] == list(pk.ang_off)
    assert np.array_equal(np.array([a[1] for a in ks.angular]).view(np.uint64), pk.ang_w.view(np.uint64))


def test_build_kernels_rejects_bad_sigma():
    with pytest.raises(ValueError):
        g.build_kernels(g.MotionNoise(0.0, 0.1, 0.1), 8, 0.1, math.pi / 4)


def test_motion_vector_known_answers():
    """test_belief_engine.cpp:79-102 through the product's host helper."""
    assert g.motion_vector(g.OdometryDelta(1.0, 0.0, 0.0), 0, 0.0, math.pi / 4, 1.0) == (1.0, 0.0)
    dx, dy = g.motion_vector(g.OdometryDelta(2.0, 0.0, 0.0), 1, 0.0, math.pi / 6, 1.0)
    assert abs(dx - math.sqrt(3.0)) < 1e-12 and abs(dy - 1.0) < 1e-12


@pytest.mark.parametrize("seed", [0, 7, 99, 0x9E3779B97F4A7C15])
def test_rng_matches_reference_draws(ref, seed):
    """The ported reference tests and the floor-plan generator rely on the
    reference Rng sequence (rng.hpp:10-74): next_u64, uniform, normal."""
    n = 200
    u64 = np.zeros(n, np.uint64)
    uni = np.zeros(n)
    nrm = np.zeros(n)
    ref.lib.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
    ref.lib.ref_rng_draws(seed, n, u64.ctypes.data_as(C.POINTER(C.c_uint64)),
                          uni.ctypes.data_as(C.POINTER(C.c_double)), nrm.ctypes.data_as(C.POINTER(C.c_double)))
    a, b, c = Rng(seed), Rng(seed), Rng(seed)
    assert [a.next_u64() for _ in range(n)] == [int(x) for x in u64]
    assert [b.uniform() for _ in range(n)] == list(uni)
    assert [c.normal() for _ in range(n)] == list(nrm)
