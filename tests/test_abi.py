"""C-ABI library checks that need no GPU: it builds, loads, exports every symbol csa.h declares,
and rejects bad arguments on the host before touching the device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def libcsa():
    from paper_2603_05503_b200 import _build

    _build.build()
    from paper_2603_05503_b200 import csa

    return csa


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "csa.h")).read()
    return sorted(set(re.findall(r"\b(csa_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_three_entry_points():
    syms = _header_symbols()
    for s in ("csa_calib_accumulate", "csa_compile_plan", "csa_sparse_attn_fwd"):
        assert s in syms


def test_library_exports_every_declared_symbol(libcsa):
    lib = libcsa.lib()
    for s in _header_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libcsa.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (csa_[a-z_]+)", out))
    assert set(_header_symbols()) <= exported
    assert set(libcsa.EXPORTS) == set(_header_symbols())


def test_library_is_sm100a_native(libcsa):
    """SASS contains tcgen05 MMA (UTC*MMA), TMEM loads (LDTM) and TMA (UTMALDG)."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libcsa.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", libcsa.LIB_PATH],
                                       capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "LDTM" in sass and "STTM" in sass
    assert "UTMALDG" in sass
    assert not re.search(r"\bHMMA", sass)  # no legacy mma.sync path


def test_host_side_argument_checks(libcsa):
    lib = libcsa.lib()
    assert lib.csa_version().decode().startswith("csa-b200")
    L = libcsa._LayoutT(2, 5, 25, 96)  # block 96 unsupported
    st = lib.csa_compile_plan(L, 1, None, 1, None, 0.87, 5, 0, None, None, 0, None)
    assert st == 2 and b"block" in lib.csa_last_error()
    L = libcsa._LayoutT(2, 5, 25, 64)
    st = lib.csa_compile_plan(L, 1, None, 1, None, 0.87, 5, 7, None, None, 0, None)
    assert st == 1 and b"phase" in lib.csa_last_error()
    L = libcsa._LayoutT(0, 5, 25, 64)
    assert lib.csa_compile_plan(L, 1, None, 1, None, 0.87, 5, 0, None, None, 0, None) == 1
    assert lib.csa_workspace_size(0, libcsa._LayoutT(2, 5, 25, 64), 1, 64) == 0


def test_host_side_argument_checks_fused_and_scatter(libcsa):
    """The round-2 entry points reject bad arguments before touching a device."""
    lib = libcsa.lib()
    T = libcsa._TensorT
    z = T(None, 0, 0, 0)
    L = libcsa._LayoutT(2, 9, 40, 128)
    # csa_calib_accumulate_sim: anchor_k outside [1, rows], missing sim_sum, eps <= 0
    st = lib.csa_calib_accumulate_sim(L, 2, 128, 0.088, z, z, 0.9, 1, None, None, 0, 1, None,
                                      None, 0, None)
    assert st == 1 and b"anchor_k" in lib.csa_last_error()
    st = lib.csa_calib_accumulate_sim(L, 2, 128, 0.088, z, z, 0.9, 1, None, None, 3, None, None,
                                      None, 0, None)
    assert st == 1 and b"sim_sum" in lib.csa_last_error()
    st = lib.csa_calib_accumulate_sim(L, 2, 128, 0.088, z, z, 0.0, 1, None, None, 3, 1, None,
                                      None, 0, None)
    assert st == 1 and b"eps" in lib.csa_last_error()
    # csa_sparse_attn_fwd_scatter: no peer table; N not divisible by the peer count; block 64
    plan = libcsa._PlanT()
    st = lib.csa_sparse_attn_fwd_scatter(L, 1, 2, 128, 0.088, z, z, z, None, 2, 0, 256, 128,
                                         None, None, 0, None, None, 1, None, 0, None)
    assert st == 1 and b"o_peers" in lib.csa_last_error()
    ptrs = ctypes.c_void_p(8)  # never dereferenced: the checks fail first
    st = lib.csa_sparse_attn_fwd_scatter(L, 1, 2, 128, 0.088, z, z, z, ptrs, 2, 0, 256, 128,
                                         None, ctypes.byref(plan), 0, ptrs, ptrs, 1, ptrs, 4096,
                                         None)
    assert st == 1  # null plan buffers
    st = lib.csa_sparse_attn_fwd(L, 1, 2, 128, 0.088, z, z, z, z, None, ctypes.byref(plan), 0,
                                 None, None, 1, 1, None, 0, None)
    assert st == 2 and b"pair" in lib.csa_last_error()
