"""C-ABI library checks that need no GPU (-m "not gpu"): libgod.so loads, exports every symbol
include/god.h declares, and rejects contract violations with GOD_EINVAL on the host before any
device work (god.h CONVENTIONS)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    so = os.path.join(ROOT, "paper_2211_08157_b200", "lib", "libgod.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-C", ROOT, "-j8"])
    from paper_2211_08157_b200 import _lib
    return _lib.load()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "god.h")).read()
    return sorted(set(re.findall(r"GOD_API\s+[\w\s\*]+?\b(god_\w+)\s*\(", txt)))


def test_header_declares_the_abi():
    syms = header_symbols()
    for s in ("god_sparsify", "god_minimizers", "god_build_index", "god_seed_reads"):
        assert s in syms
    from paper_2211_08157_b200 import _lib
    assert sorted(_lib.EXPORTS) == syms


def test_library_exports_every_header_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib._name]).decode()
    exported = set(re.findall(r"\sT\s(god_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        getattr(lib, s)
    assert b"sm_100a" in lib.god_version()


def test_library_is_sm100a_cubin():
    so = os.path.join(ROOT, "paper_2211_08157_b200", "lib", "libgod.so")
    out = subprocess.check_output(["cuobjdump", "--list-elf", so]).decode()
    assert "sm_100a" in out


def _bad_build(lib, pattern, k, w, mode=0, den=5000):
    from paper_2211_08157_b200 import _lib
    prm = _lib.GodParams(pattern, k, w)
    cut = _lib.GodCutoff(mode, 1, den, 0)
    ref = np.frombuffer(b"ACGT" * 16, np.uint8)
    off = np.array([0, ref.size], np.uint64)
    h = ctypes.c_void_p(0)
    return lib.god_build_index(ctypes.byref(prm), ctypes.c_void_p(ref.ctypes.data), ctypes.c_void_p(off.ctypes.data),
                               1, ctypes.byref(cut), ctypes.byref(h), None)


@pytest.mark.parametrize("pattern,k,w,mode,den", [
    (b"", 15, 10, 0, 5000), (b"00", 15, 10, 0, 5000), (b"012", 15, 10, 0, 5000), (b"1" * 65, 15, 10, 0, 5000),
    (b"10", 0, 10, 0, 5000), (b"10", 29, 10, 0, 5000), (b"10", 15, 0, 0, 5000), (b"10", 15, 256, 0, 5000),
    (b"10", 15, 10, 2, 5000), (b"10", 15, 10, 0, 0),
])
def test_einval_before_device_work(lib, pattern, k, w, mode, den):
    assert _bad_build(lib, pattern, k, w, mode, den) == 1  # GOD_EINVAL
    assert b"EINVAL" in lib.god_last_error()


def test_einval_null_and_python_error(lib):
    from paper_2211_08157_b200 import _lib, god_build_index, god_minimizers, GodError
    assert lib.god_build_index(None, None, None, 0, None, None, None) == 1
    with pytest.raises(GodError) as ei:
        god_build_index(np.frombuffer(b"ACGT", np.uint8), np.array([0, 4], np.uint64), "00", 15, 10)
    assert ei.value.status == _lib.GOD_EINVAL
    with pytest.raises(GodError):
        god_minimizers(np.frombuffer(b"ACGT", np.uint8), np.array([0, 4], np.uint64), "10", 30, 10)
    # host-side phase check (phase >= p) happens before any CUDA call
    with pytest.raises(GodError):
        god_minimizers(np.frombuffer(b"ACGT", np.uint8), np.array([0, 4], np.uint64), "10", 3, 2,
                       phases=np.array([2], np.uint8))


def test_einval_voting_and_containment(lib):
    """god_vote_reads / god_contain validate their arguments on the host before any CUDA call."""
    from paper_2211_08157_b200 import _lib, god_contain, GodError
    need = ctypes.c_uint64(0)
    vp = _lib.GodVoteParams(0, 3, 0)
    assert lib.god_vote_reads(None, None, None, 0, None, None, None, ctypes.byref(vp), None, None, 0,
                              ctypes.byref(need), None) == 1
    assert b"EINVAL" in lib.god_last_error()
    refs = np.frombuffer(b"ACGT" * 64, np.uint8)
    ro = np.array([0, refs.size], np.uint64)
    for kw in ({"cov": (1, 0)}, {"t": 0}):
        with pytest.raises(GodError) as ei:
            god_contain(refs, ro, refs, ro, "10", 15, 10, **kw)
        assert ei.value.status == _lib.GOD_EINVAL
    with pytest.raises(GodError) as ei:
        god_contain(refs, ro, refs, ro, "102", 15, 10)
    assert ei.value.status == _lib.GOD_EINVAL
