"""ctypes loader for libgod.so (the C ABI of include/god.h).  Fails loudly if the library is missing:
there is no CPU or PyTorch fallback for any step of the hot path."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GOD_CHECKED=1 loads the checked build (device-side bounds checks that trap, GOD_DCHECK in common.cuh)
# GOD_LIB_VARIANT=<name> loads lib/libgod_<name>.so (developer builds of the same sources, e.g. another tile size)
_VARIANT = os.environ.get("GOD_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, "lib", "libgod_checked.so" if os.environ.get("GOD_CHECKED") == "1"
                        else f"libgod_{_VARIANT}.so" if _VARIANT else "libgod.so")

GOD_OK, GOD_EINVAL, GOD_ENOMEM, GOD_ECUDA, GOD_ETRUNC = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "GOD_OK", 1: "GOD_EINVAL", 2: "GOD_ENOMEM", 3: "GOD_ECUDA", 4: "GOD_ETRUNC"}
PHASE_SELECT, PHASE_GIVEN = 0, 1


class GodParams(ctypes.Structure):
    _fields_ = [("pattern", ctypes.c_char_p), ("k", ctypes.c_int32), ("w", ctypes.c_int32)]


class GodCutoff(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("frac_num", ctypes.c_uint32), ("frac_den", ctypes.c_uint32),
                ("max_occ", ctypes.c_uint32)]


class GodVoteParams(ctypes.Structure):
    _fields_ = [("D", ctypes.c_uint32), ("V", ctypes.c_uint32), ("max_pairs", ctypes.c_uint32)]


class GodContainParams(ctypes.Structure):
    _fields_ = [("batch_bases", ctypes.c_uint64), ("min_reads", ctypes.c_uint32), ("cov_num", ctypes.c_uint32),
                ("cov_den", ctypes.c_uint32)]


STATS_FIELDS = ("n_entries_all", "n_distinct_all", "m", "tau", "kept_entries", "dropped_entries",
                "kept_distinct", "dropped_distinct")


class GodIndexStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in STATS_FIELDS] + [
        ("k", ctypes.c_uint32), ("w", ctypes.c_uint32), ("p", ctypes.c_uint32), ("x", ctypes.c_uint32),
        ("dir_bits", ctypes.c_uint32), ("dir_mode", ctypes.c_uint32)]


# every symbol include/god.h declares (tests/test_abi.py checks header <-> library agreement)
EXPORTS = ("god_last_error", "god_version", "god_sparsify", "god_minimizers", "god_build_index",
           "god_index_get_stats", "god_index_dump", "god_index_count", "god_index_free", "god_seed_reads",
           "god_seed_reads_compact", "god_build_index_and_seed",
           "god_vote_reads", "god_contain", "god_seed_harness",
           "god_harness_accepted",
           "god_profile_enable", "god_profile_reset", "god_profile_query", "god_launch_count",
           "god_profile_units")

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libgod.so not found at {LIB_PATH}: build it with `make` or __graft_entry__.build(). "
                           "There is no fallback implementation.")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    P = ctypes.POINTER
    L.god_last_error.restype = ctypes.c_char_p
    L.god_version.restype = ctypes.c_char_p
    L.god_sparsify.argtypes = [P(GodParams), vp, vp, u32, vp, vp, vp, vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_minimizers.argtypes = [P(GodParams), vp, vp, u32, vp, i32, vp, vp, vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_build_index.argtypes = [P(GodParams), vp, vp, u32, P(GodCutoff), P(vp), vp]
    L.god_index_get_stats.argtypes = [vp, P(GodIndexStats)]
    L.god_index_dump.argtypes = [vp, vp, vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_index_count.argtypes = [vp, vp, u64, vp, vp]
    L.god_index_free.argtypes = [vp]
    L.god_index_free.restype = None
    L.god_seed_reads.argtypes = [vp, vp, vp, u32, i32, vp, u32, vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_seed_reads_compact.argtypes = L.god_seed_reads.argtypes
    L.god_build_index_and_seed.argtypes = [P(GodParams), vp, vp, u32, P(GodCutoff), P(vp),
                                           vp, vp, u32, i32, vp, u32, i32, vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_vote_reads.argtypes = [vp, vp, vp, u32, vp, vp, vp, P(GodVoteParams), vp, vp, u64, P(ctypes.c_uint64), vp]
    L.god_contain.argtypes = [P(GodParams), vp, vp, u32, P(GodCutoff), vp, vp, u32, u32, P(GodVoteParams),
                              P(GodContainParams), vp, vp, vp, vp]
    L.god_seed_harness.argtypes = [P(GodParams), vp, vp, vp, u32, vp, vp, vp, vp, vp]
    L.god_harness_accepted.argtypes = [vp, vp, vp, u32, vp, u32, vp, vp]
    L.god_profile_enable.argtypes = [ctypes.c_int]
    L.god_profile_enable.restype = None
    L.god_profile_reset.argtypes = []
    L.god_profile_reset.restype = None
    L.god_profile_query.argtypes = [vp, ctypes.c_size_t, vp, vp, ctypes.c_int]
    L.god_profile_query.restype = ctypes.c_int
    L.god_profile_units.argtypes = [ctypes.c_char_p]
    L.god_profile_units.restype = ctypes.c_uint64
    L.god_launch_count.argtypes = []
    L.god_launch_count.restype = u64
    for name in ("god_sparsify", "god_minimizers", "god_build_index", "god_index_get_stats", "god_index_dump",
                 "god_index_count", "god_seed_reads", "god_seed_reads_compact", "god_build_index_and_seed"):
        getattr(L, name).restype = i32
    _lib = L
    return L


class GodError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int, allow=()):
    if status == GOD_OK or status in allow:
        return status
    raise GodError(status, load().god_last_error().decode(errors="replace"))
