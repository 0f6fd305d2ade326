"""CPU ORACLE for the Genome-on-Diet hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path (``paper_2211_08157_b200``)
never imports it and shares no code with it.

Thin ctypes marshalling over ``oracle.c`` (plain single-threaded C; every function cites the
PAPER.md passage it restates).  Parity status per function: see ``oracle.h`` and DESIGN.md §2.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

MZ_DTYPE = np.dtype([("hash", "<u8"), ("pos", "<u8"), ("strand", "u1")], align=True)
ANCHOR_DTYPE = np.dtype([("read_id", "<u4"), ("ref_pos", "<u4"), ("read_pos", "<u4"), ("strand", "<u4")])
HIT_DTYPE = np.dtype([("hash", "<u8"), ("diag", "<i8"), ("strand", "<u4"), ("ref_pos", "<u4"),
                      ("read_pos", "<u4")], align=True)
VOTE_DTYPE = np.dtype([("read_id", "<u4"), ("strand", "<u4"), ("diag", "<i8"), ("votes", "<u4"), ("rescued", "<u4"),
                       ("ref_lo", "<u4"), ("ref_hi", "<u4"), ("read_lo", "<u4"), ("read_hi", "<u4")])
STATS_FIELDS = ("n_entries_all", "n_distinct_all", "m", "tau", "kept_entries", "dropped_entries",
                "kept_distinct", "dropped_distinct")


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in STATS_FIELDS]


class _Pattern(ctypes.Structure):
    _fields_ = [("p", ctypes.c_uint32), ("x", ctypes.c_uint32), ("bit", ctypes.c_uint8 * 64)]


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"oracle: {_LIB_PATH} missing — run `make` (or __graft_entry__.build())")
    L = ctypes.CDLL(_LIB_PATH)
    vp, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    L.or_code.argtypes = [ctypes.c_uint8]; L.or_code.restype = i32
    L.or_parse_pattern.argtypes = [ctypes.c_char_p, ctypes.POINTER(_Pattern)]; L.or_parse_pattern.restype = i32
    L.or_sparsify.argtypes = [vp, u64, ctypes.POINTER(_Pattern), u32, vp, vp]; L.or_sparsify.restype = ctypes.c_int64
    L.or_hash.argtypes = [u64, i32]; L.or_hash.restype = u64
    L.or_minimizers.argtypes = [vp, u64, ctypes.POINTER(_Pattern), u32, i32, i32, u64, vp, u64]
    L.or_minimizers.restype = ctypes.c_int64
    L.or_minimizers_batch.argtypes = [vp, vp, u32, vp, ctypes.c_char_p, i32, i32, i32, vp, u64, vp]
    L.or_minimizers_batch.restype = ctypes.c_int64
    L.or_build_index.argtypes = [vp, vp, u32, ctypes.c_char_p, i32, i32, u32, u32, ctypes.c_int64]
    L.or_build_index.restype = vp
    L.or_index_free.argtypes = [vp]
    L.or_cutoff_tau.argtypes = [vp, u64, u32, u32, ctypes.POINTER(ctypes.c_uint64)]; L.or_cutoff_tau.restype = u64
    L.or_hash_batch.argtypes = [vp, u64, i32, vp]
    L.or_index_stats_get.argtypes = [vp, ctypes.POINTER(_Stats)]
    L.or_index_dump.argtypes = [vp, vp, vp, vp, u64]; L.or_index_dump.restype = u64
    L.or_index_occ.argtypes = [vp, u64]; L.or_index_occ.restype = u32
    L.or_select_phase.argtypes = [vp, vp, u64, u32, vp]; L.or_select_phase.restype = i32
    L.or_seed_read.argtypes = [vp, vp, u64, u32, u32, vp, u64]; L.or_seed_read.restype = ctypes.c_int64
    L.or_seed_reads_batch.argtypes = [vp, vp, vp, u32, i32, vp, u32, vp, u64, vp]
    L.or_seed_reads_batch.restype = ctypes.c_int64
    L.or_vote_hits.argtypes = [vp, u64, u64, u32, u32, u32, vp, u64]; L.or_vote_hits.restype = ctypes.c_int64
    L.or_vote_read.argtypes = [vp, vp, u64, u32, u32, u32, u32, u32, vp, u64]; L.or_vote_read.restype = ctypes.c_int64
    L.or_vote_reads_batch.argtypes = [vp, vp, vp, u32, vp, u32, u32, u32, vp, u64, vp]
    L.or_vote_reads_batch.restype = ctypes.c_int64
    L.or_harness_seeds.argtypes = [vp, u64, i32, i32, i32, ctypes.c_char_p, u32, vp, u64]
    L.or_harness_seeds.restype = ctypes.c_int64
    L.or_levenshtein.argtypes = [vp, u64, vp, u64]; L.or_levenshtein.restype = ctypes.c_int64
    L.or_harness_pair.argtypes = [vp, vp, u64, i32, i32, ctypes.c_char_p, vp, vp, vp]
    L.or_harness_pair.restype = ctypes.c_int64
    L.or_contain.argtypes = [vp, vp, u32, ctypes.c_char_p, i32, i32, u32, u32, ctypes.c_int64, vp, vp, u32, u32, u32,
                             u32, u32, u64, u32, u32, u32, vp, vp, vp]
    L.or_contain.restype = i32
    _lib = L
    return L


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def _u8(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def code(b: int) -> int:
    return _load().or_code(b)


def parse_pattern(text: str):
    P = _Pattern()
    rc = _load().or_parse_pattern(text.encode(), ctypes.byref(P))
    if rc:
        raise ValueError(f"invalid pattern {text!r}")
    return P


def pattern_info(text: str):
    P = parse_pattern(text)
    return P.p, P.x


def sparsify(seq, pattern: str, s: int):
    """-> (codes u8 (4 = N), orig u64)"""
    seq = _u8(seq)
    P = parse_pattern(pattern)
    n = _load().or_sparsify(_p(seq), seq.size, ctypes.byref(P), s, None, None)
    if n < 0:
        raise ValueError("phase >= p")
    codes = np.empty(n, np.uint8)
    orig = np.empty(n, np.uint64)
    _load().or_sparsify(_p(seq), seq.size, ctypes.byref(P), s, _p(codes), _p(orig))
    return codes, orig


def hash_kmer(x: int, k: int) -> int:
    return _load().or_hash(x, k)


def hash_batch(x, k: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty_like(x)
    _load().or_hash_batch(_p(x), x.size, k, _p(out))
    return out


def cutoff_tau(counts, num: int, den: int):
    """-> (tau, m) for a multiset of distinct-hash counts (O7)."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    m = ctypes.c_uint64(0)
    tau = _load().or_cutoff_tau(_p(c), c.size, num, den, ctypes.byref(m))
    return int(tau), int(m.value)


def minimizers(seq, pattern: str, s: int, k: int, w: int, pos_base: int = 0) -> np.ndarray:
    seq = _u8(seq)
    P = parse_pattern(pattern)
    L = _load()
    n = L.or_minimizers(_p(seq), seq.size, ctypes.byref(P), s, k, w, pos_base, None, 0)
    if n < 0:
        raise ValueError("invalid minimizer parameters")
    out = np.zeros(n, MZ_DTYPE)
    L.or_minimizers(_p(seq), seq.size, ctypes.byref(P), s, k, w, pos_base, _p(out), n)
    return out


def minimizers_batch(seq, offsets, pattern: str, k: int, w: int, phases=None, global_pos: bool = False):
    """-> (records MZ_DTYPE, offsets u64[n+1])"""
    seq = _u8(seq)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = offsets.size - 1
    ph = None if phases is None else np.ascontiguousarray(phases, dtype=np.uint8)
    L = _load()
    tot = L.or_minimizers_batch(_p(seq), _p(offsets), n, _p(ph), pattern.encode(), k, w, int(global_pos),
                                None, 0, None)
    if tot < 0:
        raise ValueError("invalid minimizer parameters")
    out = np.zeros(tot, MZ_DTYPE)
    oo = np.zeros(n + 1, np.uint64)
    L.or_minimizers_batch(_p(seq), _p(offsets), n, _p(ph), pattern.encode(), k, w, int(global_pos),
                          _p(out), tot, _p(oo))
    return out, oo


def vote_hits(hits, D: int, V: int = 3, max_pairs: int = 0, read_id: int = 0) -> np.ndarray:
    """Location voting steps (2)-(4) + rescue on an explicit hit list (HIT_DTYPE, or tuples
    (hash, diag, strand, ref_pos, read_pos)).  -> VOTE_DTYPE records."""
    h = np.array(hits, dtype=HIT_DTYPE) if not isinstance(hits, np.ndarray) else hits.astype(HIT_DTYPE)
    h = np.ascontiguousarray(h)
    L = _load()
    n = L.or_vote_hits(_p(h), h.size, D, V, max_pairs, read_id, None, 0)
    out = np.zeros(n, VOTE_DTYPE)
    h2 = h.copy()
    L.or_vote_hits(_p(h2), h2.size, D, V, max_pairs, read_id, _p(out), n)
    return out


def contain(refs, ref_offsets, reads, read_offsets, pattern: str, k: int, w: int, cutoff=(1, 5000),
            max_occ: int = -1, t: int = 16, D: int = 0, V: int = 3, max_pairs: int = 0, batch_bases: int = 0,
            min_reads: int = 1, cov=(1, 1)):
    """Containment search (readings C1-C4).  -> (mapped_reads u64[n], mapped_bases u64[n], accepted u8[n])"""
    refs, reads = _u8(refs), _u8(reads)
    ro = np.ascontiguousarray(ref_offsets, dtype=np.uint64)
    qo = np.ascontiguousarray(read_offsets, dtype=np.uint64)
    n = ro.size - 1
    mr, mb, acc = np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.uint8)
    rc = _load().or_contain(_p(refs), _p(ro), n, pattern.encode(), k, w, cutoff[0], cutoff[1], max_occ, _p(reads),
                            _p(qo), qo.size - 1, t, D, V, max_pairs, batch_bases, min_reads, cov[0], cov[1],
                            _p(mr), _p(mb), _p(acc))
    if rc:
        raise ValueError("invalid containment parameters")
    return mr, mb, acc


ALGOS = ("all", "minimizers", "spaced", "god")


def harness_seeds(seq, algo: int, k: int, w: int, pattern: str, s: int = 0) -> np.ndarray:
    """Seed hashes of one sequence (algo 0 all, 1 minimizers, 2 spaced, 3 Genome-on-Diet phase s)."""
    seq = _u8(seq)
    L = _load()
    n = L.or_harness_seeds(_p(seq), seq.size, algo, k, w, pattern.encode(), s, None, 0)
    if n < 0:
        raise ValueError("invalid harness parameters")
    out = np.zeros(n, np.uint64)
    L.or_harness_seeds(_p(seq), seq.size, algo, k, w, pattern.encode(), s, _p(out), n)
    return out


def levenshtein(a, b) -> int:
    a, b = _u8(a), _u8(b)
    return int(_load().or_levenshtein(_p(a), a.size, _p(b), b.size))


def harness_pairs(orig, mut, offsets, k: int, w: int, pattern: str):
    """Seed-comparison harness over CSR pairs (orig[i], mut[i] share offsets).
    -> (edit u64[n], matches u64[n, 4], totals u64[n, 4], god_phase u32[n]); algos in ALGOS order."""
    orig, mut = _u8(orig), _u8(mut)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = off.size - 1
    ed = np.zeros(n, np.uint64)
    m = np.zeros((n, 4), np.uint64)
    t = np.zeros((n, 4), np.uint64)
    ph = np.zeros(n, np.uint32)
    L = _load()
    for i in range(n):
        a, b = int(off[i]), int(off[i + 1])
        mi, ti, pi = np.zeros(4, np.uint64), np.zeros(4, np.uint64), np.zeros(1, np.uint32)
        d = L.or_harness_pair(_p(orig[a:b]) if b > a else ctypes.c_void_p(0), _p(mut[a:b]) if b > a else ctypes.c_void_p(0),
                              b - a, k, w, pattern.encode(), _p(mi), _p(ti), _p(pi))
        if d < 0:
            raise ValueError("invalid harness parameters")
        ed[i], m[i], t[i], ph[i] = d, mi, ti, pi[0]
    return ed, m, t, ph


def accepted_pairs(ed, m, t, E: int) -> np.ndarray:
    """the rate threshold of an edit-distance threshold E is the minimum seed matching rate of
    the pairs with edit distance <= E; a pair is accepted iff its rate >= that threshold.  Pairs
    without seeds (total 0) have no rate and are never accepted.  -> accepted count per algorithm."""
    out = np.zeros(m.shape[1], np.int64)
    for a in range(m.shape[1]):
        rated = [i for i in range(len(ed)) if t[i, a] > 0]
        cand = [i for i in rated if ed[i] <= E]
        if not cand:
            continue
        j = cand[0]
        for i in cand[1:]:  # minimum rate m/t, exact (cross-multiplication)
            if int(m[i, a]) * int(t[j, a]) < int(m[j, a]) * int(t[i, a]):
                j = i
        out[a] = sum(1 for i in rated if int(m[i, a]) * int(t[j, a]) >= int(m[j, a]) * int(t[i, a]))
    return out


class Index:
    """Oracle seed index (O7).  `cutoff` = (num, den) fraction of distinct hashes, or max_occ override."""

    def __init__(self, ref, offsets, pattern: str, k: int, w: int, cutoff=(1, 5000), max_occ: int = -1):
        self._ref = _u8(ref)
        self._off = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.pattern, self.k, self.w = pattern, k, w
        self.p, self.x = pattern_info(pattern)
        h = _load().or_build_index(_p(self._ref), _p(self._off), self._off.size - 1, pattern.encode(), k, w,
                                   cutoff[0], cutoff[1], max_occ)
        if not h:
            raise ValueError("invalid index parameters")
        self._h = ctypes.c_void_p(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_index_free(self._h)
            self._h = None

    def stats(self) -> dict:
        st = _Stats()
        _load().or_index_stats_get(self._h, ctypes.byref(st))
        return {f: int(getattr(st, f)) for f in STATS_FIELDS}

    def dump(self):
        n = _load().or_index_dump(self._h, None, None, None, 0)
        h = np.empty(n, np.uint64); p = np.empty(n, np.uint64); z = np.empty(n, np.uint8)
        _load().or_index_dump(self._h, _p(h), _p(p), _p(z), n)
        return h, p, z

    def occ(self, h: int) -> int:
        return _load().or_index_occ(self._h, h)

    def select_phase(self, read, t: int = 16):
        read = _u8(read)
        sc = np.zeros(64, np.uint64)
        a = _load().or_select_phase(self._h, _p(read), read.size, t, _p(sc))
        return a, sc[: self.p].copy()

    def seed_read(self, read, a: int, read_id: int = 0) -> np.ndarray:
        read = _u8(read)
        L = _load()
        n = L.or_seed_read(self._h, _p(read), read.size, a, read_id, None, 0)
        out = np.zeros(n, ANCHOR_DTYPE)
        L.or_seed_read(self._h, _p(read), read.size, a, read_id, _p(out), n)
        return out

    def seed_reads(self, reads, offsets, phases=None, t: int = 16):
        """SELECT mode if phases is None (returns computed phases), else GIVEN.
        -> (anchors ANCHOR_DTYPE sorted (read_id, ref_pos, read_pos, strand), anchor_offsets, phases)"""
        reads = _u8(reads)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        mode = 0 if phases is None else 1
        ph = np.zeros(n, np.uint8) if phases is None else np.ascontiguousarray(phases, dtype=np.uint8).copy()
        L = _load()
        tot = L.or_seed_reads_batch(self._h, _p(reads), _p(offsets), n, mode, _p(ph), t, None, 0, None)
        if tot < 0:
            raise ValueError("invalid seeding parameters")
        out = np.zeros(tot, ANCHOR_DTYPE)
        ao = np.zeros(n + 1, np.uint64)
        L.or_seed_reads_batch(self._h, _p(reads), _p(offsets), n, mode, _p(ph), t, _p(out), tot, _p(ao))
        return out, ao, ph

    def vote_read(self, read, a: int, D: int = 0, V: int = 3, max_pairs: int = 0, read_id: int = 0) -> np.ndarray:
        read = _u8(read)
        L = _load()
        n = L.or_vote_read(self._h, _p(read), read.size, a, read_id, D, V, max_pairs, None, 0)
        if n < 0:
            raise ValueError("invalid voting parameters")
        out = np.zeros(n, VOTE_DTYPE)
        L.or_vote_read(self._h, _p(read), read.size, a, read_id, D, V, max_pairs, _p(out), n)
        return out

    def vote_reads(self, reads, offsets, phases, D: int = 0, V: int = 3, max_pairs: int = 0):
        """Location voting of every read with its phase.
        -> (votes VOTE_DTYPE, vote_offsets u64[n+1])"""
        reads = _u8(reads)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        ph = np.ascontiguousarray(phases, dtype=np.uint8)
        L = _load()
        tot = L.or_vote_reads_batch(self._h, _p(reads), _p(offsets), n, _p(ph), D, V, max_pairs, None, 0, None)
        if tot < 0:
            raise ValueError("invalid voting parameters")
        out = np.zeros(tot, VOTE_DTYPE)
        vo = np.zeros(n + 1, np.uint64)
        L.or_vote_reads_batch(self._h, _p(reads), _p(offsets), n, _p(ph), D, V, max_pairs, _p(out), tot, _p(vo))
        return out, vo
