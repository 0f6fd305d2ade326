"""B200-native Genome-on-Diet hot path (arXiv 2211.08157): sparsify -> minimizers -> index -> seeds.

Thin Python binding over libgod.so (include/god.h).  Argument marshalling only: every step of the
path runs in the CUDA kernels behind the C ABI; there is no CPU or PyTorch fallback, and the
functions raise if the library is missing.  Names follow the C ABI.

Arrays may be CUDA torch tensors (device path, asynchronous on the current torch stream until a
size is needed) or host numpy arrays / CPU tensors (staged by the library; outputs come back as
numpy).  PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import GodError, PHASE_GIVEN, PHASE_SELECT  # noqa: F401

try:
    import torch
except Exception:  # pragma: no cover - torch is in the image
    torch = None

ANCHOR_DTYPE = np.dtype([("ref_pos", "<u4"), ("read_pos", "<u4"), ("read_id", "<u4"), ("strand", "<u4")])
# god_anchor_compact: 8 bytes, read id implied by the anchor offsets, strand in bit 31
ANCHOR_COMPACT_DTYPE = np.dtype([("ref_pos", "<u4"), ("read_pos_strand", "<u4")])
# god_vote (include/god.h): 40 bytes; the device path returns it as a (n, 10) u32 tensor (diag = words 2-3)
VOTE_DTYPE = np.dtype([("read_id", "<u4"), ("strand", "<u4"), ("diag", "<i8"), ("votes", "<u4"), ("rescued", "<u4"),
                       ("ref_lo", "<u4"), ("ref_hi", "<u4"), ("read_lo", "<u4"), ("read_hi", "<u4")])


# ---------------------------------------------------------------------------------------- helpers
def _is_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _ptr(x):
    if x is None:
        return None
    if torch is not None and isinstance(x, torch.Tensor):
        return ctypes.c_void_p(x.data_ptr()) if x.numel() else ctypes.c_void_p(0)
    return ctypes.c_void_p(x.ctypes.data) if x.size else ctypes.c_void_p(0)


def _host(x, dtype):
    if torch is not None and isinstance(x, torch.Tensor):
        x = x.numpy()
    return np.ascontiguousarray(x, dtype=dtype)


def _prep(x, dtype):
    """CUDA tensors pass through (must be contiguous, right dtype); everything else -> numpy."""
    if x is None:
        return None
    if _is_cuda(x):
        tdt = {np.uint8: torch.uint8, np.uint64: torch.uint64, np.uint32: torch.uint32}[dtype]
        if x.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {x.dtype}")
        return x.contiguous()
    return _host(x, dtype)


def _empty(n, dtype, like_cuda: bool, device=None):
    if like_cuda:
        tdt = {np.uint8: torch.uint8, np.uint64: torch.uint64, np.uint32: torch.uint32}[dtype]
        return torch.empty(int(n), dtype=tdt, device=device)
    return np.empty(int(n), dtype=dtype)


def _stream(device_path: bool):
    if device_path and torch is not None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(0)


def _params(pattern: str, k: int, w: int) -> _lib.GodParams:
    return _lib.GodParams(pattern.encode(), int(k), int(w))


def version() -> str:
    return _lib.load().god_version().decode()


# ---------------------------------------------------------------------------------------- stage 1
def god_sparsify(seq, offsets, pattern: str, k: int = 1, w: int = 1, phases=None):
    """-> (packed u64, nmask u64, out_offsets u64[n+1], counts u64[n])  (god.h stage 1)."""
    L = _lib.load()
    dev = _is_cuda(seq)
    seq, offsets, phases = _prep(seq, np.uint8), _prep(offsets, np.uint64), _prep(phases, np.uint8)
    n = int(offsets.shape[0]) - 1
    dv = seq.device if dev else None
    prm = _params(pattern, k, w)
    oo = _empty(n + 1, np.uint64, dev, dv)
    cnt = _empty(n, np.uint64, dev, dv)
    need = ctypes.c_uint64(0)
    st = _stream(dev)
    rc = L.god_sparsify(ctypes.byref(prm), _ptr(seq), _ptr(offsets), n, _ptr(phases), None, None, _ptr(oo),
                        _ptr(cnt), 0, ctypes.byref(need), st)
    _lib.check(rc, allow=(_lib.GOD_ETRUNC,))
    packed = _empty(max(1, need.value), np.uint64, dev, dv)
    nmask = _empty(max(1, need.value), np.uint64, dev, dv)
    rc = L.god_sparsify(ctypes.byref(prm), _ptr(seq), _ptr(offsets), n, _ptr(phases), _ptr(packed), _ptr(nmask),
                        _ptr(oo), _ptr(cnt), need.value, ctypes.byref(need), st)
    _lib.check(rc)
    return packed[: need.value], nmask[: need.value], oo, cnt


# ---------------------------------------------------------------------------------------- stage 2
def god_minimizers(seq, offsets, pattern: str, k: int, w: int, phases=None, global_pos: bool = False,
                   cap: int | None = None):
    """-> (hash u64, pos u32, strand u8, out_offsets u64[n+1])  (god.h stage 2), position order."""
    L = _lib.load()
    dev = _is_cuda(seq)
    seq, offsets, phases = _prep(seq, np.uint8), _prep(offsets, np.uint64), _prep(phases, np.uint8)
    n = int(offsets.shape[0]) - 1
    dv = seq.device if dev else None
    prm = _params(pattern, k, w)
    total = int(seq.shape[0])
    if cap is None:
        cap = total * 2 // (w + 1) + total // 8 + 1024
    oo = _empty(n + 1, np.uint64, dev, dv)
    need = ctypes.c_uint64(0)
    st = _stream(dev)
    for _ in range(2):
        h = _empty(max(1, cap), np.uint64, dev, dv)
        p = _empty(max(1, cap), np.uint32, dev, dv)
        z = _empty(max(1, cap), np.uint8, dev, dv)
        rc = L.god_minimizers(ctypes.byref(prm), _ptr(seq), _ptr(offsets), n, _ptr(phases), int(global_pos),
                              _ptr(h), _ptr(p), _ptr(z), _ptr(oo), cap, ctypes.byref(need), st)
        if rc == _lib.GOD_ETRUNC:
            cap = need.value
            continue
        _lib.check(rc)
        m = need.value
        return h[:m], p[:m], z[:m], oo
    raise GodError(_lib.GOD_ETRUNC, "minimizer capacity retry failed")


# ---------------------------------------------------------------------------------------- stage 3
class GodIndex:
    """Library-owned seed index (god.h stage 3).  Free with .free() or by garbage collection."""

    def __init__(self, handle, pattern, k, w):
        self._h = handle
        self.pattern, self.k, self.w = pattern, k, w

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        st = _lib.GodIndexStats()
        _lib.check(_lib.load().god_index_get_stats(self._h, ctypes.byref(st)))
        return {f: int(getattr(st, f)) for f, _ in _lib.GodIndexStats._fields_}

    def dump(self, device: bool = False):
        """Kept entries in (hash, pos) order -> (hash u64, pos u32, strand u8)."""
        n = self.stats()["kept_entries"]
        dv = torch.device("cuda") if device else None
        h = _empty(max(1, n), np.uint64, device, dv)
        p = _empty(max(1, n), np.uint32, device, dv)
        z = _empty(max(1, n), np.uint8, device, dv)
        need = ctypes.c_uint64(0)
        _lib.check(_lib.load().god_index_dump(self._h, _ptr(h), _ptr(p), _ptr(z), n, ctypes.byref(need),
                                              _stream(device)))
        return h[:n], p[:n], z[:n]

    def count(self, hashes):
        dev = _is_cuda(hashes)
        hashes = _prep(hashes, np.uint64)
        n = int(hashes.shape[0])
        out = _empty(max(1, n), np.uint32, dev, hashes.device if dev else None)
        _lib.check(_lib.load().god_index_count(self._h, _ptr(hashes), n, _ptr(out), _stream(dev)))
        return out[:n]

    def free(self):
        if self._h:
            _lib.load().god_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def god_build_index(ref, ref_offsets, pattern: str, k: int, w: int, cutoff=(1, 5000), max_occ=None) -> GodIndex:
    """Build the seed index.  cutoff = (num, den): drop the top num/den distinct hashes by count
    (BASELINE "top 0.02%" = (1, 5000)); max_occ = int: keep iff count <= max_occ instead."""
    L = _lib.load()
    dev = _is_cuda(ref)
    ref, ref_offsets = _prep(ref, np.uint8), _prep(ref_offsets, np.uint64)
    n = int(ref_offsets.shape[0]) - 1
    prm = _params(pattern, k, w)
    cut = _lib.GodCutoff(1, 0, 1, int(max_occ)) if max_occ is not None else _lib.GodCutoff(0, cutoff[0], cutoff[1], 0)
    h = ctypes.c_void_p(0)
    _lib.check(L.god_build_index(ctypes.byref(prm), _ptr(ref), _ptr(ref_offsets), n, ctypes.byref(cut),
                                 ctypes.byref(h), _stream(dev)))
    return GodIndex(h, pattern, k, w)


# ---------------------------------------------------------------------------------------- stage 4
def god_seed_reads(index: GodIndex, reads, read_offsets, phases=None, t: int = 16, cap: int | None = None,
                   out=None, host_out: bool = False, compact: bool = False):
    """SELECT mode if phases is None (phase per read computed), else GIVEN.
    -> (anchors, anchor_offsets u64[n+1], phases u8[n]).  Device path: anchors is a CUDA u32 tensor
    of shape (n_anchors, 4) = (ref_pos, read_pos, read_id, strand); host path: structured numpy.
    out = (anchors, anchor_offsets, phases) preallocated (device path; anchors (cap, 4) u32) avoids
    per-call allocations in a serving loop.  host_out=True with CUDA reads returns host (numpy) outputs:
    the library then streams the results of read batches back while later batches are seeded.
    compact=True: 8-byte god_anchor_compact anchors ((n, 2) u32 tensor / ANCHOR_COMPACT_DTYPE;
    expand_compact() restores the full form)."""
    L = _lib.load()
    dev = _is_cuda(reads) and not host_out
    reads, read_offsets = _prep(reads, np.uint8), _prep(read_offsets, np.uint64)
    n = int(read_offsets.shape[0]) - 1
    dv = reads.device if dev else None
    mode = _lib.PHASE_SELECT if phases is None else _lib.PHASE_GIVEN
    if out is not None:
        an_out, ao, ph = out
        if phases is not None:
            ph[:n].copy_(_prep(phases, np.uint8))
        cap = int(an_out.shape[0])
    else:
        an_out = None
        ph = _empty(max(1, n), np.uint8, dev, dv) if phases is None else _prep(phases, np.uint8).clone() if dev \
            else _prep(phases, np.uint8).copy()
        ao = _empty(n + 1, np.uint64, dev, dv)
    if cap is None:
        cap = int(reads.shape[0]) // 4 + 1024
    need = ctypes.c_uint64(0)
    st = _stream(dev)
    for _ in range(2):
        if an_out is not None and cap <= int(an_out.shape[0]):
            an = an_out
        else:
            an = torch.empty((max(1, cap), 2 if compact else 4), dtype=torch.uint32, device=dv) if dev else \
                np.zeros(max(1, cap), ANCHOR_COMPACT_DTYPE if compact else ANCHOR_DTYPE)
        fn = L.god_seed_reads_compact if compact else L.god_seed_reads
        rc = fn(index.handle, _ptr(reads), _ptr(read_offsets), n, mode, _ptr(ph), int(t), _ptr(an),
                              _ptr(ao), cap, ctypes.byref(need), st)
        if rc == _lib.GOD_ETRUNC:
            cap = need.value
            mode = _lib.PHASE_GIVEN  # phases were written by the first call
            continue
        _lib.check(rc)
        return an[: need.value], ao, ph[:n]
    raise GodError(_lib.GOD_ETRUNC, "anchor capacity retry failed")


def god_build_index_and_seed(ref, ref_offsets, reads, read_offsets, pattern: str, k: int, w: int, cutoff=(1, 5000),
                             max_occ=None, phases=None, t: int = 16, cap: int | None = None, compact: bool = False):
    """god_build_index + god_seed_reads in one call (include/god.h): with host inputs the first read
    batches go up right behind the reference, while the index is sorted.  All inputs on the host, or all
    on the device; outputs live where the inputs do.  -> (GodIndex, anchors, anchor_offsets, phases)."""
    L = _lib.load()
    dev = _is_cuda(ref)
    if dev != _is_cuda(reads):
        raise TypeError("ref and reads must both be CUDA tensors or both host arrays")
    ref, ref_offsets = _prep(ref, np.uint8), _prep(ref_offsets, np.uint64)
    reads, read_offsets = _prep(reads, np.uint8), _prep(read_offsets, np.uint64)
    n_refs, n = int(ref_offsets.shape[0]) - 1, int(read_offsets.shape[0]) - 1
    dv = reads.device if dev else None
    prm = _params(pattern, k, w)
    cut = _lib.GodCutoff(1, 0, 1, int(max_occ)) if max_occ is not None else _lib.GodCutoff(0, cutoff[0], cutoff[1], 0)
    mode = _lib.PHASE_SELECT if phases is None else _lib.PHASE_GIVEN
    ph = _empty(max(1, n), np.uint8, dev, dv) if phases is None else _prep(phases, np.uint8).clone() if dev \
        else _prep(phases, np.uint8).copy()
    ao = _empty(n + 1, np.uint64, dev, dv)
    if cap is None:
        cap = int(reads.shape[0]) // 4 + 1024
    an = torch.empty((max(1, cap), 2 if compact else 4), dtype=torch.uint32, device=dv) if dev else \
        np.zeros(max(1, cap), ANCHOR_COMPACT_DTYPE if compact else ANCHOR_DTYPE)
    need = ctypes.c_uint64(0)
    h = ctypes.c_void_p(0)
    rc = L.god_build_index_and_seed(ctypes.byref(prm), _ptr(ref), _ptr(ref_offsets), n_refs, ctypes.byref(cut),
                                    ctypes.byref(h), _ptr(reads), _ptr(read_offsets), n, mode, _ptr(ph), int(t),
                                    1 if compact else 0, _ptr(an), _ptr(ao), cap, ctypes.byref(need), _stream(dev))
    index = GodIndex(h, pattern, k, w) if h.value else None
    if rc == _lib.GOD_ETRUNC and index is not None:  # the index stands; seed again with the capacity asked for
        an, ao, ph = god_seed_reads(index, reads, read_offsets, phases=ph[:n], t=t, cap=need.value, compact=compact)
        return index, an, ao, ph
    _lib.check(rc)
    return index, an[: need.value], ao, ph[:n]


def expand_compact(anchors, anchor_offsets) -> np.ndarray:
    """god_anchor_compact (host or device) -> ANCHOR_DTYPE on the host (argument marshalling for
    callers and tests: the read id is the anchor's segment in anchor_offsets)."""
    if torch is not None and isinstance(anchors, torch.Tensor):
        a = anchors.cpu().numpy().view(ANCHOR_COMPACT_DTYPE).reshape(-1)
    else:
        a = np.asarray(anchors).view(ANCHOR_COMPACT_DTYPE).reshape(-1)
    ao = anchor_offsets.cpu().numpy() if torch is not None and isinstance(anchor_offsets, torch.Tensor) \
        else np.asarray(anchor_offsets)
    out = np.zeros(a.size, ANCHOR_DTYPE)
    out["ref_pos"] = a["ref_pos"]
    out["read_pos"] = a["read_pos_strand"] & 0x7FFFFFFF
    out["strand"] = a["read_pos_strand"] >> 31
    out["read_id"] = np.repeat(np.arange(ao.size - 1, dtype=np.uint32), np.diff(ao.astype(np.int64)))
    return out


# ---------------------------------------------------------------------------------------- voting
def _check_anchor_records(anchors, anchor_offsets, n: int):
    """god_vote_reads reads 16-B god_anchor records (include/god.h): reject the 8-B compact form
    (expand_compact() converts it) and a buffer shorter than anchor_offsets[n]."""
    if torch is not None and isinstance(anchors, torch.Tensor):
        rec = anchors.element_size() * (int(anchors.shape[-1]) if anchors.dim() == 2 else 1)
        nrec = int(anchors.shape[0]) if anchors.dim() >= 1 else 0
    else:
        a = np.asarray(anchors)
        rec = a.dtype.itemsize * (int(a.shape[-1]) if a.ndim == 2 else 1)
        nrec = int(a.shape[0]) if a.ndim >= 1 else 0
        if a.ndim == 1 and a.dtype.itemsize != 16:
            rec, nrec = 16, a.size * a.dtype.itemsize // 16
    if rec != 16:
        raise GodError(_lib.GOD_EINVAL, f"anchors must be 16-B god_anchor records (got {rec}-B rows; "
                                        "compact anchors need expand_compact())")
    ao = anchor_offsets
    need = int(ao[n].item()) if torch is not None and isinstance(ao, torch.Tensor) else int(np.asarray(ao)[n])
    if nrec < need:
        raise GodError(_lib.GOD_EINVAL, f"anchors hold {nrec} records, anchor_offsets[{n}] = {need}")


def god_vote_reads(index: GodIndex, reads, read_offsets, phases, anchors, anchor_offsets, D: int = 0, V: int = 3,
                   max_pairs: int = 0, cap: int | None = None):
    """Location voting (rescue P:398) on the anchors of god_seed_reads (same reads and
    phases).  D = 0: the read length.  -> (votes, vote_offsets u64[n+1]).  Device path: votes is a
    (n_votes, 10) u32 CUDA tensor in god_vote layout (votes_numpy() converts); host path: VOTE_DTYPE."""
    L = _lib.load()
    dev = _is_cuda(reads)
    reads, read_offsets = _prep(reads, np.uint8), _prep(read_offsets, np.uint64)
    phases, anchor_offsets = _prep(phases, np.uint8), _prep(anchor_offsets, np.uint64)
    if dev:
        anchors = anchors.contiguous()
    else:
        anchors = np.ascontiguousarray(anchors)
    n = int(read_offsets.shape[0]) - 1
    _check_anchor_records(anchors, anchor_offsets, n)
    dv = reads.device if dev else None
    vo = _empty(n + 1, np.uint64, dev, dv)
    vp = _lib.GodVoteParams(int(D), int(V), int(max_pairs))
    if cap is None:
        cap = n * (max_pairs if max_pairs else 4) + 16
    need = ctypes.c_uint64(0)
    st = _stream(dev)
    for _ in range(2):
        out = torch.empty((max(1, cap), 10), dtype=torch.uint32, device=dv) if dev else \
            np.zeros(max(1, cap), VOTE_DTYPE)
        rc = L.god_vote_reads(index.handle, _ptr(reads), _ptr(read_offsets), n, _ptr(phases), _ptr(anchors),
                              _ptr(anchor_offsets), ctypes.byref(vp), _ptr(out), _ptr(vo), cap, ctypes.byref(need), st)
        if rc == _lib.GOD_ETRUNC:
            cap = need.value
            continue
        _lib.check(rc)
        return out[: need.value], vo
    raise GodError(_lib.GOD_ETRUNC, "vote capacity retry failed")


def god_contain(refs, ref_offsets, reads, read_offsets, pattern: str, k: int, w: int, cutoff=(1, 5000),
                max_occ=None, t: int = 16, D: int = 0, V: int = 3, max_pairs: int = 0, batch_bases: int = 0,
                min_reads: int = 1, cov=(1, 1)):
    """Desk-scale containment search: per reference sequence the reads that
    receive a voted location in it, their total length, and the accept decision (mapped reads >=
    min_reads and coverage >= cov[0] / cov[1]).  -> (mapped_reads u64[n], mapped_bases u64[n],
    accepted u8[n]) on the device if `reads` is a CUDA tensor, else numpy."""
    L = _lib.load()
    dev = _is_cuda(reads)
    refs, ref_offsets = _prep(refs, np.uint8), _prep(ref_offsets, np.uint64)
    reads, read_offsets = _prep(reads, np.uint8), _prep(read_offsets, np.uint64)
    n = int(ref_offsets.shape[0]) - 1
    dv = reads.device if dev else None
    mr, mb, acc = _empty(max(1, n), np.uint64, dev, dv), _empty(max(1, n), np.uint64, dev, dv), \
        _empty(max(1, n), np.uint8, dev, dv)
    prm = _params(pattern, k, w)
    cut = _lib.GodCutoff(1, 0, 1, int(max_occ)) if max_occ is not None else _lib.GodCutoff(0, cutoff[0], cutoff[1], 0)
    vp = _lib.GodVoteParams(int(D), int(V), int(max_pairs))
    cp = _lib.GodContainParams(int(batch_bases), int(min_reads), int(cov[0]), int(cov[1]))
    _lib.check(L.god_contain(ctypes.byref(prm), _ptr(refs), _ptr(ref_offsets), n, ctypes.byref(cut), _ptr(reads),
                             _ptr(read_offsets), int(read_offsets.shape[0]) - 1, int(t), ctypes.byref(vp),
                             ctypes.byref(cp), _ptr(mr), _ptr(mb), _ptr(acc), _stream(dev)))
    return mr[:n], mb[:n], acc[:n]


def god_seed_harness(orig, mut, offsets, pattern: str, k: int, w: int):
    """Seed-comparison harness: per pair the edit distance and, for the four extractors
    (all k-mers, minimizers, spaced seeds, Genome-on-Diet), the seed matching rate as
    (matches, totals).  -> (edit u64[n], matches u64[n, 4], totals u64[n, 4], god_phase u32[n])"""
    L = _lib.load()
    dev = _is_cuda(orig)
    orig, mut, offsets = _prep(orig, np.uint8), _prep(mut, np.uint8), _prep(offsets, np.uint64)
    n = int(offsets.shape[0]) - 1
    dv = orig.device if dev else None
    ed = _empty(max(1, n), np.uint64, dev, dv)
    mm = _empty(max(1, 4 * n), np.uint64, dev, dv)
    tt = _empty(max(1, 4 * n), np.uint64, dev, dv)
    ph = _empty(max(1, n), np.uint32, dev, dv)
    prm = _params(pattern, k, w)
    _lib.check(L.god_seed_harness(ctypes.byref(prm), _ptr(orig), _ptr(mut), _ptr(offsets), n, _ptr(ed), _ptr(mm),
                                  _ptr(tt), _ptr(ph), _stream(dev)))
    return ed[:n], mm[:4 * n].reshape(n, 4), tt[:4 * n].reshape(n, 4), ph[:n]


def god_harness_accepted(edit, matches, totals, thresholds):
    """Accepted sequence pairs per edit-distance threshold and extractor.
    -> u64[len(thresholds), 4]"""
    L = _lib.load()
    dev = _is_cuda(edit)
    edit, thresholds = _prep(edit, np.uint64), _prep(thresholds, np.uint64)
    matches = matches.contiguous() if dev else np.ascontiguousarray(matches, dtype=np.uint64)
    totals = totals.contiguous() if dev else np.ascontiguousarray(totals, dtype=np.uint64)
    n, ne = int(edit.shape[0]), int(thresholds.shape[0])
    out = _empty(max(1, 4 * ne), np.uint64, dev, edit.device if dev else None)
    _lib.check(L.god_harness_accepted(_ptr(edit), _ptr(matches), _ptr(totals), n, _ptr(thresholds), ne, _ptr(out),
                                      _stream(dev)))
    return out[:4 * ne].reshape(ne, 4)


def votes_numpy(votes) -> np.ndarray:
    """(n, 10) u32 device/host array in god_vote layout -> VOTE_DTYPE numpy records."""
    if _is_cuda(votes):
        votes = votes.cpu().numpy()
    a = np.ascontiguousarray(votes)
    return a.view(VOTE_DTYPE).reshape(-1) if a.dtype != VOTE_DTYPE else a


# ---------------------------------------------------------------------------------------- tracing
def profile_enable(on: bool = True):
    _lib.load().god_profile_enable(int(on))


def profile_reset():
    _lib.load().god_profile_reset()


def profile_query() -> dict:
    """{kernel name: (total ms, launches)} accumulated since the last reset (synchronizes)."""
    L = _lib.load()
    cap = 128
    buf = ctypes.create_string_buffer(cap * 64)
    ms = (ctypes.c_double * cap)()
    ln = (ctypes.c_uint64 * cap)()
    n = L.god_profile_query(buf, len(buf), ms, ln, cap)
    names = buf.raw.split(b"\0")[:n]
    return {nm.decode(): (ms[i], int(ln[i])) for i, nm in enumerate(names)}


def profile_units(name: str) -> int:
    """Work units recorded for the launches named `name` since the last reset (extraction launches:
    k-mer start positions processed)."""
    return int(_lib.load().god_profile_units(name.encode()))


def launch_count() -> int:
    return int(_lib.load().god_launch_count())


__all__ = ["god_sparsify", "god_minimizers", "god_build_index", "god_seed_reads", "god_vote_reads", "votes_numpy",
           "god_contain", "god_seed_harness",
           "god_harness_accepted",
           "expand_compact", "god_build_index_and_seed", "GodIndex", "GodError", "ANCHOR_DTYPE", "ANCHOR_COMPACT_DTYPE", "VOTE_DTYPE", "version"]
