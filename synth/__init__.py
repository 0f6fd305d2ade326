"""Seeded synthetic inputs for the Genome-on-Diet hot path (input generation only).

This package holds NONE of the method's arithmetic: it produces ASCII genomes, ASCII reads
(concatenated, with u64 CSR offsets) and read-simulation truth.  It is the one module shared by
the CPU oracle (``oracle/``) and the CUDA path (``paper_2211_08157_b200/``); neither of those
imports the other.

Recipes: SURVEY.md §8(d) (config table) and BASELINE.json ``configs``.  The paper evaluates on
GRCh38 and GIAB HG002 reads (Supp. Table 1), which are not available
here; these synthetic stand-ins copy their shapes (read lengths, error profiles, repeat content:
"50% of the human genome consists of repeats").  DESIGN.md §3 restates the recipes.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"synth: {_LIB_PATH} missing — run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(_LIB_PATH)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    u64 = ctypes.c_uint64
    lib.synth_iid.argtypes = [u64, ctypes.c_void_p, u64]
    lib.synth_dup_segments.argtypes = [u64, ctypes.c_void_p, u64, u64, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_double, ctypes.c_double]
    lib.synth_repeats.argtypes = [u64, ctypes.c_void_p, u64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double]
    lib.synth_homopolymer_frac.argtypes = [ctypes.c_void_p, u64]
    lib.synth_homopolymer_frac.restype = ctypes.c_double
    lib.synth_reads.argtypes = [u64, ctypes.c_void_p, u64, u64, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.c_void_p, u64, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p]
    lib.synth_reads.restype = ctypes.c_int64
    lib.synth_sprinkle_n.argtypes = [u64, ctypes.c_void_p, u64, u64, ctypes.c_uint32]
    _ = u8p
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


# ----------------------------------------------------------------------------------------------
# genomes
# ----------------------------------------------------------------------------------------------
def iid_genome(length: int, seed: int) -> np.ndarray:
    out = np.empty(length, dtype=np.uint8)
    if length:
        _load().synth_iid(seed, _ptr(out), length)
    return out


def dup_genome(length: int, seed: int, dup_frac: float = 0.05, lmin: int = 1000, lmax: int = 10000,
               dmin: float = 0.01, dmax: float = 0.03) -> np.ndarray:
    """Config 2-4 reference: i.i.d. + duplicated 1-10 kbp segments at 1-3% divergence (BASELINE configs[1])."""
    g = iid_genome(length, seed)
    _load().synth_dup_segments(seed, _ptr(g), length, int(dup_frac * length), lmin, lmax, dmin, dmax)
    return g


def repeat_genome(length: int, seed: int, n_fam: int = 1000, cmin: int = 300, cmax: int = 6000,
                  dmin: float = 0.05, dmax: float = 0.20, cover: float = 0.5) -> np.ndarray:
    """Config 5 reference: i.i.d. + interspersed repeat families (BASELINE configs[4])."""
    g = iid_genome(length, seed)
    _load().synth_repeats(seed, _ptr(g), length, n_fam, cmin, cmax, dmin, dmax, cover)
    return g


def sprinkle_n(seq: np.ndarray, seed: int, n_runs: int, max_run: int) -> np.ndarray:
    seq = np.ascontiguousarray(seq).copy()
    _load().synth_sprinkle_n(seed, _ptr(seq), seq.size, n_runs, max_run)
    return seq


# ----------------------------------------------------------------------------------------------
# reads
# ----------------------------------------------------------------------------------------------
@dataclass
class ReadSet:
    seq: np.ndarray          # u8 ASCII, concatenated
    offsets: np.ndarray      # u64 [n+1]
    g: np.ndarray            # u64 origin (first reference base walked)
    span: np.ndarray         # u32 reference bases walked
    strand: np.ndarray       # u8 1 = reverse complement
    nsub: np.ndarray
    nins: np.ndarray
    ndel: np.ndarray

    @property
    def n(self) -> int:
        return int(self.offsets.size - 1)


def simulate_reads(ref: np.ndarray, n: int, seed: int, *, length: int = 0, mu: float = 0.0, sigma: float = 0.0,
                   lmin: int = 1, lmax: int = 1 << 30, start_margin: int = 200, p_sub: float = 0.0,
                   p_ins: float = 0.0, p_del: float = 0.0, homopolymer_factor: float = 0.0) -> ReadSet:
    lib = _load()
    L = ref.size
    hp_rescale = 1.0
    if homopolymer_factor > 0:
        h = lib.synth_homopolymer_frac(_ptr(ref), L)
        hp_rescale = max(0.0, (1.0 - homopolymer_factor * h) / max(1e-12, 1.0 - h))
    offsets = np.empty(n + 1, dtype=np.uint64)
    total = lib.synth_reads(seed, _ptr(ref), L, n, length, mu, sigma, lmin, lmax, start_margin,
                            p_sub, p_ins, p_del, homopolymer_factor, hp_rescale,
                            ctypes.c_void_p(0), 0, _ptr(offsets), None, None, None, None, None, None)
    seq = np.empty(total, dtype=np.uint8)
    g = np.empty(n, dtype=np.uint64)
    span = np.empty(n, dtype=np.uint32)
    strand = np.empty(n, dtype=np.uint8)
    nsub = np.empty(n, dtype=np.uint32)
    nins = np.empty(n, dtype=np.uint32)
    ndel = np.empty(n, dtype=np.uint32)
    rc = lib.synth_reads(seed, _ptr(ref), L, n, length, mu, sigma, lmin, lmax, start_margin,
                         p_sub, p_ins, p_del, homopolymer_factor, hp_rescale,
                         _ptr(seq), total, _ptr(offsets), _ptr(g), _ptr(span), _ptr(strand),
                         _ptr(nsub), _ptr(nins), _ptr(ndel))
    assert rc == total
    return ReadSet(seq, offsets, g, span, strand, nsub, nins, ndel)


# ----------------------------------------------------------------------------------------------
# BASELINE.json configs.  `scale` shrinks sizes for quick tests only.
# ----------------------------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    patterns: list
    k: int
    w: int
    cutoff: tuple = (1, 5000)    # "top 0.02%" (BASELINE.json) as a fraction num/den
    ref: np.ndarray = None
    ref_offsets: np.ndarray = None
    reads: ReadSet = None
    meta: dict = field(default_factory=dict)


CONFIG_NAMES = ("tiny", "illumina", "hifi", "ont", "human")
_REF_CACHE: dict = {}


def _lognormal_params(mean: float, sd: float):
    s2 = math.log(1.0 + (sd / mean) ** 2)
    return math.log(mean) - s2 / 2.0, math.sqrt(s2)


def reference_for(name: str, scale: float = 1.0) -> np.ndarray:
    key = (name if name in ("tiny", "human") else "ref100M", scale)
    if key in _REF_CACHE:
        return _REF_CACHE[key]
    if name == "tiny":
        ref = iid_genome(int(1_000_000 * scale), 101)
    elif name == "human":
        ref = repeat_genome(int(3_100_000_000 * scale), 501)
    else:
        L = int(100_000_000 * scale)
        ref = dup_genome(L, 201, dup_frac=0.05)
    _REF_CACHE[key] = ref
    return ref


def make_config(name: str, scale: float = 1.0, read_scale: float | None = None, read_seed_offset: int = 0) -> Config:
    """Build config `name` (BASELINE.json configs[i]); sizes × `scale` (1.0 = the real config).
    read_seed_offset shifts the read-simulation seed (independent read batches per rank)."""
    rs = scale if read_scale is None else read_scale
    so = int(read_seed_offset)
    ref = reference_for(name, scale)
    offs = np.array([0, ref.size], dtype=np.uint64)
    if name == "tiny":
        reads = simulate_reads(ref, max(1, int(10_000 * rs)), 102 + so, length=150, start_margin=200, p_sub=0.001)
        cfg = Config("tiny", ["10"], 21, 11)
    elif name == "illumina":
        reads = simulate_reads(ref, max(1, int(1_000_000 * rs)), 202 + so, length=150, start_margin=200,
                               p_sub=0.001, p_ins=0.00005, p_del=0.00005)
        cfg = Config("illumina", ["10"], 21, 11)
    elif name == "hifi":
        mu, sg = _lognormal_params(15000, 3000)
        reads = simulate_reads(ref, max(1, int(100_000 * rs)), 302 + so, mu=mu, sigma=sg, lmin=1000, lmax=100000,
                               p_sub=0.0005, p_ins=0.00025, p_del=0.00025)
        cfg = Config("hifi", ["10", "110"], 19, 19)
    elif name == "ont":
        mu, sg = _lognormal_params(10000, 8000)
        reads = simulate_reads(ref, max(1, int(50_000 * rs)), 402 + so, mu=mu, sigma=sg, lmin=200, lmax=100000,
                               p_sub=0.028, p_ins=0.021, p_del=0.021, homopolymer_factor=3.0)
        cfg = Config("ont", ["10"], 15, 10)
    elif name == "human":
        reads = simulate_reads(ref, max(1, int(10_000_000 * rs)), 502 + so, length=150, start_margin=200,
                               p_sub=0.001, p_ins=0.00005, p_del=0.00005)
        cfg = Config("human", ["10", "110", "1110", "1"], 21, 11)
    else:
        raise ValueError(f"unknown config {name!r}; expected one of {CONFIG_NAMES}")
    cfg.ref, cfg.ref_offsets, cfg.reads = ref, offs, reads
    cfg.meta = {"scale": scale, "read_scale": rs, "ref_len": int(ref.size), "n_reads": reads.n}
    return cfg


def random_acgt(rng: np.random.Generator, n: int, n_frac: float = 0.0) -> np.ndarray:
    """Small random ASCII sequence for tests (optionally with N's)."""
    s = np.frombuffer(b"ACGT", dtype=np.uint8)[rng.integers(0, 4, size=n)]
    if n_frac > 0 and n:
        s = s.copy()
        s[rng.random(n) < n_frac] = ord("N")
    return np.ascontiguousarray(s, dtype=np.uint8)


def concat(seqs) -> tuple:
    """List of u8 arrays → (concatenated u8, u64 offsets[n+1])."""
    lens = np.array([len(s) for s in seqs], dtype=np.uint64)
    offs = np.zeros(len(seqs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    cat = np.concatenate([np.asarray(s, dtype=np.uint8) for s in seqs]) if len(seqs) else np.zeros(0, np.uint8)
    return np.ascontiguousarray(cat), offs


def mutation_pairs(n: int, length: int, max_subs: int, seed: int):
    """Seed-comparison inputs: n random ACGT sequences of `length` bases and, for each, a copy
    with a uniform number in [0, max_subs] of substitutions at distinct uniform positions, each to
    one of the three other bases.  -> (orig u8, mutated u8, offsets u64[n+1], n_subs u32[n])"""
    rng = np.random.default_rng(seed)
    orig = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, size=n * length)].copy()
    mut = orig.copy()
    subs = rng.integers(0, max_subs + 1, size=n).astype(np.uint32)
    lut = {ord("A"): 0, ord("C"): 1, ord("G"): 2, ord("T"): 3}
    for i in range(n):
        pos = rng.choice(length, size=int(subs[i]), replace=False)
        for q in pos:
            c = lut[int(mut[i * length + q])]
            mut[i * length + q] = b"ACGT"[(c + int(rng.integers(1, 4))) % 4]
    offsets = (np.arange(n + 1, dtype=np.uint64) * length).astype(np.uint64)
    return orig, mut, offsets, subs
