#!/usr/bin/env python3
"""Oracle digests of the canonical dumps for every BASELINE.json config/pattern row.

SURVEY.md §8(c) O10: "Large configs are compared by streaming sha256 with chunk localisation on
mismatch."  This script imports ONLY ``oracle/`` (the CPU oracle) and ``synth/`` (the seeded input
generators); it never loads libgod.  For one (config, pattern) row it regenerates the seeded
synthetic inputs, runs the oracle over ALL of them (the whole reference, every read) and writes
``tests/golden/digests/<config>_<pattern>.json`` with the sha256 of each canonical dump, a sha256
per chunk of CHUNK records (to localise a mismatch), the index stats, record counts, and the
oracle's per-stage wall-clock times on this host (``time.perf_counter`` = steady clock).

Canonical dumps (little-endian, fixed width; the GPU side rebuilds the same bytes from its own
outputs in tests/test_gpu_digests.py):
  ref_sparsify.packed / .nmask  u64 words, 2 bits per kept base LSB-first, N stored as 0 and
                                flagged in the parallel nmask word (bit q & 31); every sequence
                                starts on a fresh word (O10); reference at phase 0 (P:286 (1)-(2))
  ref_sparsify.counts           u64 kept bases per sequence
  ref_minimizers                17-B records hash u64 | pos u64 | strand u8, position order,
                                global positions (O4-O6; P:294, P:286 (3))
  ref_minimizers.offsets        u64[n_refs + 1]
  index_dump                    17-B records hash u64 | pos u64 | strand u8, (hash, pos) order,
                                kept entries only (O7)
  phases                        u8 per read, SELECT mode, t = 16 (O8)
  anchor_counts                 u64 per read
  anchors                       16-B records read_id | ref_pos | read_pos | strand (u32 each),
                                lexicographic order (O9)
  read_sparsify.packed / .nmask / .counts   the reads under their selected phases (O3)

Usage:
  python tools/oracle_digests.py --config human --pattern 10          # one row
  python tools/oracle_digests.py --all-small                          # tiny, illumina, hifi x2, ont
Memory: the oracle keeps ~21 B per included base transiently (oracle.c or_minimizers), so the human
'1110' and '1' rows need > 62 GB and are run on the GPU box's host (see tests/golden/digests/README.md).
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

CHUNK = 1 << 22   # records per chunk digest
OUT_DIR = os.path.join(ROOT, "tests", "golden", "digests")
ROWS = [("tiny", "10"), ("illumina", "10"), ("hifi", "10"), ("hifi", "110"), ("ont", "10"),
        ("human", "10"), ("human", "110"), ("human", "1110"), ("human", "1")]
REC17 = np.dtype([("hash", "<u8"), ("pos", "<u8"), ("strand", "u1")])          # packed, 17 B
REC16 = np.dtype([("read_id", "<u4"), ("ref_pos", "<u4"), ("read_pos", "<u4"), ("strand", "<u4")])


class Digest:
    """sha256 of a record stream, plus one sha256 per CHUNK records."""

    def __init__(self):
        self.total = hashlib.sha256()
        self.chunks = []
        self._cur = hashlib.sha256()
        self._in_cur = 0
        self.n = 0

    def update(self, recs: np.ndarray):
        recs = np.ascontiguousarray(recs)
        i = 0
        while i < recs.size:
            take = min(CHUNK - self._in_cur, recs.size - i)
            b = recs[i:i + take].tobytes()
            self.total.update(b)
            self._cur.update(b)
            self._in_cur += take
            i += take
            if self._in_cur == CHUNK:
                self.chunks.append(self._cur.hexdigest())
                self._cur, self._in_cur = hashlib.sha256(), 0
        self.n += recs.size
        return self

    def result(self) -> dict:
        chunks = list(self.chunks)
        if self._in_cur:
            chunks.append(self._cur.hexdigest())
        return {"sha256": self.total.hexdigest(), "n": int(self.n), "chunk_records": CHUNK, "chunks": chunks}


def digest_of(a: np.ndarray) -> dict:
    return Digest().update(a).result()


def pack_codes(codes: np.ndarray, counts: np.ndarray):
    """O10 packing of concatenated oracle codes (0..3, 4 = N) with per-sequence counts:
    -> (packed u64, nmask u64), every sequence starting on a fresh 32-base word."""
    counts = counts.astype(np.int64)
    n = counts.size
    woff = np.zeros(n + 1, np.int64)
    np.cumsum((counts + 31) // 32, out=woff[1:])
    coff = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=coff[1:])
    packed = np.zeros(int(woff[-1]), np.uint64)
    nmask = np.zeros(int(woff[-1]), np.uint64)
    sh2 = 2 * np.arange(32, dtype=np.uint64)
    sh1 = np.arange(32, dtype=np.uint64)

    def put(pad: np.ndarray, w0: int):
        pad = pad.reshape(-1, 32)
        isn = pad == 4
        val = np.where(isn, 0, pad).astype(np.uint64)
        packed[w0:w0 + pad.shape[0]] = np.bitwise_or.reduce(val << sh2, axis=1)
        nmask[w0:w0 + pad.shape[0]] = np.bitwise_or.reduce(isn.astype(np.uint64) << sh1, axis=1)

    BIG = 1 << 24   # bases per piece (a multiple of 32)
    i = 0
    while i < n:
        if counts[i] > BIG:   # one long sequence: word-aligned pieces
            c = codes[coff[i]:coff[i + 1]]
            for a in range(0, c.size, BIG):
                piece = c[a:a + BIG]
                pad = np.zeros(-(-piece.size // 32) * 32, np.uint8)
                pad[:piece.size] = piece
                put(pad, int(woff[i]) + a // 32)
            i += 1
            continue
        j, tot = i, 0
        while j < n and counts[j] <= BIG and tot + counts[j] <= BIG:
            tot += int(counts[j])
            j += 1
        c = codes[coff[i]:coff[j]]
        pad = np.zeros(int(woff[j] - woff[i]) * 32, np.uint8)
        local = np.arange(c.size, dtype=np.int64) - np.repeat(coff[i:j] - coff[i], counts[i:j])
        pad[np.repeat((woff[i:j] - woff[i]) * 32, counts[i:j]) + local] = c
        put(pad, int(woff[i]))
        i = j
    return packed, nmask


def sparsify_batch(seq: np.ndarray, offsets: np.ndarray, pattern: str, phases=None):
    """or_sparsify (O3) of every CSR sequence at its phase -> (codes concatenated, counts u64)."""
    L = oracle._load()
    P = oracle.parse_pattern(pattern)
    n = offsets.size - 1
    off = offsets.astype(np.int64)
    base = seq.ctypes.data
    counts = np.zeros(n, np.uint64)
    fn = L.or_sparsify
    for i in range(n):
        s = 0 if phases is None else int(phases[i])
        counts[i] = fn(ctypes.c_void_p(base + int(off[i])), int(off[i + 1] - off[i]), ctypes.byref(P), s, None, None)
    codes = np.zeros(int(counts.sum()), np.uint8)
    cb = codes.ctypes.data
    q = 0
    for i in range(n):
        s = 0 if phases is None else int(phases[i])
        fn(ctypes.c_void_p(base + int(off[i])), int(off[i + 1] - off[i]), ctypes.byref(P), s,
           ctypes.c_void_p(cb + q), None)
        q += int(counts[i])
    return codes, counts


def seed_batches(ox, reads: np.ndarray, offsets: np.ndarray, mode: int, phases: np.ndarray, t: int = 16,
                 batch: int = 1_000_000):
    """or_seed_reads_batch (O8 + O9) over batches of reads (reads are independent; read ids rebased).
    -> (anchors REC16 in canonical order, anchor counts u64[n], phases u8[n])."""
    L = oracle._load()
    n = offsets.size - 1
    outs, counts = [], np.zeros(n, np.uint64)
    for a in range(0, n, batch):
        b = min(n, a + batch)
        off = (offsets[a:b + 1] - offsets[a]).astype(np.uint64)
        sub = reads[int(offsets[a]):int(offsets[b])]
        ph = phases[a:b] if mode == 1 else np.zeros(b - a, np.uint8)
        ph = np.ascontiguousarray(ph)
        cap = max(1024, sub.size // 2)
        while True:
            out = np.zeros(cap, oracle.ANCHOR_DTYPE)
            ao = np.zeros(b - a + 1, np.uint64)
            tot = L.or_seed_reads_batch(ox._h, oracle._p(sub), oracle._p(off), b - a, mode, oracle._p(ph), t,
                                        oracle._p(out), cap, oracle._p(ao))
            if tot >= 0:
                break
            cap *= 4
        if mode == 0:
            phases[a:b] = ph
        out = out[:tot]
        r = np.zeros(tot, REC16)
        r["read_id"] = out["read_id"] + a
        r["ref_pos"], r["read_pos"], r["strand"] = out["ref_pos"], out["read_pos"], out["strand"]
        outs.append(r)
        counts[a:b] = np.diff(ao)
    return (np.concatenate(outs) if outs else np.zeros(0, REC16)), counts, phases


def host_info() -> dict:
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "cores_used": 1, "node": platform.node(),
            "oracle": "oracle/liboracle.so (gcc -O2, single thread)"}


def run_row(config: str, pattern: str, scale: float = 1.0, given_check: bool = True, out_dir: str = OUT_DIR) -> dict:
    t0 = time.perf_counter()
    cfg = synth.make_config(config, scale=scale)
    t_gen = time.perf_counter() - t0
    k, w = cfg.k, cfg.w
    ref, roff, reads = cfg.ref, cfg.ref_offsets, cfg.reads
    res = {"config": config, "pattern": pattern, "k": k, "w": w, "cutoff": list(cfg.cutoff), "t": 16,
           "scale": scale, "ref_bp": int(ref.size), "n_refs": int(roff.size - 1), "n_reads": reads.n,
           "read_bp": int(reads.seq.size), "inputs": {
               "ref_sha256": hashlib.sha256(ref.tobytes()).hexdigest(),
               "reads_sha256": hashlib.sha256(reads.seq.tobytes()).hexdigest(),
               "read_offsets_sha256": hashlib.sha256(reads.offsets.astype("<u8").tobytes()).hexdigest()},
           "digests": {}, "timing_s": {"generate_inputs": round(t_gen, 3)}, "host": host_info(),
           "command": f"python tools/oracle_digests.py --config {config} --pattern {pattern}"
                      + (f" --scale {scale}" if scale != 1.0 else "")}
    D, T = res["digests"], res["timing_s"]

    def log(msg):
        print(f"[digests {config} '{pattern}'] {msg} ({time.perf_counter() - t0:.1f}s)", file=sys.stderr, flush=True)

    # stage 1: pack + sparsify the reference (phase 0)
    t = time.perf_counter()
    codes, counts = sparsify_batch(ref, roff, pattern)
    T["sparsify_ref"] = round(time.perf_counter() - t, 3)
    packed, nmask = pack_codes(codes, counts)
    del codes
    D["ref_sparsify.packed"] = digest_of(packed)
    D["ref_sparsify.nmask"] = digest_of(nmask)
    D["ref_sparsify.counts"] = digest_of(counts.astype("<u8"))
    del packed, nmask
    log("ref sparsify")

    # stage 2: minimizers of the reference (global positions, position order)
    t = time.perf_counter()
    mz, mo = oracle.minimizers_batch(ref, roff, pattern, k, w, global_pos=True)
    T["extract_ref"] = round(time.perf_counter() - t, 3)
    r17 = np.zeros(mz.size, REC17)
    r17["hash"], r17["pos"], r17["strand"] = mz["hash"], mz["pos"], mz["strand"]
    del mz
    D["ref_minimizers"] = digest_of(r17)
    del r17
    D["ref_minimizers.offsets"] = digest_of(mo.astype("<u8"))
    log("ref minimizers")

    # stage 3: index (collect -> sort -> count -> cutoff -> table)
    t = time.perf_counter()
    ox = oracle.Index(ref, roff, pattern, k, w, cutoff=cfg.cutoff)
    T["index_build"] = round(time.perf_counter() - t, 3)
    res["index_stats"] = ox.stats()
    h, p, z = ox.dump()
    r17 = np.zeros(h.size, REC17)
    r17["hash"], r17["pos"], r17["strand"] = h, p, z
    del h, p, z
    D["index_dump"] = digest_of(r17)
    del r17
    log(f"index {res['index_stats']}")

    # stage 4: SELECT-mode phase selection + seeding of every read
    t = time.perf_counter()
    phases = np.zeros(reads.n, np.uint8)
    an, acnt, phases = seed_batches(ox, reads.seq, reads.offsets, 0, phases)
    T["select_and_seed"] = round(time.perf_counter() - t, 3)
    res["n_anchors"] = int(an.size)
    D["phases"] = digest_of(phases)
    D["anchor_counts"] = digest_of(acnt.astype("<u8"))
    D["anchors"] = digest_of(an)
    res["phase_histogram"] = np.bincount(phases, minlength=len(pattern)).tolist()
    log(f"seeding: {an.size} anchors")
    if given_check:
        # seeding alone (GIVEN mode with the selected phases): splits the stage time, and the anchors
        # must be the SELECT-mode anchors (O8 then O9)
        t = time.perf_counter()
        an2, acnt2, _ = seed_batches(ox, reads.seq, reads.offsets, 1, phases.copy())
        T["seed_given"] = round(time.perf_counter() - t, 3)
        T["phase_select"] = round(max(0.0, T["select_and_seed"] - T["seed_given"]), 3)
        assert np.array_equal(an2, an) and np.array_equal(acnt2, acnt), "GIVEN-mode anchors differ from SELECT"
        del an2
        log("given-mode check")
    del an
    # stage 1 for the reads: sparsified reads under their selected phases
    t = time.perf_counter()
    codes, counts = sparsify_batch(reads.seq, reads.offsets, pattern, phases)
    T["sparsify_reads"] = round(time.perf_counter() - t, 3)
    packed, nmask = pack_codes(codes, counts)
    del codes
    D["read_sparsify.packed"] = digest_of(packed)
    D["read_sparsify.nmask"] = digest_of(nmask)
    D["read_sparsify.counts"] = digest_of(counts.astype("<u8"))
    del packed, nmask, ox
    T["total"] = round(time.perf_counter() - t0, 3)
    log("done")
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        suffix = "" if scale == 1.0 else f"_x{scale:g}"
        path = os.path.join(out_dir, f"{config}_{pattern}{suffix}.json")
        with open(path, "w") as f:
            json.dump(res, f, indent=1)
            f.write("\n")
        log(f"wrote {path}")
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config")
    ap.add_argument("--pattern")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--all-small", action="store_true", help="every non-human row")
    ap.add_argument("--no-given-check", action="store_true")
    ap.add_argument("--out-dir", default=OUT_DIR)
    a = ap.parse_args()
    rows = [r for r in ROWS if r[0] != "human"] if a.all_small else [(a.config, a.pattern)]
    for c, p in rows:
        run_row(c, p, a.scale, not a.no_given_check, a.out_dir)


if __name__ == "__main__":
    main()
