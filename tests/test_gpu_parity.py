"""GPU parity (-m gpu): the CUDA path, called through the C ABI (libgod.so), against the CPU oracle,
element by element on the same seeded inputs.  Integer work -> bit-exact.  Sizes span many tiles
(a tile = 2048 k-mer starts) and ragged tails; edge cases: empty / short / all-N sequences, even k
(palindromes), homopolymers (ties), k = 1, k = 28, w = 1, w = 255, p = 1, long patterns."""
import zlib

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2211_08157_b200 as god  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    return True


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def np_(t):
    return t.cpu().numpy()


def pack_oracle(seq, offs, pattern, phases):
    """Oracle sparsify output in god_sparsify's documented packing (god.h stage 1)."""
    words, nms, oo, cnts = [], [], [0], []
    for i in range(len(offs) - 1):
        s = int(phases[i]) if phases is not None else 0
        codes, _ = oracle.sparsify(seq[int(offs[i]):int(offs[i + 1])], pattern, s)
        n = codes.size
        cnts.append(n)
        nw = (n + 31) // 32
        for wi in range(nw):
            word, nm = 0, 0
            for b in range(32):
                q = wi * 32 + b
                if q >= n:
                    break
                c = int(codes[q])
                if c == 4:
                    nm |= 1 << b
                else:
                    word |= c << (2 * b)
            words.append(word)
            nms.append(nm)
        oo.append(oo[-1] + nw)
    return (np.array(words, np.uint64), np.array(nms, np.uint64), np.array(oo, np.uint64), np.array(cnts, np.uint64))


def random_seqs(rng, n, lo, hi, n_frac=0.0, lowcomp=False):
    seqs = []
    for i in range(n):
        L = int(rng.integers(lo, hi + 1))
        if lowcomp and i % 3 == 0:
            s = np.frombuffer(b"AAAAAAAACA", np.uint8)[rng.integers(0, 10, size=L)].copy()
        else:
            s = synth.random_acgt(rng, L, n_frac)
        seqs.append(s)
    return synth.concat(seqs)


# ------------------------------------------------------------------------------------ stage 1
@pytest.mark.parametrize("pattern", ["10", "110", "1110", "1", "0110100101", "1" + "0" * 62 + "1"])
def test_sparsify_parity(pattern):
    rng = np.random.default_rng(1)
    seq, offs = random_seqs(rng, 300, 0, 700, 0.03)
    p = len(pattern)
    phases = rng.integers(0, p, size=len(offs) - 1).astype(np.uint8)
    for ph in (None, phases):
        want = pack_oracle(seq, offs, pattern, ph)
        for dev in (True, False):
            args = (cu(seq), cu(offs)) if dev else (seq, offs)
            pk, nm, oo, cnt = god.god_sparsify(*args, pattern, phases=None if ph is None else (cu(ph) if dev else ph))
            got = [np_(x) if dev else x for x in (pk, nm, oo, cnt)]
            for g, w_ in zip(got, want):
                assert np.array_equal(g, w_)


# ------------------------------------------------------------------------------------ stage 2
MZ_CASES = [
    # (pattern, k, w, nseq, lo, hi, nfrac, lowcomp)
    ("10", 21, 11, 40, 0, 30000, 0.0, False),
    ("10", 21, 11, 200, 0, 400, 0.02, True),
    ("110", 19, 19, 60, 0, 5000, 0.01, True),
    ("1110", 15, 10, 60, 0, 5000, 0.0, False),
    ("1", 15, 10, 30, 0, 20000, 0.005, True),
    ("10", 4, 3, 100, 0, 600, 0.05, True),        # even k: palindromes
    ("1", 1, 1, 50, 0, 300, 0.1, True),
    ("101", 28, 40, 30, 0, 4000, 0.0, False),
    ("1", 12, 255, 20, 0, 6000, 0.002, True),
    ("11", 6, 2, 80, 0, 200, 0.2, True),
    ("1" + "0" * 20, 5, 4, 20, 0, 3000, 0.0, False),
]


@pytest.mark.parametrize("case", MZ_CASES, ids=[f"{c[0]}-k{c[1]}-w{c[2]}" for c in MZ_CASES])
def test_minimizer_parity(case):
    pattern, k, w, nseq, lo, hi, nf, lc = case
    rng = np.random.default_rng(zlib.crc32(repr(case).encode()))
    seq, offs = random_seqs(rng, nseq, lo, hi, nf, lc)
    p = len(pattern)
    phases = rng.integers(0, p, size=len(offs) - 1).astype(np.uint8)
    for gp in (False, True):
        want, wo = oracle.minimizers_batch(seq, offs, pattern, k, w, phases=phases, global_pos=gp)
        h, ps, z, oo = god.god_minimizers(cu(seq), cu(offs), pattern, k, w, phases=cu(phases), global_pos=gp)
        assert np.array_equal(np_(oo), wo)
        assert np.array_equal(np_(h), want["hash"])
        assert np.array_equal(np_(ps).astype(np.uint64), want["pos"])
        assert np.array_equal(np_(z), want["strand"])
    # host-pointer path through the same ABI
    h2, p2, z2, oo2 = god.god_minimizers(seq, offs, pattern, k, w, phases=phases)
    want, wo = oracle.minimizers_batch(seq, offs, pattern, k, w, phases=phases)
    assert np.array_equal(h2, want["hash"]) and np.array_equal(oo2, wo)


def test_minimizer_edge_inputs():
    # no sequences; only empty sequences; all-N; shorter than k
    for seqs in ([], [np.zeros(0, np.uint8)] * 5, [np.frombuffer(b"N" * 500, np.uint8)],
                 [np.frombuffer(b"ACGTAC", np.uint8), np.frombuffer(b"A", np.uint8)]):
        seq, offs = synth.concat(seqs)
        want, wo = oracle.minimizers_batch(seq, offs, "10", 5, 3)
        h, ps, z, oo = god.god_minimizers(seq, offs, "10", 5, 3)
        assert np.array_equal(oo, wo)
        assert np.array_equal(h, want["hash"]) and np.array_equal(ps.astype(np.uint64), want["pos"])


# ------------------------------------------------------------------------------------ stage 3
def _index_parity(ref, offs, pattern, k, w, cutoff=(1, 5000), max_occ=None, host=False):
    ix = god.god_build_index(ref if host else cu(ref), offs if host else cu(offs), pattern, k, w, cutoff=cutoff,
                             max_occ=max_occ)
    ox = oracle.Index(ref, offs, pattern, k, w, cutoff=cutoff, max_occ=-1 if max_occ is None else max_occ)
    st, ost = ix.stats(), ox.stats()
    for f in oracle.STATS_FIELDS:
        assert st[f] == ost[f], (f, st[f], ost[f])
    h, p, z = ix.dump()
    oh, op, oz = ox.dump()
    assert np.array_equal(h, oh)
    assert np.array_equal(p.astype(np.uint64), op)
    assert np.array_equal(z, oz)
    # occ() probes, present and absent hashes
    q = np.concatenate([oh[:: max(1, oh.size // 2000)], np.arange(0, 3000, dtype=np.uint64) * 7919 % (4 ** k)])
    got = np_(ix.count(cu(q)))
    want = np.array([ox.occ(int(v)) for v in q], np.uint32)
    assert np.array_equal(got, want)
    return ix, ox


def test_index_parity_tiny_config():
    cfg = synth.make_config("tiny")
    ix, ox = _index_parity(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    assert ix.stats()["kept_entries"] > 50000


@pytest.mark.parametrize("pattern,k,w", [("10", 15, 10), ("110", 13, 7), ("1", 11, 5), ("1110", 9, 4)])
def test_index_parity_repeats_and_cutoff(pattern, k, w):
    rng = np.random.default_rng(7)
    rep = synth.random_acgt(rng, 700)
    parts = []
    for i in range(60):
        parts += [synth.random_acgt(rng, int(rng.integers(500, 5000)), 0.001), rep]
    seqs = [np.concatenate(parts[i:i + 10]) for i in range(0, len(parts), 10)] + [np.zeros(0, np.uint8)]
    ref, offs = synth.concat(seqs)
    for cut in [(1, 5000), (1, 200), (1, 20)]:
        _index_parity(ref, offs, pattern, k, w, cutoff=cut)
    for mo in [0, 1, 3, 60]:
        _index_parity(ref, offs, pattern, k, w, max_occ=mo)


def test_index_parity_homopolymer_heavy():
    # all-ties runs make single hashes with very large counts (exercises the large-count select)
    rng = np.random.default_rng(3)
    parts = []
    for i in range(40):
        parts += [synth.random_acgt(rng, 3000), np.frombuffer(b"A" * int(rng.integers(100, 9000)), np.uint8)]
    ref, offs = synth.concat([np.concatenate(parts)])
    for cut in [(1, 5000), (1, 3), (1, 2)]:
        _index_parity(ref, offs, "1", 7, 5, cutoff=cut)


@pytest.mark.parametrize("mode0", [False, True])
@pytest.mark.parametrize("k,w", [(21, 11), (15, 10), (9, 5)])
def test_index_probe_every_hash(k, w, mode0, monkeypatch):
    """Every kept hash and both its neighbours probed (god_index_count) against the oracle's kept
    entries: slots of <= 6 entries, long slots of 1-3 distinct keys (answered from the slot
    record) and of more keys (searched), absent keys between and around the runs."""
    if mode0:
        monkeypatch.setenv("GOD_DIR_MODE0", "1")
    rng = np.random.default_rng(53 + k)
    base = synth.dup_genome(600_000, 5 + k, dup_frac=0.3, lmin=100, lmax=3000)
    reps = [synth.random_acgt(rng, int(rng.integers(30, 400))) for _ in range(40)]
    parts = [base]
    for i, r in enumerate(reps):  # copy numbers 2..80: hashes of every count up to the cutoff
        parts += [r] * (2 + 2 * i)
    ref, offs = synth.concat([np.concatenate(parts)])
    ix = god.god_build_index(cu(ref), cu(offs), "10", k, w, max_occ=70)
    ox = oracle.Index(ref, offs, "10", k, w, max_occ=70)
    oh, _, _ = ox.dump()
    dist = np.unique(oh)
    top = np.uint64((1 << (2 * k)) - 1)
    q = np.unique(np.concatenate([dist, dist + np.uint64(1), dist - np.uint64(1)]))
    q = q[q <= top]
    got = np_(ix.count(cu(q)))
    want = (np.searchsorted(oh, q, side="right") - np.searchsorted(oh, q, side="left")).astype(np.uint32)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    assert (want > 6).sum() > 100  # frequent hashes present: long slots


@pytest.mark.parametrize("env", [{}, {"GOD_BIN_TARGET": "6000"}, {"GOD_BIN_TARGET": "3000"}, {"GOD_BIN_TARGET": "40"},
                                 {"GOD_DIR_MODE0": "1"}, {"GOD_SORT_FULL": "1"},
                                 {"GOD_BIN_TARGET": "40", "GOD_BIN_3PASS": "1"}, {"GOD_SEG_SAMPLE": "3"}],
                         ids=["default", "big-bins", "mid-bins", "tiny-bins", "dir-mode0", "full-lsd", "three-pass",
                              "sampled-seg-hist"])
def test_index_parity_sort_and_directory_variants(env, monkeypatch):
    """k = 21 on a repeat-rich reference through every sort/directory path: bins above the SMEM
    capacity (chunked global kernel), bins between one and two capacities (in-SMEM bitonic path),
    one-record bins, the top-bit directory, the full LSD, a third LSD pass over the bin bits (what an
    input of > 373 M records takes), a block-sampled segment histogram."""
    for kk, vv in env.items():
        monkeypatch.setenv(kk, vv)
    ref = synth.dup_genome(3_000_000, 31, dup_frac=0.35, lmin=200, lmax=4000)
    rng = np.random.default_rng(31)
    rep = synth.random_acgt(rng, 900)
    ref = np.concatenate([ref] + [rep] * 300 + [np.frombuffer(b"ACGTTGCA" * 2000, np.uint8)])
    offs = np.array([0, 1_000_000, ref.size], np.uint64)
    ix, ox = _index_parity(ref, offs, "10", 21, 11, cutoff=(1, 2000))
    reads = synth.simulate_reads(ref, 3000, 41, length=150, p_sub=0.002)
    _seed_parity(ix, ox, reads.seq, reads.offsets)


@pytest.mark.parametrize("chunk", ["4096", "50000", "0"])
@pytest.mark.parametrize("pattern,k,w", [("10", 21, 11), ("110", 21, 11), ("1", 19, 19), ("10", 15, 10), ("110", 13, 7)])
def test_index_streamed_host_reference(pattern, k, w, chunk, monkeypatch):
    """A host reference goes up in chunks while K1 runs on the tiles whose bytes are in (god_build_index;
    GOD_STREAM_CHUNK_BYTES shrinks the chunks so that a small input takes 16 of them): the unordered
    specialised kernel consumes the stream range by range (k = 21, 19), the ordered and the generic
    kernels wait for all of it (k = 15, 13); "0" disables streaming.  Several sequences, an empty one,
    N runs across chunk borders."""
    monkeypatch.setenv("GOD_STREAM_CHUNK_BYTES", chunk)
    rng = np.random.default_rng(97)
    seqs = [synth.random_acgt(rng, int(n), 0.002) for n in (90_000, 0, 3, 150_001, 40, 77_777)]
    seqs[3][49_990:50_040] = ord("N")
    seqs[0][4090:4100] = ord("N")
    ref, offs = synth.concat(seqs)
    ix, ox = _index_parity(ref, offs, pattern, k, w, cutoff=(1, 1000), host=True)
    pinned = torch.from_numpy(ref).pin_memory()
    ix2 = god.god_build_index(pinned.numpy(), offs, pattern, k, w, cutoff=(1, 1000))
    for a, b in zip(ix.dump(), ix2.dump()):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------------------------ stage 4
def canon(an):
    """anchors -> array sorted by (read_id, ref_pos, read_pos, strand)"""
    a = np.asarray(an)
    if a.dtype.names is None:
        a = a.reshape(-1, 4)
        rec = np.zeros(a.shape[0], oracle.ANCHOR_DTYPE)
        rec["ref_pos"], rec["read_pos"], rec["read_id"], rec["strand"] = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
        a = rec
    else:
        rec = np.zeros(a.size, oracle.ANCHOR_DTYPE)
        for f in ("ref_pos", "read_pos", "read_id", "strand"):
            rec[f] = a[f]
        a = rec
    return np.sort(a, order=["read_id", "ref_pos", "read_pos", "strand"])


def _seed_parity(ix, ox, reads, roffs, phases=None, t=16, sample=None):
    an, ao, ph = god.god_seed_reads(ix, cu(reads), cu(roffs), phases=None if phases is None else cu(phases), t=t)
    an, ao, ph = np_(an), np_(ao), np_(ph)
    ids = np.arange(len(roffs) - 1) if sample is None else sample
    sub_seqs = [reads[int(roffs[i]):int(roffs[i + 1])] for i in ids]
    sub, soffs = synth.concat(sub_seqs)
    sph = None if phases is None else phases[ids]
    oan, oao, oph = ox.seed_reads(sub, soffs, phases=sph, t=t)
    assert np.array_equal(ph[ids], oph)
    # per-read anchor counts and canonical anchor lists
    assert np.array_equal((ao[ids + 1] - ao[ids]), np.diff(oao))
    g = np.concatenate([an[int(ao[i]):int(ao[i + 1])] for i in ids]) if len(ids) else an[:0]
    g = canon(g)
    remap = np.zeros(len(roffs), np.uint32)
    remap[ids] = np.arange(len(ids), dtype=np.uint32)
    g["read_id"] = remap[g["read_id"]]
    g = np.sort(g, order=["read_id", "ref_pos", "read_pos", "strand"])
    assert np.array_equal(g, canon(oan))
    return an, ao, ph


def test_seed_parity_tiny_config():
    cfg = synth.make_config("tiny")
    ix = god.god_build_index(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    an, ao, ph = _seed_parity(ix, ox, cfg.reads.seq, cfg.reads.offsets)
    assert an.shape[0] > 50000
    # GIVEN mode with the selected phases and with flipped phases
    _seed_parity(ix, ox, cfg.reads.seq, cfg.reads.offsets, phases=ph)
    _seed_parity(ix, ox, cfg.reads.seq, cfg.reads.offsets, phases=(1 - ph).astype(np.uint8))


@pytest.mark.parametrize("pattern,k,w,t", [("110", 15, 10, 16), ("1110", 13, 6, 4), ("1", 15, 10, 16),
                                           ("10", 9, 5, 1), ("0101", 11, 8, 40)])
def test_seed_parity_mixed_reads(pattern, k, w, t):
    rng = np.random.default_rng(17)
    ref = synth.dup_genome(400_000, 9, dup_frac=0.2, lmin=300, lmax=2000)
    roffs_ref = np.array([0, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 700, 5, mu=6.5, sigma=1.0, lmin=1, lmax=6000, p_sub=0.01, p_ins=0.005,
                                 p_del=0.005)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    seqs += [np.zeros(0, np.uint8), np.frombuffer(b"N" * 400, np.uint8), synth.random_acgt(rng, 3000, 0.3),
             np.frombuffer(b"ACGTTGCAAC", np.uint8)]
    rs, ro = synth.concat(seqs)
    ix = god.god_build_index(cu(ref), cu(roffs_ref), pattern, k, w, cutoff=(1, 500))
    ox = oracle.Index(ref, roffs_ref, pattern, k, w, cutoff=(1, 500))
    _seed_parity(ix, ox, rs, ro, t=t)
    ph = rng.integers(0, len(pattern), size=len(ro) - 1).astype(np.uint8)
    _seed_parity(ix, ox, rs, ro, phases=ph, t=t)


@pytest.mark.parametrize("pattern,k,w", [("10", 21, 11), ("1", 15, 10), ("110", 19, 19)])
def test_seed_long_reads_slotted_and_overflow(pattern, k, w, monkeypatch, capfd):
    """Long reads through the specialised kernel's slotted position-ordered output (tile t at slot
    t * 512, then scan + copy), and its fallback to the look-back kernel: a homopolymer run makes every
    position of a tile a minimizer (more than the 512 records a slot holds)."""
    rng = np.random.default_rng(23)
    ref = synth.dup_genome(600_000, 13, dup_frac=0.2, lmin=300, lmax=3000)
    ref = np.concatenate([ref, np.frombuffer(b"A" * 9000, np.uint8), synth.random_acgt(rng, 5000)])
    roffs_ref = np.array([0, ref.size], np.uint64)
    ix = god.god_build_index(cu(ref), cu(roffs_ref), pattern, k, w, cutoff=(1, 100))
    ox = oracle.Index(ref, roffs_ref, pattern, k, w, cutoff=(1, 100))
    reads = synth.simulate_reads(ref, 60, 7, mu=9.0, sigma=0.5, lmin=2000, lmax=30000, p_sub=0.005, p_ins=0.002,
                                 p_del=0.002)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    monkeypatch.setenv("GOD_DEBUG_SLOTS", "1")
    _seed_parity(ix, ox, *synth.concat(seqs))  # slotted path only
    err = capfd.readouterr().err
    assert "extract_seed slotted" in err and "overflow=1" not in err
    seqs.insert(20, np.concatenate([synth.random_acgt(rng, 4000), np.frombuffer(b"A" * 8000, np.uint8),
                                    synth.random_acgt(rng, 3000)]))
    rs, ro = synth.concat(seqs)
    _seed_parity(ix, ox, rs, ro)  # a tile overflows its slot: the look-back kernel
    assert "overflow=1" in capfd.readouterr().err
    ph = rng.integers(0, len(pattern), size=len(ro) - 1).astype(np.uint8)
    _seed_parity(ix, ox, rs, ro, phases=ph)
    monkeypatch.setenv("GOD_SEED_GENERAL", "1")  # the per-record writer behind the read-ordered copy
    _seed_parity(ix, ox, rs, ro, phases=ph)
    _seed_parity(ix, ox, rs, ro)


def test_seed_host_pointer_path():
    cfg = synth.make_config("tiny", read_scale=0.1)
    ix = god.god_build_index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    an, ao, ph = god.god_seed_reads(ix, cfg.reads.seq, cfg.reads.offsets)
    oan, oao, oph = ox.seed_reads(cfg.reads.seq, cfg.reads.offsets)
    assert np.array_equal(ph, oph) and np.array_equal(ao, oao)
    assert np.array_equal(canon(an), canon(oan))


@pytest.mark.parametrize("given,reads_dev", [(False, False), (True, False), (False, True), (True, True)])
def test_seed_host_pipelined_batches(given, reads_dev, monkeypatch):
    """All-host buffers above the batch threshold take the pipelined path (read batches copied in,
    seeded and copied out on three streams); batches shrunk by the test hook so that it runs here,
    with long reads (the dedicated PQ_a extraction) and edge reads spread over the batches."""
    monkeypatch.setenv("GOD_PIPE_MIN_READS", "97")
    rng = np.random.default_rng(23)
    ref = synth.dup_genome(300_000, 13, dup_frac=0.2, lmin=300, lmax=2000)
    roffs_ref = np.array([0, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 800, 7, mu=5.5, sigma=1.2, lmin=1, lmax=5000, p_sub=0.01, p_ins=0.005,
                                 p_del=0.005)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    seqs[100:100] = [np.zeros(0, np.uint8), np.frombuffer(b"N" * 400, np.uint8), synth.random_acgt(rng, 3000, 0.3)]
    rs, ro = synth.concat(seqs)
    ix = god.god_build_index(cu(ref), cu(roffs_ref), "10", 15, 10, cutoff=(1, 500))
    ox = oracle.Index(ref, roffs_ref, "10", 15, 10, cutoff=(1, 500))
    ph = rng.integers(0, 2, size=len(ro) - 1).astype(np.uint8) if given else None
    if reads_dev:  # reads on the device, results streamed back to host buffers batch by batch
        an, ao, gph = god.god_seed_reads(ix, cu(rs), cu(ro), phases=ph, host_out=True)
    else:
        an, ao, gph = god.god_seed_reads(ix, rs, ro, phases=ph)
    oan, oao, oph = ox.seed_reads(rs, ro, phases=ph)
    assert np.array_equal(gph, oph) and np.array_equal(ao, oao)
    assert np.array_equal(canon(an), canon(oan))


@pytest.mark.parametrize("compact", [False, True])
@pytest.mark.parametrize("where", ["host_overlapped", "host_plain", "device"])
def test_build_index_and_seed(where, compact, monkeypatch):
    """god_build_index_and_seed = god_build_index then god_seed_reads(_compact): with host buffers above the
    batch threshold the first read batches are queued behind the streamed reference (both test hooks
    shrink chunks and batches so that 16 chunks and 8 batches over a ring of 4 slots run here); below it,
    and with device buffers, the two calls run in sequence.  Index, phases, offsets and anchors against the
    oracle; a capacity that is too small keeps the index and reports the count."""
    if where == "host_overlapped":
        monkeypatch.setenv("GOD_PIPE_MIN_READS", "97")
        monkeypatch.setenv("GOD_STREAM_CHUNK_BYTES", "20000")
    rng = np.random.default_rng(29)
    ref = synth.dup_genome(400_000, 17, dup_frac=0.2, lmin=300, lmax=2000)
    roffs_ref = np.array([0, 150_000, 150_000, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 800, 11, mu=5.5, sigma=1.0, lmin=1, lmax=4000, p_sub=0.01, p_ins=0.003,
                                 p_del=0.003)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    seqs[50:50] = [np.zeros(0, np.uint8), np.frombuffer(b"N" * 300, np.uint8)]
    rs, ro = synth.concat(seqs)
    ox = oracle.Index(ref, roffs_ref, "10", 21, 11, cutoff=(1, 500))
    oan, oao, oph = ox.seed_reads(rs, ro)
    conv = cu if where == "device" else (lambda a: a)
    for cap in (None, 1000):
        ix, an, ao, ph = god.god_build_index_and_seed(conv(ref), conv(roffs_ref), conv(rs), conv(ro), "10", 21, 11,
                                                      cutoff=(1, 500), compact=compact, cap=cap)
        for a, b in zip(ix.dump(), ox.dump()):
            assert np.array_equal(np.asarray(a).astype(np.uint64), np.asarray(b).astype(np.uint64))
        if where == "device":
            an, ao, ph = np_(an), np_(ao), np_(ph)
        assert np.array_equal(ph, oph) and np.array_equal(ao, oao)
        full = god.expand_compact(an, ao) if compact else an
        assert np.array_equal(canon(full), canon(oan))
    ph_in = rng.integers(0, 2, size=len(ro) - 1).astype(np.uint8)
    ix, an, ao, ph = god.god_build_index_and_seed(conv(ref), conv(roffs_ref), conv(rs), conv(ro), "10", 21, 11,
                                                  cutoff=(1, 500), compact=compact, phases=conv(ph_in))
    oan2, oao2, _ = ox.seed_reads(rs, ro, phases=ph_in)
    if where == "device":
        an, ao = np_(an), np_(ao)
    assert np.array_equal(ao, oao2)
    assert np.array_equal(canon(god.expand_compact(an, ao) if compact else an), canon(oan2))


@pytest.mark.parametrize("where", ["device", "host", "host_pipelined", "reads_dev_pipelined"])
def test_seed_compact_anchors(where, monkeypatch):
    """god_seed_reads_compact: the 8-byte anchors expand (read id from the offsets, strand from bit
    31) to exactly god_seed_reads' anchors, in the same order, on every buffer path; a too-small
    capacity reports the needed count and the retry matches too."""
    if where.endswith("pipelined"):
        monkeypatch.setenv("GOD_PIPE_MIN_READS", "97")
    rng = np.random.default_rng(41)
    ref = synth.dup_genome(300_000, 19, dup_frac=0.2, lmin=300, lmax=2000)
    roffs_ref = np.array([0, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 700, 3, mu=5.5, sigma=1.2, lmin=1, lmax=5000, p_sub=0.01, p_ins=0.005,
                                 p_del=0.005)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    seqs[50:50] = [np.zeros(0, np.uint8), np.frombuffer(b"N" * 300, np.uint8), synth.random_acgt(rng, 2000, 0.3)]
    rs, ro = synth.concat(seqs)
    ix = god.god_build_index(cu(ref), cu(roffs_ref), "10", 15, 10, cutoff=(1, 500))
    ox = oracle.Index(ref, roffs_ref, "10", 15, 10, cutoff=(1, 500))
    args = {"device": (cu(rs), cu(ro), {}), "host": (rs, ro, {}), "host_pipelined": (rs, ro, {}),
            "reads_dev_pipelined": (cu(rs), cu(ro), {"host_out": True})}[where]
    full = god.god_seed_reads(ix, args[0], args[1], **args[2])
    for cap in (None, 7):
        cmp_ = god.god_seed_reads(ix, args[0], args[1], compact=True, cap=cap, **args[2])
        ao = cmp_[1].cpu().numpy() if isinstance(cmp_[1], torch.Tensor) else cmp_[1]
        fao = full[1].cpu().numpy() if isinstance(full[1], torch.Tensor) else full[1]
        assert np.array_equal(ao, fao)
        exp = god.expand_compact(cmp_[0], cmp_[1])
        fa = full[0].cpu().numpy().view(god.ANCHOR_DTYPE).reshape(-1) if isinstance(full[0], torch.Tensor) \
            else full[0]
        assert np.array_equal(exp, fa)
    oan, oao, _ = ox.seed_reads(rs, ro)
    assert np.array_equal(canon(exp), canon(oan))


# ------------------------------------------------------------------------------------ K1 v2 (specialised)
X2_COMBOS = [("10", 21, 11), ("01", 21, 11), ("1", 21, 11), ("10", 19, 19), ("1", 19, 19), ("10", 15, 10),
             ("1", 15, 10), ("110", 21, 11), ("1110", 21, 11), ("110", 19, 19), ("1110", 19, 19), ("110", 15, 10),
             ("1110", 15, 10), ("10", 19, 16), ("1", 19, 16), ("110", 19, 16), ("1110", 19, 16), ("100", 21, 11),
             ("010", 19, 19), ("001", 15, 10), ("100", 19, 16)]


@pytest.mark.parametrize("combo", X2_COMBOS, ids=[f"{c[0]}-k{c[1]}-w{c[2]}" for c in X2_COMBOS])
@pytest.mark.parametrize("keybits", [None, "9"])
def test_x2_specialised_kernel_parity(combo, keybits, monkeypatch):
    """The register-resident kernel (extract2.cu) on long N-free sequences (fast path), sequences
    with N runs and short sequences (exact slow path); keybits=9 makes 31-bit key ties frequent so
    the exactness check + slow path run on most tiles."""
    pattern, k, w = combo
    if keybits:
        monkeypatch.setenv("GOD_DEBUG_KEYBITS", keybits)
    rng = np.random.default_rng(zlib.crc32(repr(combo).encode()))
    seqs = [synth.random_acgt(rng, int(rng.integers(20000, 60000))) for _ in range(3)]
    seqs += [synth.sprinkle_n(synth.random_acgt(rng, 30000), 5, 6, 40)]
    seqs += [synth.random_acgt(rng, int(rng.integers(0, 200)), 0.01) for _ in range(60)]
    seqs += [np.frombuffer(b"ACGT" * 3000, np.uint8).copy(), np.frombuffer(b"A" * 5000, np.uint8).copy()]
    seq, offs = synth.concat(seqs)
    phases = rng.integers(0, len(pattern), size=len(offs) - 1).astype(np.uint8)
    for gp, ph in ((True, None), (False, phases)):
        want, wo = oracle.minimizers_batch(seq, offs, pattern, k, w, phases=ph, global_pos=gp)
        h, ps, z, oo = god.god_minimizers(cu(seq), cu(offs), pattern, k, w,
                                          phases=None if ph is None else cu(ph), global_pos=gp)
        assert np.array_equal(np_(oo), wo)
        assert np.array_equal(np_(h), want["hash"])
        assert np.array_equal(np_(ps).astype(np.uint64), want["pos"])
        assert np.array_equal(np_(z), want["strand"])


def test_x2_matches_generic_kernel(monkeypatch):
    cfg = synth.make_config("tiny", read_scale=0.2)
    a = god.god_minimizers(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11, global_pos=True)
    monkeypatch.setenv("GOD_DISABLE_X2", "1")
    b = god.god_minimizers(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11, global_pos=True)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_misaligned_device_buffers():
    """Sequence buffers that start at any byte address (tensor slices): K1 aligns its word loads in
    the address space, so results equal the aligned case and the oracle."""
    cfg = synth.make_config("tiny")
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    n = 300
    sub, soffs = synth.concat([cfg.reads.seq[int(cfg.reads.offsets[i]):int(cfg.reads.offsets[i + 1])]
                               for i in range(n)])
    oan, oao, oph = ox.seed_reads(sub, soffs)
    for shift in (1, 2, 3, 5):
        big = torch.zeros(cfg.ref.size + 16, dtype=torch.uint8, device="cuda")
        big[shift:shift + cfg.ref.size] = cu(cfg.ref)
        ref_view = big[shift:shift + cfg.ref.size]
        assert ref_view.data_ptr() % 4 == shift % 4
        ix = god.god_build_index(ref_view, cu(cfg.ref_offsets), "10", 21, 11)
        h, p, z = ix.dump()
        oh, op, oz = ox.dump()
        assert np.array_equal(h, oh) and np.array_equal(p.astype(np.uint64), op) and np.array_equal(z, oz)
        rb = torch.zeros(sub.size + 16, dtype=torch.uint8, device="cuda")
        rb[shift:shift + sub.size] = cu(sub)
        an, ao, ph = god.god_seed_reads(ix, rb[shift:shift + sub.size], cu(soffs))
        assert np.array_equal(np_(ph), oph) and np.array_equal(np_(ao), oao)
        assert np.array_equal(canon(np_(an)), canon(oan))


def test_rebuild_and_reseed_are_byte_identical():
    """re-indexing is byte-identical; seeding and voting are deterministic too (anchor order,
    phases, voted locations), on a repeat-rich reference whose sort paths include big bins."""
    rng = np.random.default_rng(31)
    rep = synth.random_acgt(rng, 3000)
    ref = np.concatenate([synth.dup_genome(500_000, 17, dup_frac=0.3, lmin=300, lmax=3000)] + [rep] * 200)
    offs = np.array([0, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 3000, 19, length=150, p_sub=0.002)
    outs = []
    for _ in range(2):
        ix = god.god_build_index(cu(ref), cu(offs), "10", 21, 11, cutoff=(1, 1000))
        h, p, z = ix.dump()
        an, ao, ph = god.god_seed_reads(ix, cu(reads.seq), cu(reads.offsets))
        v, vo = god.god_vote_reads(ix, cu(reads.seq), cu(reads.offsets), ph, an, ao, V=2)
        outs.append([np.asarray(x) for x in (h, p, z)] + [np_(x) for x in (an, ao, ph, v, vo)])
        ix.free()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
