"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/) is checked against things other than itself: the worked examples in
tests/golden/ (each cited), closed forms, exhaustive bijectivity, an independent big-integer
hash, a brute-force window enumerator (tests/brute.py) on tiny random inputs, and invariants the
paper or the mathematics fix.  Each test names the PAPER.md passage (P:n) it pins.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from brute import brute_minimizers, revcomp, sparsify_str, true_phases, wang_hash_bigint

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def b(s: str) -> np.ndarray:
    return np.frombuffer(s.encode(), dtype=np.uint8).copy()


@pytest.fixture(scope="module", autouse=True)
def _libs(built):
    return built


# ---------------------------------------------------------------------------- O1 encoding
def test_encoding_table_exhaustive():
    want = {ord("A"): 0, ord("a"): 0, ord("C"): 1, ord("c"): 1, ord("G"): 2, ord("g"): 2, ord("T"): 3, ord("t"): 3}
    for v in range(256):
        assert oracle.code(v) == want.get(v, 4), v
    spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in spec["encode"]:
        assert oracle.code(ord(e["base"])) == e["code"]
        if "complement" in e:
            assert 3 - e["code"] == e["complement"]


# ---------------------------------------------------------------------------- O2 pattern
def test_parse_pattern_examples():
    spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in spec["parse_pattern"]:
        if e.get("error"):
            with pytest.raises(ValueError):
                oracle.parse_pattern(e["text"])
        else:
            p, x = oracle.pattern_info(e["text"])
            assert (p, x) == (e["p"], e["x"])
            assert p * e["beta"][1] == x * e["beta"][0]   # beta = p/x
    with pytest.raises(ValueError):
        oracle.parse_pattern("1" * 65)
    assert oracle.pattern_info("1" * 64) == (64, 64)


# ---------------------------------------------------------------------------- O3 sparsify
def test_sparsify_examples():
    spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in spec["apply_pattern"]:
        codes, orig = oracle.sparsify(b(e["seq"]), e["pattern"], e["s"])
        assert "".join("ACGTN"[c] for c in codes) == e["included"]
        assert orig.tolist() == e["orig"]


@pytest.mark.parametrize("pattern", ["10", "110", "1110", "1", "101001", "0001", "10" * 32])
def test_sparsify_closed_form_and_shift(pattern):
    rng = np.random.default_rng(5)
    p = len(pattern)
    x = pattern.count("1")
    for L in [0, 1, p - 1, p, 3 * p + 1, 257]:
        seq = synth.random_acgt(rng, L, 0.05)
        for s in range(p):
            codes, orig = oracle.sparsify(seq, pattern, s)
            # |J| = x*floor((L-s)/p) + #ones in P[0..(L-s) mod p)
            if L > s:
                full, rem = divmod(L - s, p)
                want = x * full + pattern[:rem].count("1")
            else:
                want = 0
            assert codes.size == want
            # origin map strictly increasing; equals the brute "repeated diet pattern" formulation
            sub, o2 = sparsify_str(seq.tobytes().decode(), pattern, s)
            assert orig.tolist() == o2
            assert np.all(np.diff(orig.astype(np.int64)) > 0)
            # composition: shift s on Q == shift 0 on Q[s:], positions + s
            c0, o0 = oracle.sparsify(seq[s:], pattern, 0)
            assert np.array_equal(c0, codes) and np.array_equal(o0 + s, orig)
    # all-ones pattern is the identity
    seq = synth.random_acgt(rng, 100)
    codes, orig = oracle.sparsify(seq, "1", 0)
    assert orig.tolist() == list(range(100))


# ---------------------------------------------------------------------------- O5 hash (ref. 120)
@pytest.mark.parametrize("k", range(1, 8))
def test_hash_closed_form_small_k(k):
    """For 2k <= 14 the xor-shifts and the 2^21, 2^31 terms vanish mod 4^k, so
    H_k(x) = 21*265*(4^k - 1 - x) mod 4^k = 5565*(4^k - 1 - x) mod 4^k (derived in SURVEY §8(c) O5)."""
    m = 4 ** k
    xs = np.arange(m, dtype=np.uint64)
    got = oracle.hash_batch(xs, k)
    want = (5565 * (m - 1 - xs.astype(object))) % m
    assert got.tolist() == [int(v) for v in want]


@pytest.mark.parametrize("k", range(1, 11))
def test_hash_is_bijection(k):
    m = 4 ** k
    got = oracle.hash_batch(np.arange(m, dtype=np.uint64), k)
    assert got.max() < m
    assert np.unique(got).size == m


def test_hash_vs_independent_bigint():
    rng = np.random.default_rng(7)
    for k in [8, 11, 15, 16, 19, 21, 24, 28]:
        xs = rng.integers(0, 4 ** k, size=2000, dtype=np.uint64)
        got = oracle.hash_batch(xs, k)
        for xv, gv in zip(xs.tolist(), got.tolist()):
            assert gv == wang_hash_bigint(int(xv), k)


def _unxorshift(y, s, bits):
    """x with x ^ (x >> s) == y (mod 2^bits): x = y ^ y>>s ^ y>>2s ^ ..."""
    x, t = 0, y
    while t:
        x ^= t
        t >>= s
    return x & ((1 << bits) - 1)


@pytest.mark.parametrize("k", [8, 11, 12, 14, 15, 16, 19, 21, 24, 28])
def test_hash_is_undone_by_the_inverse_of_its_definition(k):
    """P:370 calls the hash invertible.  The inverse is derived here step by step from the definition
     with modular inverses of the three multipliers and un-xor-shifts, none of which
    the oracle contains: a wrong shift or multiplier in the oracle (the constants that only act for
    k >= 8..15) would still be a bijection but would not be undone by this inverse."""
    bits = 2 * k
    M = 1 << bits
    rng = np.random.default_rng(100 + k)
    xs = rng.integers(0, M, size=3000, dtype=np.uint64)
    hs = oracle.hash_batch(xs, k)
    i31, i21, i265, im = pow((1 << 31) + 1, -1, M), pow(21, -1, M), pow(265, -1, M), pow((1 << 21) - 1, -1, M)
    for x, h in zip(xs.tolist(), hs.tolist()):
        x6 = (h * i31) % M
        x5 = _unxorshift(x6, 28, bits)
        x4 = (x5 * i21) % M
        x3 = _unxorshift(x4, 14, bits)
        x2 = (x3 * i265) % M
        x1 = _unxorshift(x2, 24, bits)
        assert ((x1 + 1) * im) % M == x


# ---------------------------------------------------------------------------- O4+O6 minimizers
def _mz_list(arr):
    return [(int(r["hash"]), int(r["pos"]), int(r["strand"])) for r in arr]


def test_minimizers_appendix_a():
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    ref = b(g["reference"])
    codes, orig = oracle.sparsify(ref, g["pattern"], 0)
    assert "".join("ACGT"[c] for c in codes) == g["patterned_reference"]
    assert orig.tolist() == g["patterned_reference_orig"]
    for km in g["kmers"]:
        assert oracle.hash_kmer(km["canon"], g["k"]) == km["hash"]
    mz = oracle.minimizers(ref, g["pattern"], 0, g["k"], g["w"])
    assert _mz_list(mz) == [tuple(t) for t in g["reference_minimizers"]]
    for rd in g["reads"]:
        for ph in rd["phases"]:
            mz = oracle.minimizers(b(rd["seq"]), g["pattern"], ph["s"], g["k"], g["w"])
            assert _mz_list(mz) == [tuple(t) for t in ph["minimizers"]]
    t = g["tie_example"]
    mz = oracle.minimizers(b(t["seq"]), t["pattern"], 0, t["k"], t["w"])
    assert [int(r["pos"]) for r in mz] == t["selected_pos"] and set(mz["strand"].tolist()) == {t["strand"]}
    mz = oracle.minimizers(b(t["revcomp_seq"]), t["pattern"], 0, t["k"], t["w"])
    assert [int(r["pos"]) for r in mz] == t["revcomp_selected_pos"] and set(mz["strand"].tolist()) == {1}
    n = g["n_example"]
    c0, _ = oracle.sparsify(b(n["seq"]), n["pattern"], 0)
    c1, _ = oracle.sparsify(b(n["seq"]), n["pattern"], 1)
    assert "".join("ACGTN"[c] for c in c0) == n["s0_patterned"]
    assert "".join("ACGTN"[c] for c in c1) == n["s1_patterned"]


def test_minimizers_vs_brute_force():
    rng = np.random.default_rng(11)
    patterns = ["1", "10", "01", "110", "101", "1110", "1001"]
    n_cases = 0
    for trial in range(700):
        pat = patterns[trial % len(patterns)]
        k = int(rng.integers(1, 7))
        w = int(rng.integers(1, 6))
        L = int(rng.integers(0, 40))
        nf = [0.0, 0.0, 0.08][trial % 3]
        alphabet = b"ACGT" if trial % 5 else b"AC"      # low-entropy strings force ties and palindromes
        seq = np.frombuffer(alphabet, np.uint8)[rng.integers(0, len(alphabet), size=L)].copy()
        if nf:
            seq[rng.random(L) < nf] = ord("N")
        for s in range(len(pat)):
            got = _mz_list(oracle.minimizers(seq, pat, s, k, w))
            want = brute_minimizers(seq.tobytes().decode(), pat, s, k, w)
            assert got == want, (seq.tobytes(), pat, s, k, w)
            n_cases += 1
    assert n_cases > 1000


def test_minimizer_invariants():
    """Strand mirror, window coverage, subset law in w (S:192 under all-ties),
    '10' == subsample, interior N == independent segments."""
    rng = np.random.default_rng(3)
    for trial in range(60):
        L = int(rng.integers(30, 300))
        seq = synth.random_acgt(rng, L)
        k, w = int(rng.integers(3, 12)), int(rng.integers(1, 9))
        m1 = oracle.minimizers(seq, "1", 0, k, w)
        # strand mirror: minimizers of revcomp(seq) are the mirrored positions with flipped strands
        rc = b(revcomp(seq.tobytes().decode()))
        m2 = oracle.minimizers(rc, "1", 0, k, w)
        mirror = sorted((int(h), L - k - int(p), 1 - int(z)) for h, p, z in _mz_list(m1))
        assert mirror == sorted(_mz_list(m2))
        # window coverage: every w consecutive k-mer starts contain a selected one (no N, odd k)
        if k % 2:
            pos = set(int(p) for p in m1["pos"])
            for a in range(0, L - k + 1 - w + 1):
                assert any(j in pos for j in range(a, a + w))
        # subset law: M(w2) ⊆ M(w1) for w2 >= w1
        m3 = oracle.minimizers(seq, "1", 0, k, w + 2)
        assert set(_mz_list(m3)) <= set(_mz_list(m1))
        # '10' on seq == sketching the subsample with positions mapped through orig
        sub = seq[0::2]
        ms = oracle.minimizers(sub, "1", 0, k, w)
        m10 = oracle.minimizers(seq, "10", 0, k, w)
        assert [(h, 2 * p, z) for h, p, z in _mz_list(ms)] == _mz_list(m10)
    # interior N: minimizers == those of each side sketched separately
    seq = synth.random_acgt(rng, 200)
    seq[97] = ord("N")
    left = oracle.minimizers(seq[:97], "1", 0, 9, 5)
    right = oracle.minimizers(seq[98:], "1", 0, 9, 5, pos_base=98)
    assert _mz_list(oracle.minimizers(seq, "1", 0, 9, 5)) == _mz_list(left) + _mz_list(right)


def test_minimizer_edge_cases():
    # patterned length < k -> empty;  empty input -> empty
    assert oracle.minimizers(b("ACGTACG"), "10", 0, 5, 3).size == 0
    assert oracle.minimizers(np.zeros(0, np.uint8), "1", 0, 3, 3).size == 0
    # all-ones pattern, sequence of length k, w=1 -> one minimizer at 0
    mz = oracle.minimizers(b("ACGTTGCA"[:7]), "1", 0, 7, 1)
    assert [int(p) for p in mz["pos"]] == [0]
    # all-N -> empty
    assert oracle.minimizers(b("N" * 50), "1", 0, 3, 2).size == 0
    # palindromic k-mers never selected (k even)
    seq = b("ACGTACGTACGT")
    mz = oracle.minimizers(seq, "1", 0, 4, 1)
    pal = [p for p in range(9) if seq[p:p + 4].tobytes() in (b"ACGT", b"GTAC")]
    assert pal and not set(pal) & set(mz["pos"].tolist())
    assert set(mz["pos"].tolist()) == set(range(9)) - set(pal)   # w = 1: every non-palindrome


# ---------------------------------------------------------------------------- O7 index (P:286(3))
def test_cutoff_rule_examples():
    """S:249-251 (quantile convention of reading O7)."""
    tau, m = oracle.cutoff_tau(np.ones(1000, np.uint64), 1, 1000)
    assert m == 1 and tau == 1   # all unique: nothing dropped (every count <= tau)
    c = np.ones(1000, np.uint64)
    c[17] = 1000
    tau, m = oracle.cutoff_tau(c, 1, 1000)
    assert (m, tau) == (1, 1)    # tau = a_{n-m-1} = a_998 = 1  ->  the x1000 hash is dropped
    assert int((c > tau).sum()) == 1
    tau, m = oracle.cutoff_tau(np.ones(4, np.uint64), 1, 5000)
    assert m == 0 and tau == 1   # m = floor(4/5000) = 0 -> keep all (App. A)
    # at most m distinct hashes are dropped; ties at the boundary are kept
    rng = np.random.default_rng(1)
    for _ in range(50):
        c = rng.integers(1, 30, size=int(rng.integers(1, 3000))).astype(np.uint64)
        tau, m = oracle.cutoff_tau(c, 1, 100)
        assert int((c > tau).sum()) <= m
        assert m == 0 or int((c >= tau).sum()) >= m + 1 or tau == c.max()


def test_index_appendix_a_and_spec():
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    ref = b(g["reference"])
    ix = oracle.Index(ref, np.array([0, ref.size], np.uint64), g["pattern"], g["k"], g["w"])
    h, p, z = ix.dump()
    assert list(zip(h.tolist(), p.tolist(), z.tolist())) == [tuple(t) for t in g["index_sorted"]]
    st = ix.stats()
    for key, v in g["index_stats"].items():
        assert st[key] == v
    spec = json.load(open(os.path.join(GOLD, "spec_examples.json")))["build_index_5_entries"]
    s = b(spec["seq"])
    ix = oracle.Index(s, np.array([0, s.size], np.uint64), spec["pattern"], spec["k"], spec["w"])
    h, p, z = ix.dump()
    assert sorted(p.tolist()) == spec["positions"]


def test_index_invariants_and_cutoff():
    rng = np.random.default_rng(9)
    # a reference whose segment `rep` is repeated many times -> its minimizers get high counts
    rep = synth.random_acgt(rng, 400)
    parts = []
    for i in range(30):
        parts.append(synth.random_acgt(rng, 2000))
        parts.append(rep)
    seqs = parts + [synth.random_acgt(rng, 500, 0.02)]
    cat, offs = synth.concat([np.concatenate(seqs[i:i + 6]) for i in range(0, len(seqs), 6)])
    for pat, k, w in [("10", 11, 5), ("110", 13, 7), ("1", 9, 4)]:
        E, _ = oracle.minimizers_batch(cat, offs, pat, k, w, global_pos=True)
        for frac in [(1, 5000), (1, 100), (1, 20)]:
            ix = oracle.Index(cat, offs, pat, k, w, cutoff=frac)
            st = ix.stats()
            assert st["kept_entries"] + st["dropped_entries"] == st["n_entries_all"] == E.size
            assert st["kept_distinct"] + st["dropped_distinct"] == st["n_distinct_all"]
            hs, cnt = np.unique(E["hash"], return_counts=True)
            assert st["n_distinct_all"] == hs.size
            assert st["m"] == hs.size * frac[0] // frac[1]
            assert st["dropped_distinct"] <= st["m"]
            h, p, z = ix.dump()
            # kept entries == the emitted multiset restricted to counts <= tau, in (hash, pos) order
            keep = np.isin(E["hash"], hs[cnt <= st["tau"]])
            want = sorted(zip(E["hash"][keep].tolist(), E["pos"][keep].tolist(), E["strand"][keep].tolist()))
            assert list(zip(h.tolist(), p.tolist(), z.tolist())) == want
            for hv, c in zip(hs[:50].tolist(), cnt[:50].tolist()):
                assert ix.occ(hv) == (c if c <= st["tau"] else 0)
        # index-size ordering with sparsification (Fig. 6B): '10' has <= entries than '1'
    i1 = oracle.Index(cat, offs, "1", 15, 10).stats()["n_entries_all"]
    i10 = oracle.Index(cat, offs, "10", 15, 10).stats()["n_entries_all"]
    assert i10 < i1


# ---------------------------------------------------------------------------- O8/O9 phase + seeding
def test_phase_and_seed_appendix_a():
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    ref = b(g["reference"])
    ix = oracle.Index(ref, np.array([0, ref.size], np.uint64), g["pattern"], g["k"], g["w"])
    for rid, rd in enumerate(g["reads"]):
        a, sc = ix.select_phase(b(rd["seq"]))
        assert a == rd["a"] == rd["true_phase"]
        assert sc.tolist() == [ph["score"] for ph in rd["phases"]]
        an = ix.seed_read(b(rd["seq"]), a, read_id=rid)
        assert [tuple(int(v) for v in x) for x in an] == [(rid,) + tuple(t[1:]) for t in rd["anchors"]]


def test_exact_substring_invariant_and_phase_selection():
    """P:300 premise: reads copied from the reference find their origin.  GIVEN mode with the true
    phase: every read minimizer is in the index (none dropped here) and yields an anchor with
    ref - read = g (forward) or ref + qend = g + L - 1 (reverse).  SELECT mode picks the true phase
    for > 99% of error-free reads on an i.i.d. reference."""
    rng = np.random.default_rng(21)
    ref = synth.iid_genome(200_000, 77)
    offs = np.array([0, ref.size], np.uint64)
    for pat, k, w in [("10", 21, 11), ("110", 19, 19), ("1110", 15, 10), ("1", 15, 10)]:
        ix = oracle.Index(ref, offs, pat, k, w)
        correct = 0
        n = 300
        for r in range(n):
            L = int(rng.integers(120, 400))
            g0 = int(rng.integers(0, ref.size - L))
            strand = int(rng.integers(0, 2))
            read = ref[g0:g0 + L].copy()
            if strand:
                read = b(revcomp(read.tobytes().decode()))
            ok = true_phases(pat, g0, L, strand)
            assert ok
            a, _ = ix.select_phase(read)
            correct += a in ok
            s = ok[0]
            mz = oracle.minimizers(read, pat, s, k, w)
            an = ix.seed_read(read, s)
            _, orig = oracle.sparsify(read, pat, s)
            pos2j = {int(o): j for j, o in enumerate(orig.tolist())}
            for hv, qpos, qz in _mz_list(mz):
                if ix.occ(hv) == 0:
                    continue  # dropped by the cutoff
                hits = an[an["read_pos"] == qpos]
                if not strand:
                    assert any(int(x["ref_pos"]) - qpos == g0 and int(x["strand"]) == 0 for x in hits)
                else:
                    qend = int(orig[pos2j[qpos] + k - 1])
                    assert any(int(x["ref_pos"]) + qend == g0 + L - 1 and int(x["strand"]) == 1 for x in hits)
        assert correct >= 0.99 * n, (pat, correct)


def test_phase_edge_cases():
    ref = synth.iid_genome(20000, 5)
    ix = oracle.Index(ref, np.array([0, ref.size], np.uint64), "10", 15, 10)
    assert ix.select_phase(b("N" * 300))[0] == 0            # all-N read -> phase 0
    assert ix.select_phase(b("ACGT"))[0] == 0               # too short -> no minimizers -> 0
    assert ix.seed_read(b("N" * 300), 1).size == 0          # no matches -> empty
    ix1 = oracle.Index(ref, np.array([0, ref.size], np.uint64), "1", 15, 10)
    assert ix1.select_phase(ref[100:250])[0] == 0           # p = 1 -> a = 0
