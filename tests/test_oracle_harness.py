"""Pins for the oracle's seed-comparison harness (-m "not gpu"): P:83-103 (section 2.1.1-2.1.2,
Fig. 4), readings S1-S5 (oracle/oracle.c).  Pinned by textbook edit distances and a
memoised recursive Levenshtein, special cases that reduce one extractor to another (spaced with an
all-ones mask = all k-mers; Genome-on-Diet with '1' = minimizers), constructed substitutions that a
pattern must ignore, the best-phase rule on a shifted copy, the no-false-negative property of the
accepted-pairs rule, and the rate-vs-edit-distance trend."""
import functools

import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module", autouse=True)
def _libs(built):
    return built


def b(s: str) -> np.ndarray:
    return np.frombuffer(s.encode(), np.uint8).copy()


def lev_rec(x: str, y: str) -> int:
    @functools.lru_cache(maxsize=None)
    def d(i, j):
        if i == 0:
            return j
        if j == 0:
            return i
        return min(d(i - 1, j) + 1, d(i, j - 1) + 1, d(i - 1, j - 1) + (x[i - 1] != y[j - 1]))
    return d(len(x), len(y))


def test_levenshtein_textbook_and_recursion():
    assert oracle.levenshtein(b("kitten"), b("sitting")) == 3
    assert oracle.levenshtein(b("flaw"), b("lawn")) == 2
    assert oracle.levenshtein(b(""), b("ACGT")) == 4 and oracle.levenshtein(b("ACGT"), b("ACGT")) == 0
    rng = np.random.default_rng(3)
    for _ in range(200):
        x = "".join(rng.choice(list("ACGT"), int(rng.integers(0, 9))))
        y = "".join(rng.choice(list("ACGT"), int(rng.integers(0, 9))))
        assert oracle.levenshtein(b(x), b(y)) == lev_rec(x, y)


def test_levenshtein_bounds_on_substitution_pairs():
    o, m, off, subs = synth.mutation_pairs(30, 300, 60, 9)
    for i in range(30):
        a, c = o[int(off[i]):int(off[i + 1])], m[int(off[i]):int(off[i + 1])]
        d = oracle.levenshtein(a, c)
        assert d <= int((a != c).sum()) == int(subs[i])  # <= Hamming = the substitutions made
        if subs[i] == 1:
            assert d == 1


def _rate(a, c, algo, k, w, pat, s=0):
    sa = set(oracle.harness_seeds(a, algo, k, w, pat).tolist())
    sb = oracle.harness_seeds(c, algo, k, w, pat, s)
    return sum(1 for h in sb.tolist() if h in sa), sb.size


def test_extractor_special_cases():
    rng = np.random.default_rng(4)
    seq = synth.random_acgt(rng, 500)
    for k, w in [(8, 6), (13, 9), (21, 11)]:
        allk = oracle.harness_seeds(seq, 0, k, w, "10")
        assert allk.size == 500 - k + 1
        # the hash of the canonical k-mer, restated
        for i in (0, 17, 300):
            s = seq[i:i + k].tobytes().decode()
            f = int("".join("ACGT".index(ch).__str__() for ch in s), 4)
            r = int("".join(str(3 - "ACGT".index(ch)) for ch in reversed(s)), 4)
            assert allk[i] == oracle.hash_kmer(min(f, r), k)
        # spaced seeds with an all-ones mask are all k-mers; Genome-on-Diet with '1' is minimizers
        assert np.array_equal(oracle.harness_seeds(seq, 2, k, w, "1" * k), allk)
        assert np.array_equal(oracle.harness_seeds(seq, 3, k, w, "1"), oracle.harness_seeds(seq, 1, k, w, "10"))
    # disjoint content -> rate 0; identical -> rate 1 for all four extractors
    assert _rate(b("A" * 100), b("C" * 100), 0, 8, 6, "10") == (0, 93)
    for algo in range(4):
        m, t = _rate(seq, seq, algo, 13, 9, "110")
        assert m == t > 0


def test_patterns_ignore_excluded_substitutions():
    rng = np.random.default_rng(5)
    seq = synth.random_acgt(rng, 400)
    # spaced '100', k = 8: mask 10010010, the last base is excluded from the only window covering it
    mut = seq.copy()
    mut[-1] = b"C"[0] if mut[-1] != b"C"[0] else b"G"[0]
    m, t = _rate(seq, mut, 2, 8, 6, "100")
    assert m == t
    m, t = _rate(seq, mut, 0, 8, 6, "100")
    assert m < t
    # Genome-on-Diet '10': a substitution at an odd position never enters the phase-0 sequence
    mut = seq.copy()
    mut[201] = b"A"[0] if mut[201] != b"A"[0] else b"T"[0]
    assert _rate(seq, mut, 3, 13, 9, "10") == _rate(seq, seq, 3, 13, 9, "10")
    assert _rate(seq, mut, 0, 13, 9, "10")[0] < _rate(seq, mut, 0, 13, 9, "10")[1]


def test_god_best_phase_on_shifted_copy():
    """S3: the mutated sequence is scored in every phase; a copy shifted by one base aligns with
    phase 1 of pattern '10' (its included bases are the original's phase-0 bases)."""
    rng = np.random.default_rng(6)
    seq = synth.random_acgt(rng, 600)
    shifted = np.concatenate([b("A"), seq[:-1]])
    ed, mm, tt, ph = oracle.harness_pairs(seq, shifted, np.array([0, 600], np.uint64), 13, 9, "10")
    assert ph[0] == 1 and mm[0, 3] >= tt[0, 3] - 2
    assert _rate(seq, shifted, 3, 13, 9, "10", 0)[0] < mm[0, 3]
    assert ed[0] == 2  # one insertion at the start, one deletion at the end


def test_accepted_pairs_no_false_negatives_and_trend():
    o, m, off, subs = synth.mutation_pairs(120, 1000, 300, 11)
    ed, mm, tt, _ = oracle.harness_pairs(o, m, off, 8, 6, "10")
    for E in (0, 20, 138, 295, int(ed.max())):
        acc = oracle.accepted_pairs(ed, mm, tt, E)
        for a in range(4):
            rated = tt[:, a] > 0
            # every rated pair within the edit threshold is accepted ("none of them reject a
            # sequence pair whose edit distance is less than or equal to the target threshold")
            assert acc[a] >= int((rated & (ed <= E)).sum())
        if E == int(ed.max()):
            assert acc.tolist() == [int((tt[:, a] > 0).sum()) for a in range(4)]
    # the matching rate falls with the edit distance ("inversely proportional")
    for a in (0, 1, 3):
        r = mm[:, a] / np.maximum(tt[:, a], 1)
        lo, hi = r[ed <= np.percentile(ed, 25)].mean(), r[ed >= np.percentile(ed, 75)].mean()
        assert lo > hi


def test_mutation_pairs_generator():
    """S1 inputs: the mutated copy differs from the original at exactly n_subs positions, every
    difference a substitution to another base; same seed, same pairs."""
    o, m, off, subs = synth.mutation_pairs(50, 400, 120, 3)
    assert off[-1] == 50 * 400 and set(np.unique(o).tolist()) <= set(b"ACGT")
    for i in range(50):
        a, c = o[int(off[i]):int(off[i + 1])], m[int(off[i]):int(off[i + 1])]
        assert int((a != c).sum()) == int(subs[i]) <= 120
    o2, m2, _, s2 = synth.mutation_pairs(50, 400, 120, 3)
    assert np.array_equal(o, o2) and np.array_equal(m, m2) and np.array_equal(subs, s2)
