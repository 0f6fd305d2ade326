"""Pins for the oracle's location voting (-m "not gpu"): P:312-324 (section 3.4), Fig. 8
(P:332-334), rescue.  Readings V1-V6: oracle/oracle.c, DESIGN.md §2.

Pinned by the figure captions' numbers (tests/golden/voting.json), SPEC's hand sweep, the
App. A worked example, invariants of the sweep on random hit lists, and the exact-substring
property of reads copied from an i.i.d. reference (every true anchor shares one diagonal)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from brute import revcomp, true_phases

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _libs(built):
    return built


def b(s: str) -> np.ndarray:
    return np.frombuffer(s.encode(), dtype=np.uint8).copy()


def _gold():
    return json.load(open(os.path.join(GOLD, "voting.json")))


def _check(got, expect):
    assert len(got) == len(expect), (got, expect)
    for g, e in zip(got, expect):
        assert int(g["strand"]) == e["strand"] and int(g["diag"]) == e["diag"]
        assert int(g["votes"]) == e["votes"] and int(g["rescued"]) == e["rescued"]
        if "ref" in e:
            assert [int(g["ref_lo"]), int(g["ref_hi"])] == e["ref"]
        if "read" in e:
            assert [int(g["read_lo"]), int(g["read_hi"])] == e["read"]


def test_fig8a_twelve_votes():
    """Fig. 8A: 'location 1017 receives 12 votes'."""
    f = _gold()["fig8a"]
    _check(oracle.vote_hits([tuple(h) for h in f["hits"]], f["D"], f["V"]), f["expect"])


def test_fig8b_three_subsequence_pairs():
    """Fig. 8B: D = 100, V = 3 -> [3004-7832], [10020-15000], [71303-72437] with 7, 8, 3
    votes; the list is sorted by votes; a 2-vote group fails V."""
    f = _gold()["fig8b"]
    hits = [tuple(h) for h in f["hits"]]
    _check(oracle.vote_hits(hits, f["D"], f["V"]), f["expect"])
    # the input order does not matter (step (2) sorts)
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(hits))
    _check(oracle.vote_hits([hits[i] for i in perm], f["D"], f["V"]), f["expect"])
    # max_pairs caps the winners' list ("limit the size of the list ... to a user-defined number")
    _check(oracle.vote_hits(hits, f["D"], f["V"], max_pairs=2), f["expect"][:2])


def test_spec_sweep_and_rescue():
    f = _gold()["spec_sweep"]
    hits = [tuple(h) for h in f["hits"]]
    _check(oracle.vote_hits(hits, f["D"], f["V"]), f["expect"])
    # rescue: no group reaches V -> the best group, flagged
    r = oracle.vote_hits(hits[3:], f["D"], f["V"])
    _check(r, [{"strand": 0, "diag": 500, "votes": 2, "rescued": 1}])
    # tie between two sub-threshold groups -> the smaller Delta0 (reading V4/V5)
    r = oracle.vote_hits([(1, 0, 0, 5, 5), (2, 0, 0, 6, 6), (3, 900, 0, 905, 5), (4, 901, 0, 907, 6)], 100, 3)
    _check(r, [{"strand": 0, "diag": 0, "votes": 2, "rescued": 1}])
    # no hits -> unmapped (no location)
    assert oracle.vote_hits(np.zeros(0, oracle.HIT_DTYPE), 100, 3).size == 0


def test_repeated_seeds_counted_once():
    """repeated seeds (same hash) and repeated locations count once per adjusted location."""
    hits = [(7, 100, 0, 110, 10), (7, 100, 0, 130, 30), (7, 100, 0, 150, 50), (8, 100, 0, 170, 70),
            (9, 101, 0, 171, 70)]
    r = oracle.vote_hits(hits, 50, 1)
    _check(r, [{"strand": 0, "diag": 100, "votes": 3, "rescued": 0, "ref": [110, 171], "read": [10, 70]}])
    # the same hash on the other strand or another diagonal is another vote
    r = oracle.vote_hits(hits + [(7, 100, 1, 110, 10), (7, 102, 0, 112, 10)], 50, 1)
    assert [(int(x["strand"]), int(x["votes"])) for x in r] == [(0, 4), (1, 1)]


def test_sweep_invariants_random():
    """Properties of the sweep on random hit lists: with V = 0 every cluster is
    returned; Delta0s of one strand are > D apart; each hit lies in exactly one cluster's
    [Delta0, Delta0 + D]; total votes = number of distinct (hash, strand, diag); V filters a
    subset; D = infinity gives one cluster per strand."""
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.integers(1, 60))
        D = int(rng.integers(0, 40))
        h = np.zeros(n, oracle.HIT_DTYPE)
        h["hash"] = rng.integers(0, 6, n)
        h["diag"] = rng.integers(-100, 200, n)
        h["strand"] = rng.integers(0, 2, n)
        h["ref_pos"] = rng.integers(0, 1000, n)
        h["read_pos"] = rng.integers(0, 150, n)
        allc = oracle.vote_hits(h, D, 0)
        distinct = {(int(x["hash"]), int(x["strand"]), int(x["diag"])) for x in h}
        assert int(allc["votes"].sum()) == len(distinct)
        for s in (0, 1):
            d0 = sorted(int(c["diag"]) for c in allc if c["strand"] == s)
            assert all(b_ - a_ > D for a_, b_ in zip(d0, d0[1:]))
            for x in h[h["strand"] == s]:
                own = [d for d in d0 if d <= int(x["diag"]) <= d + D]
                assert len(own) >= 1
                # the owning cluster is the last Delta0 <= diag
                assert max(d for d in d0 if d <= int(x["diag"])) in own
        # votes-descending order
        v = allc["votes"].astype(int).tolist()
        assert v == sorted(v, reverse=True)
        V = int(rng.integers(1, 5))
        sub = oracle.vote_hits(h, D, V)
        keys_all = {(int(c["strand"]), int(c["diag"]), int(c["votes"])) for c in allc}
        if (allc["votes"] >= V).any():
            assert not sub["rescued"].any()
            assert {(int(c["strand"]), int(c["diag"]), int(c["votes"])) for c in sub} == \
                {k for k in keys_all if k[2] >= V}
        else:
            assert sub.size == 1 and sub["rescued"][0] == 1 and int(sub["votes"][0]) == int(allc["votes"].max())
        one = oracle.vote_hits(h, 10**9, 0)
        assert len(one) == len(set(h["strand"].tolist()))


def test_vote_read_appendix_a():
    g = json.load(open(os.path.join(GOLD, "appendix_a.json")))
    f = _gold()["appendix_a"]
    ref = b(g["reference"])
    ix = oracle.Index(ref, np.array([0, ref.size], np.uint64), g["pattern"], g["k"], g["w"])
    for rd in f["reads"]:
        _check(ix.vote_read(b(rd["seq"]), rd["a"], V=f["V"]), rd["expect"])


def test_vote_exact_reads_share_one_diagonal():
    """Reads copied from an i.i.d. reference (P:300 premise), voted with their true phase: the best
    location is the true one — forward: Delta0 = g (= ref - read of every true anchor); reverse:
    Delta0 = g + L - 1 (= ref + read_end, O9) — with one vote per distinct read minimizer hash kept
    in the index."""
    rng = np.random.default_rng(5)
    ref = synth.iid_genome(300_000, 91)
    offs = np.array([0, ref.size], np.uint64)
    for pat, k, w in [("10", 21, 11), ("110", 19, 19), ("1", 15, 10)]:
        ix = oracle.Index(ref, offs, pat, k, w)
        for r in range(60):
            L = int(rng.integers(150, 600))
            g0 = int(rng.integers(0, ref.size - L))
            strand = int(rng.integers(0, 2))
            read = ref[g0:g0 + L].copy()
            if strand:
                read = b(revcomp(read.tobytes().decode()))
            s = true_phases(pat, g0, L, strand)[0]
            mz = oracle.minimizers(read, pat, s, k, w)
            nh = len({int(x["hash"]) for x in mz if ix.occ(int(x["hash"])) > 0})
            v = ix.vote_read(read, s, V=3)
            assert v.size >= 1
            top = v[0]
            assert int(top["strand"]) == strand
            assert int(top["diag"]) == (g0 + L - 1 if strand else g0)
            assert int(top["votes"]) == nh
            assert int(top["ref_lo"]) >= g0 and int(top["ref_hi"]) < g0 + L
