"""GPU parity of the seed-comparison harness (-m gpu): god_seed_harness (CUDA, through the C ABI)
against the oracle (readings S1-S5), bit-exact per pair: edit distance, matches and totals
of the four extractors, and the Genome-on-Diet phase.  Every (k, w, pattern) of the paper's
section 2.1.1, pairs with 0..300 substitutions, plus N bytes, lowercase, shifted copies,
ragged lengths up to the 4096-base limit, the host path and the length error."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2211_08157_b200 as god  # noqa: E402

PAPER_CONFIGS = [(8, 6, "110"), (8, 6, "10"), (8, 6, "101001"), (8, 6, "100"), (13, 9, "10"),
                 (13, 9, "1110110110111"), (18, 12, "10"), (18, 12, "111001011001010111"), (21, 11, "10"),
                 (21, 11, "111101101101011101111")]


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    return True


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _parity(o, m, off, k, w, pat, host=False):
    want = oracle.harness_pairs(o, m, off, k, w, pat)
    got = god.god_seed_harness(o, m, off, pat, k, w) if host else \
        [x.cpu().numpy() for x in god.god_seed_harness(cu(o), cu(m), cu(off), pat, k, w)]
    for g, x, name in zip(got, want, ("edit", "matches", "totals", "god_phase")):
        g = np.asarray(g)
        if not np.array_equal(g, x):
            bad = np.flatnonzero((g != x).reshape(len(off) - 1, -1).any(axis=1))[:5]
            raise AssertionError(f"{name} differs for pairs {bad}: got {g[bad]} want {x[bad]}")
    return want


@pytest.mark.parametrize("k,w,pat", PAPER_CONFIGS, ids=[f"k{c[0]}-w{c[1]}-{c[2]}" for c in PAPER_CONFIGS])
def test_harness_parity_paper_configs(k, w, pat):
    o, m, off, subs = synth.mutation_pairs(80, 1000, 300, 100 + k + len(pat))
    ed, mm, tt, _ = _parity(o, m, off, k, w, pat)
    assert (ed <= subs).all()


def test_harness_edge_pairs_and_host_path():
    rng = np.random.default_rng(8)
    pairs = []
    for L in (0, 1, 7, 20, 64, 65, 1000, 4095, 4096):
        a = synth.random_acgt(rng, L, 0.0)
        c = a.copy()
        if L > 10:
            c[rng.choice(L, L // 10, replace=False)] = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, L // 10)]
        pairs.append((a, c))
    base = synth.random_acgt(rng, 800)
    pairs.append((base, np.concatenate([np.frombuffer(b"A", np.uint8), base[:-1]])))  # shifted copy
    with_n = base.copy()
    with_n[100:104] = ord("N")
    pairs.append((base, with_n))                                                     # N bytes
    low = base.copy()
    low[::7] = np.frombuffer(base[::7].tobytes().lower(), np.uint8)
    pairs.append((base, low))                                                        # lowercase
    pairs.append((np.frombuffer(b"ACGT" * 200, np.uint8).copy(), np.frombuffer(b"AAAA" * 200, np.uint8).copy()))
    o = np.concatenate([p[0] for p in pairs])
    m = np.concatenate([p[1] for p in pairs])
    off = np.concatenate([[0], np.cumsum([p[0].size for p in pairs])]).astype(np.uint64)
    for k, w, pat in [(8, 6, "10"), (13, 9, "1110110110111"), (21, 11, "10"), (16, 5, "1")]:
        _parity(o, m, off, k, w, pat)
    _parity(o, m, off, 13, 9, "110", host=True)
    big = synth.random_acgt(rng, 4097)
    with pytest.raises(god.GodError):
        god.god_seed_harness(cu(big), cu(big), cu(np.array([0, 4097], np.uint64)), "10", 8, 6)


def test_harness_accepted_pairs():
    o, m, off, _ = synth.mutation_pairs(300, 1000, 300, 77)
    for k, w, pat in [(8, 6, "100"), (21, 11, "10")]:
        ed, mm, tt, _ = god.god_seed_harness(cu(o), cu(m), cu(off), pat, k, w)
        E = np.array([0, 20, 138, 295, 1000], np.uint64)
        got = god.god_harness_accepted(ed, mm, tt, cu(E)).cpu().numpy()
        oed, omm, ott, _ = oracle.harness_pairs(o, m, off, k, w, pat)
        want = np.stack([oracle.accepted_pairs(oed, omm, ott, int(e)) for e in E])
        assert np.array_equal(got, want.astype(np.uint64)), (got, want)
