"""GPU parity of desk-scale containment search (-m gpu): god_contain (CUDA, through the C ABI)
against the oracle's or_contain (readings C1-C4), bit-exact per reference sequence: mapped reads,
mapped bases and the accept flag.  A RefSeq-like set of many contigs (shared segments between
some), reads simulated from a subset of them, several patterns, batch sizes ("-I"),
thresholds, and the host-pointer path."""
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


def _contigs(seed, n=40):
    rng = np.random.default_rng(seed)
    cs = [synth.iid_genome(int(rng.integers(5_000, 40_000)), seed * 100 + i) for i in range(n)]
    for i in range(0, n - 1, 7):  # shared segments: contig i+1 carries a copy of part of contig i
        L = min(3000, cs[i].size, cs[i + 1].size)
        cs[i + 1][:L] = cs[i][:L]
    return cs


def _reads_from(cs, present, seed, n_per, **kw):
    seqs = []
    for j, i in enumerate(present):
        rd = synth.simulate_reads(cs[i], n_per, seed + j, **kw)
        seqs += [rd.seq[int(rd.offsets[q]):int(rd.offsets[q + 1])] for q in range(rd.n)]
    return synth.concat(seqs)


def _parity(refs, ro, reads, qo, pattern, k, w, host=False, **kw):
    want = oracle.contain(refs, ro, reads, qo, pattern, k, w, **kw)
    okw = dict(kw)
    if "max_occ" in okw and okw["max_occ"] < 0:
        okw.pop("max_occ")
    if host:
        got = god.god_contain(refs, ro, reads, qo, pattern, k, w, **okw)
    else:
        got = [x.cpu().numpy() for x in god.god_contain(cu(refs), cu(ro), cu(reads), cu(qo), pattern, k, w, **okw)]
    for g, o, name in zip(got, want, ("mapped_reads", "mapped_bases", "accepted")):
        assert np.array_equal(np.asarray(g), o), (name, np.flatnonzero(np.asarray(g) != o)[:10])
    return want


@pytest.mark.parametrize("pattern,k,w", [("10", 21, 11), ("110", 19, 16), ("1", 15, 10)])
def test_contain_parity_short_reads(pattern, k, w):
    cs = _contigs(7)
    refs, ro = synth.concat(cs)
    present = [0, 1, 5, 12, 13, 30]
    reads, qo = _reads_from(cs, present, 50, 60, length=150, p_sub=0.002, p_ins=0.0005, p_del=0.0005)
    mr, mb, acc = _parity(refs, ro, reads, qo, pattern, k, w, min_reads=20, cov=(1, 10))
    assert all(acc[i] for i in present) and mr[present].min() >= 50
    for I in (60_000, 200_000):
        _parity(refs, ro, reads, qo, pattern, k, w, batch_bases=I, min_reads=20, cov=(1, 10))
    _parity(refs, ro, reads, qo, pattern, k, w, min_reads=0, cov=(0, 1), V=1, max_pairs=2, D=40)


def test_contain_parity_long_reads_and_host_path():
    cs = _contigs(11, n=25)
    refs, ro = synth.concat(cs)
    present = [2, 3, 17]
    reads, qo = _reads_from(cs, present, 70, 25, mu=8.0, sigma=0.5, lmin=500, lmax=8000, p_sub=0.01, p_ins=0.005,
                            p_del=0.005)
    _parity(refs, ro, reads, qo, "10", 19, 19, min_reads=5, cov=(1, 4), max_occ=200)
    _parity(refs, ro, reads, qo, "10", 19, 19, min_reads=5, cov=(1, 4), batch_bases=50_000, host=True)
