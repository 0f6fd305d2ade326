"""Pins for the oracle's containment search (-m "not gpu"): P:174-176, P:184 (mapped read = a read
that receives a location from the voting step; accept = enough mapped reads and genome coverage),
P:182/P:202 (references in batches of at most I bases, index built on the fly).  Readings C1-C4:
oracle/oracle.c, DESIGN.md §2.  Pinned by planted-source simulations (reads drawn from one of two
disjoint random references), threshold boundaries computed from the read lengths, the empty read
set, batch-independence on disjoint references and a shared segment mapping to two references."""
import numpy as np
import pytest

import oracle
import synth
from brute import revcomp

K, W, PAT = 21, 11, "10"


@pytest.fixture(scope="module", autouse=True)
def _libs(built):
    return built


def _exact_reads(ref, n, seed, L=150):
    rng = np.random.default_rng(seed)
    seqs = []
    for _ in range(n):
        g = int(rng.integers(0, ref.size - L))
        s = ref[g:g + L].copy()
        if rng.integers(0, 2):
            s = np.frombuffer(revcomp(s.tobytes().decode()).encode(), np.uint8).copy()
        seqs.append(s)
    return synth.concat(seqs)


def _refs(*seqs):
    return synth.concat(list(seqs))


def test_planted_source_accepted_other_rejected():
    A, B = synth.iid_genome(200_000, 301), synth.iid_genome(150_000, 302)
    refs, ro = _refs(A, B)
    reads, qo = _exact_reads(A, 400, 7)
    mr, mb, acc = oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=100, cov=(1, 10))
    assert mr.tolist() == [400, 0]                  # every exact read votes a location in A, none in B
    assert int(mb[0]) == int(qo[-1]) and int(mb[1]) == 0
    assert acc.tolist() == [1, 0]
    # boundary of the coverage rule: mapped_bases * den >= num * len(A)
    assert oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=1, cov=(int(mb[0]), A.size))[2][0] == 1
    assert oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=1, cov=(int(mb[0]) + 1, A.size))[2][0] == 0
    # boundary of the read-count rule
    assert oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=400, cov=(0, 1))[2][0] == 1
    assert oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=401, cov=(0, 1))[2][0] == 0
    # zero thresholds accept everything; an empty read set maps nothing
    assert oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=0, cov=(0, 1))[2].tolist() == [1, 1]
    e, eo = synth.concat([])
    mr0, mb0, acc0 = oracle.contain(refs, ro, e, eo, PAT, K, W, min_reads=1, cov=(1, 10))
    assert mr0.tolist() == [0, 0] and mb0.tolist() == [0, 0] and acc0.tolist() == [0, 0]


def test_batches_and_shared_segments():
    """C1: one batch per reference gives the same stats as one batch when the references share no
    seed; a segment copied into two references maps its reads to both (sum of mapped reads over
    references >= reads mapped anywhere)."""
    A, B, C = synth.iid_genome(120_000, 311), synth.iid_genome(100_000, 312), synth.iid_genome(80_000, 313)
    refs, ro = _refs(A, B, C)
    ra, ra_o = _exact_reads(A, 150, 1)
    rc, rc_o = _exact_reads(C, 150, 2)
    reads, qo = synth.concat([ra[int(ra_o[i]):int(ra_o[i + 1])] for i in range(150)] +
                             [rc[int(rc_o[i]):int(rc_o[i + 1])] for i in range(150)])
    one = oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=50, cov=(1, 10))
    for I in (1, 130_000, 220_000):
        got = oracle.contain(refs, ro, reads, qo, PAT, K, W, min_reads=50, cov=(1, 10), batch_bases=I)
        assert all(np.array_equal(x, y) for x, y in zip(one, got)), I
    assert one[0].tolist() == [150, 0, 150] and one[2].tolist() == [1, 0, 1]
    # D2 = B with A's first 20 kbp pasted in: reads from that segment map to A and D2
    D2 = B.copy()
    D2[10_000:30_000] = A[:20_000]
    refs2, ro2 = _refs(A, D2)
    seg, so = _exact_reads(A[:20_000], 100, 3)
    mr, mb, _ = oracle.contain(refs2, ro2, seg, so, PAT, K, W, min_reads=1, cov=(0, 1))
    assert mr.tolist() == [100, 100] and mb.tolist() == [int(so[-1])] * 2
    assert int(mr.sum()) >= 100
