"""GPU parity of location voting (-m gpu): god_vote_reads (CUDA, through the C ABI) against the
oracle's or_vote_reads_batch (Fig. 8, rescue P:398; readings V1-V6), bit-exact on every
field and in output order.  Covers every kernel path (<= 16 / 32 anchors per read: registers;
<= 128 / 512: a warp on a shared-memory slice; <= 2048: a CTA in shared memory; larger: a CTA on
global scratch), repeated seeds on one diagonal (V2), both strands, D / V / max_pairs variants,
reads without anchors, the host-pointer path and the inconsistent-phase error."""
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


def _as_oracle(v):
    out = np.zeros(v.size, oracle.VOTE_DTYPE)
    for f in oracle.VOTE_DTYPE.names:
        out[f] = v[f]
    return out


def _vote_parity(ix, ox, reads, roffs, D=0, V=3, max_pairs=0, t=16, phases=None):
    """GPU: seed (SELECT, or GIVEN with `phases`) -> vote.  Oracle: its own seeding's phases -> vote."""
    an, ao, ph = god.god_seed_reads(ix, cu(reads), cu(roffs), phases=None if phases is None else cu(phases), t=t)
    v, vo = god.god_vote_reads(ix, cu(reads), cu(roffs), ph, an, ao, D=D, V=V, max_pairs=max_pairs)
    got = _as_oracle(god.votes_numpy(v))
    vo = vo.cpu().numpy()
    if phases is None:
        _, _, oph = ox.seed_reads(reads, roffs, t=t)
        assert np.array_equal(ph.cpu().numpy(), oph)
    else:
        oph = phases
    want, wo = ox.vote_reads(reads, roffs, oph, D=D, V=V, max_pairs=max_pairs)
    assert np.array_equal(vo, wo), np.flatnonzero(vo != wo)[:10]
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)[:5]
        raise AssertionError(f"vote mismatch at {bad}: got {got[bad]} want {want[bad]}")
    return got, vo, (an, ao, ph)


def test_vote_parity_tiny_config():
    cfg = synth.make_config("tiny")
    ix = god.god_build_index(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    got, vo, _ = _vote_parity(ix, ox, cfg.reads.seq, cfg.reads.offsets)
    # error-light reads from an i.i.d. reference: nearly every read votes its origin with >= V votes
    assert (got["rescued"] == 0).sum() > 0.95 * (len(vo) - 1)
    for D, V, mp in [(20, 1, 1), (150, 5, 2), (0, 0, 0), (1, 2, 3)]:
        _vote_parity(ix, ox, cfg.reads.seq, cfg.reads.offsets, D=D, V=V, max_pairs=mp)


@pytest.mark.parametrize("pattern,k,w", [("10", 15, 10), ("110", 13, 7), ("1", 11, 5)])
def test_vote_parity_repeats_long_reads(pattern, k, w):
    """Repeat-rich reference (a 2 kbp element x 300, a tandem 8-mer array, duplicated segments) and
    mixed read lengths: reads with thousands of anchors (global-scratch path), many clusters,
    tandem repeats (repeated hashes on one diagonal)."""
    rng = np.random.default_rng(29)
    base = synth.dup_genome(300_000, 13, dup_frac=0.2, lmin=300, lmax=2000)
    rep = synth.random_acgt(rng, 2000)
    tandem = np.frombuffer(b"ACGTTGCA" * 500, np.uint8)
    ref = np.concatenate([base] + [rep] * 300 + [tandem])
    roffs_ref = np.array([0, base.size, ref.size], np.uint64)
    reads = synth.simulate_reads(ref, 400, 7, mu=7.0, sigma=1.0, lmin=50, lmax=8000, p_sub=0.005, p_ins=0.002,
                                 p_del=0.002)
    seqs = [reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in range(reads.n)]
    seqs += [np.zeros(0, np.uint8), np.frombuffer(b"N" * 300, np.uint8), rep[:1500].copy(), rep.copy(),
             tandem[:600].copy(), synth.random_acgt(rng, 5000), np.frombuffer(b"ACGTAC", np.uint8)]
    rs, ro = synth.concat(seqs)
    ix = god.god_build_index(cu(ref), cu(roffs_ref), pattern, k, w, max_occ=400)
    ox = oracle.Index(ref, roffs_ref, pattern, k, w, max_occ=400)
    got, vo, (an, ao, _) = _vote_parity(ix, ox, rs, ro)
    per_read = np.diff(ao.cpu().numpy())
    # every kernel path: <= 16, <= 32 (registers), <= 128, <= 512 (warp + SMEM), <= 2048 (CTA), more
    if pattern != "1":  # ('1', 11, 5) gives almost every read > 32 anchors
        for lo, hi in [(0, 16), (16, 32), (32, 128), (128, 512), (512, 2048), (2048, 1 << 40)]:
            assert ((per_read > lo) & (per_read <= hi)).any(), (lo, hi)
    for D, V, mp in [(50, 2, 4), (500, 1, 0), (0, 10, 1)]:
        _vote_parity(ix, ox, rs, ro, D=D, V=V, max_pairs=mp)


def test_vote_given_phases_and_host_path():
    cfg = synth.make_config("tiny")
    ix = god.god_build_index(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    n = 2000
    sub, soffs = synth.concat([cfg.reads.seq[int(cfg.reads.offsets[i]):int(cfg.reads.offsets[i + 1])]
                               for i in range(n)])
    ph = (np.arange(n) % 2).astype(np.uint8)
    _vote_parity(ix, ox, sub, soffs, phases=ph, V=1)
    # host buffers through the same ABI call
    an, ao, gph = god.god_seed_reads(ix, sub, soffs)
    v, vo = god.god_vote_reads(ix, sub, soffs, gph, an, ao, V=3, max_pairs=2)
    want, wo = ox.vote_reads(sub, soffs, gph, V=3, max_pairs=2)
    assert np.array_equal(vo, wo) and np.array_equal(_as_oracle(god.votes_numpy(v)), want)


def test_vote_rejects_inconsistent_phases():
    cfg = synth.make_config("tiny")
    ix = god.god_build_index(cu(cfg.ref), cu(cfg.ref_offsets), "10", 21, 11)
    n = 500
    sub, soffs = synth.concat([cfg.reads.seq[int(cfg.reads.offsets[i]):int(cfg.reads.offsets[i + 1])]
                               for i in range(n)])
    an, ao, ph = god.god_seed_reads(ix, cu(sub), cu(soffs))
    with pytest.raises(god.GodError):
        god.god_vote_reads(ix, cu(sub), cu(soffs), (1 - ph).contiguous(), an, ao)
