"""GPU parity at BASELINE.json's full sizes (-m gpu), in the launch configuration bench.py times.

configs[1..3] (100 Mbp reference): the whole index is compared with the oracle's; reads are seeded
on the GPU in one batch and a seeded sample of them is compared read by read with the oracle
(phases and canonically sorted anchors).  configs[4] (3.1 Gbp): the oracle cannot index the whole
genome in test time, so the GPU output is checked on sampled outputs and by properties that hold
at any size: minimizers of sampled windows, index counts per hash, the cutoff rule (tau) recomputed
independently from all minimizer hashes, and the exact-substring invariant of error-free reads."""
import numpy as np
import pytest

import oracle
import synth
from brute import revcomp, true_phases

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2211_08157_b200 as god  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def canon(a):
    a = np.asarray(a).reshape(-1, 4)
    rec = np.zeros(a.shape[0], oracle.ANCHOR_DTYPE)
    rec["ref_pos"], rec["read_pos"], rec["read_id"], rec["strand"] = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    return np.sort(rec, order=["read_id", "ref_pos", "read_pos", "strand"])


def _sampled_seed_parity(ix, ox, cfg, n_sample, seed):
    reads = cfg.reads
    an, ao, ph = god.god_seed_reads(ix, cu(reads.seq), cu(reads.offsets))
    an, ao, ph = an.cpu().numpy(), ao.cpu().numpy(), ph.cpu().numpy()
    rng = np.random.default_rng(seed)
    ids = np.sort(rng.choice(reads.n, size=min(n_sample, reads.n), replace=False))
    sub, soff = synth.concat([reads.seq[int(reads.offsets[i]):int(reads.offsets[i + 1])] for i in ids])
    oan, oao, oph = ox.seed_reads(sub, soff)
    assert np.array_equal(ph[ids], oph)
    assert np.array_equal(ao[ids + 1] - ao[ids], np.diff(oao))
    g = canon(np.concatenate([an[int(ao[i]):int(ao[i + 1])] for i in ids]))
    remap = np.zeros(reads.n, np.uint32)
    remap[ids] = np.arange(ids.size, dtype=np.uint32)
    g["read_id"] = remap[g["read_id"]]
    g = np.sort(g, order=["read_id", "ref_pos", "read_pos", "strand"])
    assert np.array_equal(g, np.sort(oan, order=["read_id", "ref_pos", "read_pos", "strand"]))
    return an, ao, ph, ids, sub, soff, oph


def _sampled_vote_parity(ix, ox, cfg, seeded, D, V, max_pairs):
    """Location voting of ALL reads on the GPU (the launch configuration bench.py times), compared
    on the sampled reads with the oracle's voting of the same reads."""
    an, ao, ph, ids, sub, soff, oph = seeded
    reads = cfg.reads
    v, vo = god.god_vote_reads(ix, cu(reads.seq), cu(reads.offsets), cu(ph), cu(an), cu(ao), D=D, V=V,
                               max_pairs=max_pairs)
    gv, vo = god.votes_numpy(v), vo.cpu().numpy()
    want, wo = ox.vote_reads(sub, soff, oph, D=D, V=V, max_pairs=max_pairs)
    assert np.array_equal(vo[ids + 1] - vo[ids], np.diff(wo))
    got = np.concatenate([gv[int(vo[i]):int(vo[i + 1])] for i in ids]) if ids.size else gv[:0]
    remap = np.zeros(reads.n, np.uint32)
    remap[ids] = np.arange(ids.size, dtype=np.uint32)
    got = got.copy()
    got["read_id"] = remap[got["read_id"]]
    for f in oracle.VOTE_DTYPE.names:
        assert np.array_equal(got[f], want[f]), f


@pytest.mark.parametrize("name,pattern,n_sample", [("illumina", "10", 3000), ("hifi", "10", 40), ("hifi", "110", 30),
                                                   ("ont", "10", 40)])
def test_fullsize_configs_2_to_4(name, pattern, n_sample):
    cfg = synth.make_config(name)
    k, w = cfg.k, cfg.w
    ix = god.god_build_index(cu(cfg.ref), cu(cfg.ref_offsets), pattern, k, w)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, pattern, k, w)
    st, ost = ix.stats(), ox.stats()
    for f in oracle.STATS_FIELDS:
        assert st[f] == ost[f], (f, st[f], ost[f])
    h, p, z = ix.dump()
    oh, op, oz = ox.dump()
    assert np.array_equal(h, oh) and np.array_equal(p.astype(np.uint64), op) and np.array_equal(z, oz)
    seeded = _sampled_seed_parity(ix, ox, cfg, n_sample, 5)
    _sampled_vote_parity(ix, ox, cfg, seeded, D=0, V=3, max_pairs=0)
    if name != "illumina":  # long reads: the Fig. 8B distance (D = 100) and a capped list
        _sampled_vote_parity(ix, ox, cfg, seeded, D=100, V=3, max_pairs=8)


def test_fullsize_human_scale_sampled_and_properties():
    cfg = synth.make_config("human")
    pattern, k, w = "10", 21, 11
    ref = cfg.ref
    dref, doff = cu(ref), cu(cfg.ref_offsets)
    ix = god.god_build_index(dref, doff, pattern, k, w)
    st = ix.stats()
    assert st["kept_entries"] + st["dropped_entries"] == st["n_entries_all"]
    assert st["kept_distinct"] + st["dropped_distinct"] == st["n_distinct_all"]
    # all reference minimizers (same kernel as the index path, position order)
    hz, pos, z, oo = god.god_minimizers(dref, doff, pattern, k, w, global_pos=True)
    assert hz.shape[0] == st["n_entries_all"]
    # (1) sampled windows: exact minimizers away from the window edges
    rng = np.random.default_rng(11)
    pos_np = None
    margin = 2 * (k + w) + 4
    for _ in range(25):
        a = int(rng.integers(0, ref.size - 60000))
        b = a + 60000
        want = oracle.minimizers(ref[a:b], pattern, 0 if a % 2 == 0 else 1, k, w, pos_base=a)
        # phase: global pattern phase 0 at reference position 0 -> local shift (-a) mod 2
        want = want[(want["pos"] >= a + margin) & (want["pos"] < b - margin)]
        lo = int(torch.searchsorted(pos.to(torch.int64), torch.tensor([a + margin], device=pos.device)).item())
        hi = int(torch.searchsorted(pos.to(torch.int64), torch.tensor([b - margin], device=pos.device)).item())
        got_h = hz[lo:hi].cpu().numpy()
        got_p = pos[lo:hi].cpu().numpy().astype(np.uint64)
        assert np.array_equal(got_p, want["pos"]) and np.array_equal(got_h, want["hash"])
    # (2) the cutoff rule recomputed independently (torch unique on every minimizer hash)
    uh, cnt = torch.unique(hz.to(torch.int64), return_counts=True)
    n = uh.numel()
    assert n == st["n_distinct_all"]
    m = n // 5000
    srt = torch.sort(cnt).values
    tau = int(srt[n - m - 1].item())
    assert (st["m"], st["tau"]) == (m, tau)
    kept = int(cnt[cnt <= tau].sum().item())
    assert st["kept_entries"] == kept
    # (3) index counts per hash == number of occurrences (kept) or 0 (dropped)
    sel = torch.randint(0, n, (20000,), device=uh.device)
    q = uh[sel]
    got = ix.count(q.to(torch.uint64)).to(torch.int64)
    want_c = torch.where(cnt[sel] <= tau, cnt[sel], torch.zeros_like(cnt[sel]))
    assert torch.equal(got, want_c)
    # (4) exact-substring invariant: error-free reads from the reference find their origin (GIVEN mode)
    reads, gs, strands = [], [], []
    for _ in range(400):
        L = 150
        g0 = int(rng.integers(0, ref.size - L))
        s = int(rng.integers(0, 2))
        r = ref[g0:g0 + L].copy()
        if s:
            r = np.frombuffer(revcomp(r.tobytes().decode()).encode(), np.uint8).copy()
        reads.append(r); gs.append(g0); strands.append(s)
    rs, ro = synth.concat(reads)
    ph = np.array([true_phases(pattern, g0, 150, s)[0] for g0, s in zip(gs, strands)], np.uint8)
    an, ao, _ = god.god_seed_reads(ix, cu(rs), cu(ro), phases=cu(ph))
    an, ao = an.cpu().numpy().reshape(-1, 4), ao.cpu().numpy()
    for i, (g0, s) in enumerate(zip(gs, strands)):
        mz = oracle.minimizers(reads[i], pattern, int(ph[i]), k, w)
        _, orig = oracle.sparsify(reads[i], pattern, int(ph[i]))
        pos2j = {int(o): j for j, o in enumerate(orig.tolist())}
        a_i = an[int(ao[i]):int(ao[i + 1])]
        occ = ix.count(np.array(mz["hash"], np.uint64)) if mz.size else np.zeros(0, np.uint32)
        for (hv, qpos, qz), c in zip(mz[["hash", "pos", "strand"]].tolist(), occ.tolist()):
            if c == 0:
                continue
            hits = a_i[a_i[:, 1] == qpos]
            assert hits.shape[0] == c
            if not s:
                assert any(int(x[0]) - qpos == g0 and int(x[3]) == 0 for x in hits)
            else:
                qend = int(orig[pos2j[qpos] + k - 1])
                assert any(int(x[0]) + qend == g0 + 149 and int(x[3]) == 1 for x in hits)
    # (5) voting: the true location of every exact read is a location with the most votes
    v, vo = god.god_vote_reads(ix, cu(rs), cu(ro), cu(ph), cu(an), cu(ao), D=0, V=3)
    gv, vo = god.votes_numpy(v), vo.cpu().numpy()
    for i, (g0, s) in enumerate(zip(gs, strands)):
        loc = gv[int(vo[i]):int(vo[i + 1])]
        if int(ao[i + 1] - ao[i]) == 0:
            assert loc.size == 0
            continue
        want_d = g0 + 149 if s else g0
        # the cluster whose [Delta0, Delta0 + D] (D = read length) holds the true diagonal
        hit = loc[(loc["strand"] == s) & (loc["diag"] <= want_d) & (want_d <= loc["diag"] + 150)]
        assert hit.size == 1 and int(hit["votes"][0]) == int(loc["votes"].max()), (i, loc[:3])
