"""Whole-config bit-exact parity (-m gpu) on every BASELINE.json config/pattern row, by digest.

`north_star`: "bit-exact agreement with the CPU oracle on all five configs" ("for the same
input sequence and the same input parameters, both implementations return the same list of
minimizers").  The oracle cannot run inside GPU test time at human scale, so
`tools/oracle_digests.py` (imports only oracle/ and synth/) ran it once over ALL inputs of each
row and stored the sha256 of each canonical dump under tests/golden/digests/ (SURVEY §8(c) O10:
"streaming sha256 with chunk localisation on mismatch").  This test runs the CUDA path through the
C ABI in the launch configuration bench.py times (device-resident inputs, the whole reference in
one god_build_index, all reads in one SELECT-mode god_seed_reads) and rebuilds the same canonical
bytes from the GPU outputs — its own packing code, nothing shared with the oracle script — then
compares every digest.  A mismatch names the first differing chunk of CHUNK records.

Rows: tiny '10', illumina '10', hifi '10'/'110', ont '10', human '10'/'110'/'1110'/'1'.
Results go to gpurun_out/parity_digests.jsonl (BASELINE.md's "Bit-exact" column is generated
from it by tools/measure_table.py)."""
import hashlib
import json
import os
import time

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import paper_2211_08157_b200 as god  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "digests")
ROWS = [("tiny", "10"), ("illumina", "10"), ("hifi", "10"), ("hifi", "110"), ("ont", "10"),
        ("human", "10"), ("human", "110"), ("human", "1110"), ("human", "1")]
LOG = os.environ.get("GOD_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_digests.jsonl"))


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    return True


class Sha:
    """Streaming sha256 over fixed-width records + one sha256 per `chunk` records."""

    def __init__(self, chunk):
        self.chunk, self.h, self.c, self.in_c, self.n, self.chunks = chunk, hashlib.sha256(), hashlib.sha256(), 0, 0, []

    def feed(self, b: bytes, nrec: int, rec_size: int):
        off = 0
        while nrec:
            take = min(self.chunk - self.in_c, nrec)
            piece = b[off:off + take * rec_size]
            self.h.update(piece)
            self.c.update(piece)
            off += take * rec_size
            nrec -= take
            self.n += take
            self.in_c += take
            if self.in_c == self.chunk:
                self.chunks.append(self.c.hexdigest())
                self.c, self.in_c = hashlib.sha256(), 0

    def done(self):
        if self.in_c:
            self.chunks.append(self.c.hexdigest())
            self.in_c = 0
        return self


def host(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def sha_array(a, chunk):
    a = np.ascontiguousarray(a)
    s = Sha(chunk)
    s.feed(memoryview(a.view(np.uint8).reshape(-1)), a.size, a.itemsize)
    return s.done()


def sha_records17(h, p, z, chunk):
    """(hash u64, pos -> u64, strand u8) as 17-byte little-endian records, built chunk by chunk."""
    n = int(h.shape[0])
    s = Sha(chunk)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        buf = np.empty((b - a, 17), np.uint8)
        buf[:, 0:8] = host(h[a:b]).astype("<u8").view(np.uint8).reshape(-1, 8)
        buf[:, 8:16] = host(p[a:b]).astype("<u8").view(np.uint8).reshape(-1, 8)
        buf[:, 16] = host(z[a:b]).astype(np.uint8)
        s.feed(buf.tobytes(), b - a, 17)
    return s.done()


def sha_anchors(an, chunk):
    """GPU anchors (n, 4) u32 = (ref_pos, read_pos, read_id, strand) -> canonical order
    (read_id, ref_pos, read_pos, strand) as 16-byte records (two stable sorts on the device)."""
    n = int(an.shape[0])
    s = Sha(chunk)
    if n == 0:
        return s.done()
    a64 = an.to(torch.int64)
    k2 = (a64[:, 1] << 1) | a64[:, 3]
    perm = torch.sort(k2, stable=True).indices
    k1 = (a64[:, 2] << 32) | a64[:, 0]
    perm = perm[torch.sort(k1[perm], stable=True).indices]
    del k1, k2
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        rows = a64[perm[a:b]]
        rec = torch.stack([rows[:, 2], rows[:, 0], rows[:, 1], rows[:, 3]], dim=1).to(torch.int32)
        s.feed(rec.cpu().numpy().astype("<u4").tobytes(), b - a, 16)
    return s.done()


def compare(name, got: Sha, want: dict, failures: list):
    if got.h.hexdigest() == want["sha256"] and got.n == want["n"]:
        return True
    first = next((i for i, (x, y) in enumerate(zip(got.chunks, want["chunks"])) if x != y),
                 min(len(got.chunks), len(want["chunks"])))
    failures.append(f"{name}: n {got.n} vs oracle {want['n']}; first differing chunk {first} "
                    f"(records {first * want['chunk_records']}..{(first + 1) * want['chunk_records'] - 1})")
    return False


def _log(rec):
    try:
        os.makedirs(os.path.dirname(LOG), exist_ok=True)
        with open(LOG, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass


@pytest.mark.parametrize("config,pattern", ROWS, ids=[f"{c}-{p}" for c, p in ROWS])
def test_digest_parity(config, pattern):
    path = os.path.join(GOLD, f"{config}_{pattern}.json")
    assert os.path.exists(path), f"missing oracle digests {path} (tools/oracle_digests.py)"
    gold = json.load(open(path))
    D = gold["digests"]
    chunk = D["anchors"]["chunk_records"]
    t0 = time.time()
    cfg = synth.make_config(config)
    ref, roff, reads = cfg.ref, cfg.ref_offsets, cfg.reads
    # the inputs must be the ones the oracle saw (generator determinism across hosts)
    assert hashlib.sha256(ref.tobytes()).hexdigest() == gold["inputs"]["ref_sha256"]
    assert hashlib.sha256(reads.seq.tobytes()).hexdigest() == gold["inputs"]["reads_sha256"]
    k, w = gold["k"], gold["w"]
    assert (k, w) == (cfg.k, cfg.w)
    fails, done = [], []

    def check(name, sha):
        if compare(name, sha, D[name], fails):
            done.append(name)

    dref, droff = torch.from_numpy(ref).cuda(), torch.from_numpy(roff).cuda()
    # stage 1: the sparsified reference
    packed, nmask, oo, cnt = god.god_sparsify(dref, droff, pattern)
    check("ref_sparsify.packed", sha_array(host(packed), chunk))
    check("ref_sparsify.nmask", sha_array(host(nmask), chunk))
    check("ref_sparsify.counts", sha_array(host(cnt), chunk))
    del packed, nmask, oo, cnt
    # stage 2: reference minimizers (position order, global positions)
    h, p, z, mo = god.god_minimizers(dref, droff, pattern, k, w, global_pos=True)
    check("ref_minimizers", sha_records17(h, p, z, chunk))
    check("ref_minimizers.offsets", sha_array(host(mo), chunk))
    del h, p, z, mo
    torch.cuda.empty_cache()
    # stage 3: the index, exactly as bench.py builds it
    ix = god.god_build_index(dref, droff, pattern, k, w, cutoff=tuple(gold["cutoff"]))
    st = ix.stats()
    for f, v in gold["index_stats"].items():
        if st[f] != v:
            fails.append(f"index_stats.{f}: {st[f]} vs oracle {v}")
    h, p, z = ix.dump(device=True)
    check("index_dump", sha_records17(h, p, z, chunk))
    del h, p, z
    torch.cuda.empty_cache()
    # stage 4: SELECT-mode phase selection + seeding of ALL reads in one call (bench.py's launch)
    dreads, droffs = torch.from_numpy(reads.seq).cuda(), torch.from_numpy(reads.offsets).cuda()
    an, ao, ph = god.god_seed_reads(ix, dreads, droffs, t=gold["t"])
    check("phases", sha_array(host(ph), chunk))
    check("anchor_counts", sha_array(np.diff(host(ao)).astype("<u8"), chunk))
    check("anchors", sha_anchors(an, chunk))
    del an, ao
    torch.cuda.empty_cache()
    # stage 1 for the reads at their selected phases
    packed, nmask, oo, cnt = god.god_sparsify(dreads, droffs, pattern, phases=ph)
    check("read_sparsify.packed", sha_array(host(packed), chunk))
    check("read_sparsify.nmask", sha_array(host(nmask), chunk))
    check("read_sparsify.counts", sha_array(host(cnt), chunk))
    ix.free()
    missing = sorted(set(D) - set(done) - {f.split(":")[0] for f in fails})
    ok = not fails and not missing
    _log({"config": config, "pattern": pattern, "bit_exact": ok, "compared": sorted(done), "failures": fails,
          "index_stats": st if isinstance(st, dict) else None, "n_anchors": gold["n_anchors"],
          "n_reads": gold["n_reads"], "ref_bp": gold["ref_bp"], "seconds": round(time.time() - t0, 1)})
    assert not missing, f"digests not compared: {missing}"
    assert not fails, "; ".join(fails)


@pytest.mark.parametrize("config,pattern", [("tiny", "10"), ("human", "10")], ids=["tiny-10", "human-10"])
def test_digest_parity_host_call(config, pattern):
    """The e2e launch configuration bench.py times: pinned HOST buffers through ONE
    god_build_index_and_seed call (reference streamed up under K1, read batches queued behind it,
    8-byte anchors streamed back).  The index dump, the SELECT phases, the anchor counts and the
    canonically sorted anchors of all reads against the same oracle digests."""
    gold = json.load(open(os.path.join(GOLD, f"{config}_{pattern}.json")))
    D = gold["digests"]
    chunk = D["anchors"]["chunk_records"]
    t0 = time.time()
    cfg = synth.make_config(config)
    assert hashlib.sha256(cfg.ref.tobytes()).hexdigest() == gold["inputs"]["ref_sha256"]
    assert hashlib.sha256(cfg.reads.seq.tobytes()).hexdigest() == gold["inputs"]["reads_sha256"]
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    ref, roff, rs, ro = pin(cfg.ref), pin(cfg.ref_offsets), pin(cfg.reads.seq), pin(cfg.reads.offsets)
    fails, done = [], []

    def check(name, sha):
        if compare(name, sha, D[name], fails):
            done.append(name)

    ix, an, ao, ph = god.god_build_index_and_seed(ref, roff, rs, ro, pattern, gold["k"], gold["w"],
                                                  cutoff=tuple(gold["cutoff"]), t=gold["t"], compact=True,
                                                  cap=gold["n_anchors"] + 1024)
    st = ix.stats()
    for f, v in gold["index_stats"].items():
        if st[f] != v:
            fails.append(f"index_stats.{f}: {st[f]} vs oracle {v}")
    h, p, z = ix.dump(device=True)
    check("index_dump", sha_records17(h, p, z, chunk))
    del h, p, z
    ix.free()
    torch.cuda.empty_cache()
    check("phases", sha_array(np.asarray(ph), chunk))
    cnts = np.diff(np.asarray(ao)).astype("<u8")
    check("anchor_counts", sha_array(cnts, chunk))
    # 8-B anchors -> (ref_pos, read_pos, read_id, strand) on the device (read id = the anchor's segment)
    c = torch.from_numpy(np.ascontiguousarray(an).view(np.uint32).reshape(-1, 2).astype(np.int64)).cuda()
    rid = torch.repeat_interleave(torch.arange(cnts.size, device="cuda"), torch.from_numpy(cnts.astype(np.int64)).cuda())
    full = torch.stack([c[:, 0], c[:, 1] & 0x7FFFFFFF, rid, c[:, 1] >> 31], dim=1)
    del c, rid
    check("anchors", sha_anchors(full, chunk))
    _log({"config": config, "pattern": pattern, "call": "god_build_index_and_seed (host buffers)", "bit_exact": not fails,
          "compared": sorted(done), "failures": fails, "seconds": round(time.time() - t0, 1)})
    assert not fails, "; ".join(fails)
    assert sorted(done) == ["anchor_counts", "anchors", "index_dump", "phases"]
