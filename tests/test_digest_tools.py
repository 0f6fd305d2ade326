"""CPU tests (-m "not gpu") of the digest tooling behind tests/test_gpu_digests.py.

- tools/oracle_digests.py's vectorised O10 packing equals a per-base loop (god.h stage-1 layout);
- its chunked sha256 equals the plain sha256 of the bytes, chunk by chunk;
- the GPU test's independent digest code produces the same digests from the same records (the
  two sides agree on the canonical byte format without sharing code);
- the committed tiny-config golden file is reproduced by the committed oracle + generator."""
import hashlib
import importlib.util
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name, path):
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def od(built):
    return _load("oracle_digests", os.path.join(ROOT, "tools", "oracle_digests.py"))


def naive_pack(codes, counts):
    words, nms, q = [], [], 0
    for n in counts.tolist():
        c = codes[q:q + n]
        q += n
        for wi in range((n + 31) // 32):
            word = nm = 0
            for b in range(32):
                j = wi * 32 + b
                if j >= n:
                    break
                if c[j] == 4:
                    nm |= 1 << b
                else:
                    word |= int(c[j]) << (2 * b)
            words.append(word)
            nms.append(nm)
    return np.array(words, np.uint64), np.array(nms, np.uint64)


def test_pack_codes_matches_per_base_loop(od):
    rng = np.random.default_rng(3)
    counts = np.array([0, 1, 31, 32, 33, 64, 100, 0, 257, 5], np.uint64)
    codes = rng.integers(0, 5, size=int(counts.sum())).astype(np.uint8)
    p, m = od.pack_codes(codes, counts)
    wp, wm = naive_pack(codes, counts)
    assert np.array_equal(p, wp) and np.array_equal(m, wm)
    # a long single sequence crosses the tool's piece boundary
    big = rng.integers(0, 5, size=(1 << 24) + 77).astype(np.uint8)
    p, m = od.pack_codes(big, np.array([big.size], np.uint64))
    tail = np.array([big.size - 77 - 31 * 32], np.int64)
    sl = big[int(tail[0]):]
    wp, wm = naive_pack(sl, np.array([sl.size], np.uint64))
    assert np.array_equal(p[-wp.size:], wp) and np.array_equal(m[-wm.size:], wm)


def test_chunked_digest(od, monkeypatch):
    monkeypatch.setattr(od, "CHUNK", 10)
    a = np.arange(37, dtype="<u8")
    d = od.Digest().update(a[:13]).update(a[13:]).result()
    assert d["sha256"] == hashlib.sha256(a.tobytes()).hexdigest() and d["n"] == 37
    assert d["chunks"] == [hashlib.sha256(a[i:i + 10].tobytes()).hexdigest() for i in range(0, 37, 10)]


def test_gpu_side_digest_format_agrees(od, monkeypatch):
    torch = pytest.importorskip("torch")
    gd = _load("gpu_digests", os.path.join(ROOT, "tests", "test_gpu_digests.py"))
    rng = np.random.default_rng(5)
    n = 1000
    h = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
    p = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    z = rng.integers(0, 2, size=n).astype(np.uint8)
    r17 = np.zeros(n, od.REC17)
    r17["hash"], r17["pos"], r17["strand"] = h, p, z
    monkeypatch.setattr(od, "CHUNK", 128)
    want = od.digest_of(r17)
    got = gd.sha_records17(h, p, z, 128)
    assert got.h.hexdigest() == want["sha256"] and got.chunks == want["chunks"]
    # anchors: GPU column order (ref_pos, read_pos, read_id, strand), arbitrary order in -> canonical
    an = np.stack([rng.integers(0, 50, n), rng.integers(0, 5, n), rng.integers(0, 7, n), rng.integers(0, 2, n)],
                  axis=1).astype(np.uint32)
    r16 = np.zeros(n, od.REC16)
    r16["ref_pos"], r16["read_pos"], r16["read_id"], r16["strand"] = an[:, 0], an[:, 1], an[:, 2], an[:, 3]
    r16 = np.sort(r16, order=["read_id", "ref_pos", "read_pos", "strand"])
    want = od.digest_of(r16)
    got = gd.sha_anchors(torch.from_numpy(an.astype(np.int64)), 128)
    assert got.h.hexdigest() == want["sha256"] and got.chunks == want["chunks"]
    u8 = rng.integers(0, 4, 300).astype(np.uint8)
    assert gd.sha_array(u8, 128).h.hexdigest() == od.digest_of(u8)["sha256"]


def test_tiny_golden_reproduces(od, tmp_path):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "digests", "tiny_10.json")))
    res = od.run_row("tiny", "10", 1.0, True, str(tmp_path))
    assert res["inputs"] == gold["inputs"]
    assert res["index_stats"] == gold["index_stats"]
    for name, d in gold["digests"].items():
        assert res["digests"][name]["sha256"] == d["sha256"], name


def test_every_row_has_a_golden_file(od):
    have = set(os.listdir(os.path.join(ROOT, "tests", "golden", "digests")))
    missing = [f"{c}_{p}.json" for c, p in od.ROWS if f"{c}_{p}.json" not in have]
    assert not missing, missing
