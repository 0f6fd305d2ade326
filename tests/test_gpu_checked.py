"""Memory-safety layer (-m gpu).  compute-sanitizer is refused on the GPU pool, so libgod also ships a
checked build (libgod_checked.so, -DGOD_CHECKED): every GOD_DCHECK on a computed global index or
address in K1, the index build and seeding traps with the violated bound printed (common.cuh).
This test reruns the whole stage-by-stage parity suite (tests/test_gpu_parity.py: tiny, repeat-rich,
every sort/directory variant, every specialised kernel, N runs, multi-length and misaligned buffers)
and the voting suite in a child process with GOD_CHECKED=1 (the binding then loads the checked library) and requires that they pass
and that the checked library is the one mapped.  Also: anchors handed to seeding's output and to
voting at 4-/8-byte offsets (the scalar fallbacks of the 128-bit anchor paths), against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2211_08157_b200 as god  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _gpu(built):
    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")


def test_checked_build_is_loaded():
    code = ("import os, paper_2211_08157_b200._lib as L; L.load(); "
            "maps = open('/proc/self/maps').read(); "
            "assert L.LIB_PATH.endswith('libgod_checked.so'), L.LIB_PATH; "
            "assert 'libgod_checked.so' in maps; print('checked library mapped')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env={**os.environ, "GOD_CHECKED": "1"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_parity_cases_under_checked_build():
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py",
                        "tests/test_gpu_vote.py", "-p", "no:cacheprovider"], cwd=ROOT,
                       env={**os.environ, "GOD_CHECKED": "1"}, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "GOD_CHECKED" not in r.stdout, tail
    assert " passed" in r.stdout, tail


def _canon(a):
    return np.array(sorted(map(tuple, a.tolist())), dtype=np.int64).reshape(-1, 4)


def test_misaligned_anchor_buffers():
    """god_seed_reads writing into, and god_vote_reads reading from, anchor buffers 4 / 8 bytes off a
    16-byte boundary (views of a u32 tensor): results equal the oracle (scalar anchor paths)."""
    cfg = synth.make_config("tiny", read_scale=0.1)
    ox = oracle.Index(cfg.ref, cfg.ref_offsets, "10", 21, 11)
    oan, oao, oph = ox.seed_reads(cfg.reads.seq, cfg.reads.offsets)
    ov, ovo = ox.vote_reads(cfg.reads.seq, cfg.reads.offsets, oph, D=0, V=3)
    dref, droff = torch.from_numpy(cfg.ref).cuda(), torch.from_numpy(cfg.ref_offsets).cuda()
    dreads, droffs = torch.from_numpy(cfg.reads.seq).cuda(), torch.from_numpy(cfg.reads.offsets).cuda()
    ix = god.god_build_index(dref, droff, "10", 21, 11)
    want = _canon(np.stack([oan["read_id"], oan["ref_pos"], oan["read_pos"], oan["strand"]], 1).astype(np.int64))
    n = cfg.reads.n
    for off_words in (1, 2):  # 4 and 8 bytes past a 16-B boundary
        cap = int(oan.size) + 64
        flat = torch.zeros(cap * 4 + 4, dtype=torch.uint32, device="cuda")
        an_view = flat[off_words:off_words + cap * 4].view(cap, 4)
        assert an_view.data_ptr() % 16 == 4 * off_words
        ao = torch.empty(n + 1, dtype=torch.uint64, device="cuda")
        ph = torch.empty(n, dtype=torch.uint8, device="cuda")
        an, ao, ph = god.god_seed_reads(ix, dreads, droffs, out=(an_view, ao, ph))
        assert an.data_ptr() % 16 == 4 * off_words
        got = an.cpu().numpy().astype(np.int64)
        assert np.array_equal(_canon(got[:, [2, 0, 1, 3]]), want)
        assert np.array_equal(ao.cpu().numpy(), oao) and np.array_equal(ph.cpu().numpy(), oph)
        v, vo = god.god_vote_reads(ix, dreads, droffs, ph, an, ao, D=0, V=3)
        assert np.array_equal(vo.cpu().numpy(), ovo)
        gv = god.votes_numpy(v)
        assert all(np.array_equal(gv[f], ov[f]) for f in ov.dtype.names)
    ix.free()
