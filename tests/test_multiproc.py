"""Multi-process (N > 1) host logic on CPU with the gloo backend, world_size 2 (-m "not gpu").

bench.py runs N replicas: every rank indexes the same reference and seeds its own
read batch; the only collective is the max over ranks of the timed region.  These tests check that
plumbing without a GPU: the reduction, the whole-job aggregate and the per-rank input split."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import bench
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.make_config("tiny", scale=0.05, read_seed_offset=7919 * rank)
    local_ms = 100.0 + 50.0 * rank
    m = bench.max_over_ranks(local_ms, dist, "cpu")
    v = bench.aggregate_rate(cfg.reads.n, world, m)
    q.put((rank, m, v, cfg.reads.n, hashlib.sha256(cfg.ref.tobytes()).hexdigest(),
           hashlib.sha256(cfg.reads.seq.tobytes()).hexdigest()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module", autouse=True)
def _libs(built):
    return built


def test_replicas_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (r0, m0, v0, n0, ref0, rd0), (r1, m1, v1, n1, ref1, rd1) = res
    assert m0 == m1 == 150.0                     # max over ranks
    assert v0 == v1 == pytest.approx(2 * n0 / 0.150)
    assert ref0 == ref1                          # same reference on every replica
    assert rd0 != rd1 and n0 == n1               # independent read batches of equal size


def test_single_process_reduction_is_identity():
    import bench
    assert bench.max_over_ranks(12.5) == 12.5
    assert bench.aggregate_rate(1000, 1, 500.0) == pytest.approx(2000.0)
    assert np.isfinite(bench.aggregate_rate(10, 8, 1.0))
