"""N > 1 host logic on CPU (world_size 2, gloo): bench.py's rendezvous, barrier and
MAX-over-ranks timing reduction, and the gid-range sharding whose per-rank digests combine
(XOR / +) into the single-range digest -- the data path has no collective."""
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
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench
    import oracle
    from workloads import shard_range
    D = bench.Dist("gloo")
    try:
        assert D.world == world and D.rank == rank
        n, i = 10007, 5
        b, c = shard_range(n, rank, world)
        x, s = oracle.digest(n, i, 3, gid_begin=b, count=c)
        D.barrier()
        t = D.max(float(rank + 1) * 0.5)
        q.put((rank, b, c, x.tolist(), s.tolist(), t))
    finally:
        D.close()


def test_two_rank_gloo_shards_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    import oracle
    n, i = 10007, 5
    # contiguous, disjoint, covering
    assert res[0][1] == 0 and res[0][1] + res[0][2] == res[1][1] and res[1][1] + res[1][2] == n
    # MAX over ranks seen identically by every rank
    assert all(r[5] == 1.0 for r in res)
    x = np.bitwise_xor(np.array(res[0][3], np.uint64), np.array(res[1][3], np.uint64))
    s = np.array(res[0][4], np.uint64) + np.array(res[1][4], np.uint64)
    wx, ws = oracle.digest(n, i, 3)
    assert np.array_equal(x, wx) and np.array_equal(s, ws)


@pytest.mark.parametrize("n,world", [(1 << 28, 8), (1 << 24, 3), (7, 8), (10007, 4)])
def test_shard_range_partitions(n, world):
    from workloads import shard_range
    spans = [shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0
    for (b0, c0), (b1, _) in zip(spans, spans[1:]):
        assert b0 + c0 == b1
    assert sum(c for _, c in spans) == n
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
