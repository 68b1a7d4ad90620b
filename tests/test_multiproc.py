"""Multi-process (world_size 2, gloo) coverage of the N>1 bench path: the
per-rank query shards partition the workload, and the rank reduction merges
records and takes the max step time.  CPU only."""

import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import bench
    w, r, _ = bench.dist_setup()
    Q = 6
    mine = [bench.query_index(s, j, Q, w, r) for s in range(3) for j in range(Q)]
    recs = [dict(k=k, rank=r) for k in mine]
    all_recs, mx = bench.merge_ranks(w, recs, [10.0 * (r + 1), 20.0 * (r + 1)])
    bench.barrier(w)
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((r, mine, all_recs, mx))


def test_two_rank_sharding_and_reduction():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    shards = [set(o[1]) for o in out]
    assert not (shards[0] & shards[1])                 # disjoint shards
    assert len(shards[0]) == len(shards[1]) == 18      # weak scaling: same load per rank
    for _, _, all_recs, mx in out:
        assert len(all_recs) == 36 and {r["rank"] for r in all_recs} == {0, 1}
        assert mx == 30.0                               # max over ranks of the mean step time
