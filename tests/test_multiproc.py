"""Multi-process (world_size 2, gloo) coverage of the N>1 path: the per-rank
query shards partition the workload, the rank reduction gathers records and
takes the max step time (CPU), and -- on a GPU -- two ranks each plan their
own shard of real queries (two processes on cuda:0 here; one GPU per rank in
bench.py --gpus N), with no data-path collective."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world=2):
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda o: o[0])


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import bench
    return bench


def _shard_worker(rank, world, port, q):
    bench = _init(rank, world, port)
    w, r, _ = bench.dist_setup()
    Q = 6
    mine = [bench.query_index(s, j, Q, w, r) for s in range(3) for j in range(Q)]
    recs = [dict(k=k, rank=r) for k in mine]
    all_recs = sum(bench.gather(w, recs), [])
    mx = max(bench.gather(w, float(np.mean([10.0 * (r + 1), 20.0 * (r + 1)]))))
    bench.barrier(w)
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((r, mine, all_recs, mx))


def test_two_rank_sharding_and_reduction():
    out = _spawn(_shard_worker)
    shards = [set(o[1]) for o in out]
    assert not (shards[0] & shards[1])                 # disjoint shards
    assert len(shards[0]) == len(shards[1]) == 18      # weak scaling: same load per rank
    for _, _, all_recs, mx in out:
        assert len(all_recs) == 36 and {r["rank"] for r in all_recs} == {0, 1}
        assert mx == 30.0                               # max over ranks of the mean step time


def _plan_worker(rank, world, port, q):
    bench = _init(rank, world, port)
    w, r, _ = bench.dist_setup()
    import fixtures as fx
    from oracle import oracle as orc
    from paper_2505_06791_b200.planner import PlanParams, plan_many
    m, sc, sp = fx.robot("arm7"), fx.scene("table"), fx.spec("table_plane")
    s, g, seeds = bench.batch_arrays(7)
    B = 64
    lo, hi = r * B, (r + 1) * B                        # this rank's contiguous shard
    res = plan_many(m, sc, sp, s[lo:hi], g[lo:hi], seeds[lo:hi], PlanParams(width=16, max_iterations=2000))
    bad = 0
    for i in np.nonzero(res.solved)[0][:8]:
        for qn in res.path(int(i)):                   # nodes on the manifold, collision-free in FP64
            e = orc.task_error_at(sp.packed, orc.ee_pose(m.packed, qn))
            ok, *_ = orc.validate_waypoints(qn[None], m.packed, sc.packed(), False)
            bad += (not float(np.sqrt((e * e).sum())) < sp.tau_task) or (not ok)
    mine = (r, int(res.solved.sum()), bad, float(res.device_ms.max()))
    everyone = bench.gather(w, mine)
    bench.barrier(w)
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((r, everyone))


@pytest.mark.gpu
def test_two_ranks_plan_their_shards():
    out = _spawn(_plan_worker)
    for r, everyone in out:
        assert [e[0] for e in everyone] == [0, 1]
        for _, solved, bad, dev_ms in everyone:
            assert solved >= 60 and bad == 0 and dev_ms > 0


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu(tmp_path):
    """bench.py --gpus 2 end to end (relaunch under torch.distributed.run,
    gloo control plane, per-rank shards, max-over-ranks timing), both ranks on
    cuda:0 via the CPRRTC_BENCH_ONE_GPU test mode."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CPRRTC_BENCH_ONE_GPU="1")
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup",
                        "3", "--queries", "4", "--no-extras", "--no-cpu", "--records-dir", str(tmp_path)],
                       capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["queries"] == 8
    assert line["throughput"]["value"] > 0 and line["throughput"]["success_rate"] > 0.95
    assert "2 GPU(s)" in line["throughput"]["config"]
