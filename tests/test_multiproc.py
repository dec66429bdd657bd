"""CPU, world_size 2 over gloo: the stream-sharding host logic of bench.py
(disjoint seeds per rank, max-over-ranks timing, whole-job aggregation)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    seeds = bench.shard_seeds(rank, 4)
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    fake_ms = torch.tensor([100.0 + 50.0 * rank], dtype=torch.float64)
    dist.all_reduce(fake_ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((gathered, float(fake_ms.item()), bench.aggregate_fps([fake_ms.item()], world, 4, 10)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, ms, fps = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert gathered[0] == [0, 1, 2, 3] and gathered[1] == [4, 5, 6, 7]
    assert not set(gathered[0]) & set(gathered[1])
    assert ms == 150.0
    assert fps == pytest.approx(2 * 4 * 10 / 0.150)


def _gather_worker(rank, world, port, out, n_streams, policy):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    from paper_1810_02648_b200.sharding import assign_streams, gather_results
    ids = assign_streams(n_streams, world, rank, policy)
    F, N = 3, 5
    poses = np.stack([np.full((F, 36), float(s)) for s in ids]) if ids else np.zeros((0, F, 36))
    verts = np.stack([np.full((F, N, 3), 10.0 + s) for s in ids]) if ids else np.zeros((0, F, N, 3))
    res = gather_results(poses, verts, n_streams, policy)
    if rank == 0:
        out.put((ids, res[0], res[1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_streams,policy", [(8, "block"), (7, "round_robin"), (5, "block")])
def test_result_gather_two_ranks(n_streams, policy):
    """§8e: results of unevenly sharded streams gathered to rank 0 in global order."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q, n_streams, policy)) for r in range(world)]
    for p in procs:
        p.start()
    ids0, P, V = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert P.shape == (n_streams, 3, 36) and V.shape == (n_streams, 3, 5, 3)
    for s in range(n_streams):
        assert (P[s] == s).all() and (V[s] == 10.0 + s).all()


def test_assign_streams_partition():
    from paper_1810_02648_b200.sharding import assign_streams
    for n in (1, 7, 8, 64):
        for world in (1, 2, 4, 8):
            for policy in ("block", "round_robin"):
                ids = [assign_streams(n, world, r, policy) for r in range(world)]
                flat = sorted(i for x in ids for i in x)
                assert flat == list(range(n))
                assert max(map(len, ids)) - min(map(len, ids)) <= 1


def test_bench_spawns_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (the
    driver's torchrun command line); the dry run exercises the whole
    multi-rank path of run_ours on CPU (gloo): sharding, barrier,
    max-over-ranks, gather to rank 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                        "--streams", "3", "--steps", "2"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"]
    assert d["shards"] == [[0, 1, 2], [3, 4, 5]]
    assert d["gathered_streams"] == 6 and d["gather_ok"]
    assert d["config"]["total_streams"] == 6
