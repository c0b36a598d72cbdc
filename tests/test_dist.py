"""CPU: the N>1 host path (instance sharding + final gather) with world_size 2
over gloo, as the 8-GPU box runs it over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_09258_b200 import abi, dist as cdist


def test_shard_by_weight_balances_and_covers():
    w = [5, 1, 1, 1, 1, 1, 5, 5]
    for world in [1, 2, 3, 4, 8]:
        shards = cdist.shard_by_weight(w, world)
        assert len(shards) == world
        assert shards[0][0] == 0 and shards[-1][1] == len(w)
        for (b0, e0), (b1, e1) in zip(shards, shards[1:]):
            assert e0 == b1 and b0 <= e0
    s = cdist.shard_by_weight([1] * 1024, 8)
    assert all(e - b == 128 for b, e in s)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank "analyses" its shard of instances and emits alert rows
        shards = cdist.shard_by_weight([3, 1, 4, 1, 5, 9, 2, 6], world)
        b, e = shards[rank]
        alerts = np.zeros(e - b + rank, dtype=abi.ALERT_DTYPE)
        alerts["cycle"] = np.arange(len(alerts)) + 1000 * rank
        alerts["episode_id"] = np.arange(len(alerts))
        got = cdist.gather_bytes(alerts.view(np.uint8))
        t = cdist.max_over_ranks(1.5 + rank)
        if rank == 0:
            rows = [g.view(abi.ALERT_DTYPE) for g in got]
            q.put(([len(r) for r in rows], [list(r["cycle"]) for r in rows], t))
    finally:
        dist.destroy_process_group()


def test_gather_alerts_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    sizes, cycles, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = cdist.shard_by_weight([3, 1, 4, 1, 5, 9, 2, 6], 2)
    assert sizes == [shards[0][1] - shards[0][0], shards[1][1] - shards[1][0] + 1]
    assert cycles[1][0] == 1000
    assert t == 2.5
