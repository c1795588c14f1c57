"""Multi-process (world size 2, gloo, CPU) tests of the sharding host logic."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_16834_b200 import sharding


def test_partitions_cover_exactly_once():
    for n, w in [(8, 1), (8, 2), (8, 3), (16, 8), (64, 6)]:
        got = sorted(g for r in range(w) for g in sharding.assign_groups(n, w, r))
        assert got == list(range(n))
        blocks = sharding.channel_shards(n, w)
        assert [i for b in blocks for i in b] == list(range(n))
        assert max(len(b) for b in blocks) - min(len(b) for b in blocks) <= 1


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
        groups = sharding.assign_groups(8, world, rank)
        # each rank "evaluates" its groups: a deterministic function of the group id
        local = {g: np.full(4, g * 10.0 + rank) for g in groups}
        allres = sharding.gather_group_results(local, world)
        t = sharding.max_over_ranks(1.5 + rank, world)
        q.put((rank, sorted(allres), float(t)))
    finally:
        dist.destroy_process_group()


def test_group_sharding_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, groups, t in res:
        assert groups == list(range(8))          # every group evaluated exactly once, visible everywhere
        assert t == 2.5                          # max over ranks
