"""World-size-2 gloo tests of the multi-GPU host logic (CPU): (batch x head)
sharding and the single-collective pattern broadcast."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_12578_b200.dist import broadcast_pattern, shard


def test_shard_partitions_exactly():
    for total in (1, 7, 128, 256):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard(total, r, world) for r in range(world)]
            covered = [i for a, b in ranges for i in range(a, b)]
            assert covered == list(range(total))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a packed pattern buffer as rank 0 would produce it (values arbitrary int32)
        n = 1000
        flat = torch.arange(n, dtype=torch.int32) * 7 - 3 if rank == 0 else torch.zeros(n, dtype=torch.int32)
        broadcast_pattern(flat, src=0)
        ok_bcast = bool((flat == torch.arange(n, dtype=torch.int32) * 7 - 3).all())
        # every rank regenerates its own (batch, head) slices from global indices
        import synth
        a, b = shard(6, rank, world)
        mine = synth.qkvdo(b - a, 16, 8, seed=5, dtype=torch.float32, start_bh=a)[0]
        full = synth.qkvdo(6, 16, 8, seed=5, dtype=torch.float32)[0]
        ok_shard = bool(torch.equal(mine, full[a:b]))
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_bcast, ok_shard, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_bcast, ok_shard, tmax in res:
        assert ok_bcast and ok_shard
        assert tmax == 2.0
