"""World-size-2 gloo tests of the multi-GPU host logic (CPU): (batch x head)
sharding (the bench's strong-scaling split), the single-collective broadcast of a
real packed BlockPattern, and that per-rank results reassemble the 1-rank result."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_12578_b200.dist import allreduce_pool, broadcast_pattern, pattern_rows, shard


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


def _fill_pattern(bp, fl):
    """Write a block mask and its CSR/CSC (from the oracle) into a BlockPattern's views, as rank 0's
    spion_pattern would (the plan words stay as allocated: they are opaque bytes to the broadcast)."""
    import numpy as np

    import oracle
    n = fl.shape[0]
    bsr = oracle.mask_to_bsr(fl)
    k = bsr["nnzb"]
    bp.brow_ptr.copy_(torch.from_numpy(bsr["brow_ptr"]))
    bp.bcol_idx[:k].copy_(torch.from_numpy(bsr["bcol_idx"]))
    bp.bcol_ptr.copy_(torch.from_numpy(bsr["bcol_ptr"]))
    bp.brow_idx[:k].copy_(torch.from_numpy(bsr["brow_idx"]))
    bp.mask.copy_(torch.from_numpy(np.ascontiguousarray(fl, dtype=np.uint8).reshape(-1)))
    bp.nnzb_dev[0] = k
    bp.plan.copy_(torch.arange(bp.plan.numel(), dtype=torch.int32).to(torch.uint8))


def _worker_pattern(rank, world, port, out_q):
    """The bench's multi-GPU data path on CPU: rank 0 owns the pattern and broadcasts the whole
    BlockPattern.flat in ONE collective; every rank runs its strong-scaling shard of the
    (batch, head) slices (regenerated from global slice indices) through the fp64 oracle; the
    shards gathered on rank 0 equal the 1-rank result exactly."""
    import math

    import numpy as np

    import bench
    import oracle
    import synth
    from paper_2309_12578_b200 import spion
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, B, d = 64, 8, 16
        cfg = dict(bench.CONFIGS["image"], L=L, block=B, d=d, batch=3, heads=2)
        n = L // B
        bp = spion.empty_pattern(L, B, "cpu")
        if rank == 0:
            A = synth.syn_scores(L, B, heads=2, seed=4).numpy()
            fl, _, _ = oracle.pattern(A, B, 31, 75.0)
            _fill_pattern(bp, fl)
        broadcast_pattern(bp.flat, src=0)
        fl_r = bp.mask.view(n, n).numpy().copy()
        # every field of the packed buffer arrived (compare with a freshly filled copy)
        ref = spion.empty_pattern(L, B, "cpu")
        _fill_pattern(ref, fl_r)
        ok_flat = bool(torch.equal(ref.flat, bp.flat)) and int(bp.nnzb_dev[0]) == int(fl_r.sum())
        a, b = bench.rank_slices(cfg, "strong", rank, world)
        q, k, v, do = synth.qkvdo(b - a, L, d, seed=17, dtype=torch.float32, start_bh=a)
        outs = []
        for i in range(b - a):
            Q, K, V, dO = (x[i].double().numpy() for x in (q, k, v, do))
            O, _ = oracle.attn_fwd(Q, K, V, fl_r, B, 1 / math.sqrt(d), "paper")
            dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl_r, B, 1 / math.sqrt(d), "paper")
            outs.append(np.stack([O, dQ, dK, dV]))
        mine = torch.from_numpy(np.stack(outs)) if outs else torch.zeros((0, 4, L, d), dtype=torch.float64)
        sizes = [bench.rank_slices(cfg, "strong", r, world) for r in range(world)]
        gathered = [torch.zeros((hi - lo, 4, L, d), dtype=torch.float64) for lo, hi in sizes]
        dist.all_gather(gathered, mine)
        ok_join = True
        if rank == 0:
            full = torch.cat(gathered)
            bh_total = cfg["batch"] * cfg["towers"] * cfg["heads"]
            ok_join = full.shape[0] == bh_total
            q1, k1, v1, do1 = synth.qkvdo(bh_total, L, d, seed=17, dtype=torch.float32)
            for i in range(bh_total):
                Q, K, V, dO = (x[i].double().numpy() for x in (q1, k1, v1, do1))
                O, _ = oracle.attn_fwd(Q, K, V, fl_r, B, 1 / math.sqrt(d), "paper")
                dQ, dK, dV = oracle.attn_bwd(Q, K, V, dO, fl_r, B, 1 / math.sqrt(d), "paper")
                ok_join &= bool(torch.equal(full[i], torch.from_numpy(np.stack([O, dQ, dK, dV]))))
        out_q.put((rank, ok_flat, ok_join, b - a))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_pattern_broadcast_and_shard_reassembly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pattern, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_flat, ok_join, nb in res:
        assert ok_flat and ok_join, (rank, ok_flat, ok_join)
        assert nb == 3  # 3 batch x 2 heads split over 2 ranks


def test_bench_rank_slices():
    import bench
    for name, cfg in bench.CONFIGS.items():
        bh = cfg["batch"] * cfg["towers"] * cfg["heads"]
        for world in (1, 2, 4, 8):
            r = [bench.rank_slices(cfg, "strong", k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == bh and all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            assert len({b - a for a, b in r}) == 1  # every config divides evenly at 1/2/4/8 GPUs
            w = [bench.rank_slices(cfg, "weak", k, world) for k in range(world)]
            assert all(b - a == bh for a, b in w)


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


def _worker_pool(rank, world, port, out_q):
    """The bench's default multi-GPU pattern exchange on CPU: each rank pools its own slab of score
    rows (the oracle's Eq. 3-4 on the matrix that keeps only those rows, as spion_pattern_pool
    computes on the rank's GPU), ONE all-reduce sums the int64 pools, and every rank thresholds and
    flood-fills the sum: every rank holds exactly the 1-rank pattern."""
    import numpy as np

    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for L, B, F, alpha in ((64, 8, 31, 75.0), (96, 4, 63, 60.0), (256, 32, 31, 90.0)):
            A = synth.syn_scores(L, B, heads=2, seed=L + F).numpy()
            r0, r1 = pattern_rows(L, B, rank, world)
            As = np.zeros_like(A)
            As[r0:r1] = A[r0:r1]
            part = oracle.pool_sum(oracle.diag_conv(oracle.quantize(As), F), B)
            region = torch.from_numpy(part.reshape(-1).copy())
            allreduce_pool(region)
            pool = region.numpy().reshape(part.shape)
            gt, _ = oracle.threshold_gt(pool, B, alpha)
            fl = oracle.flood_fill(pool, gt)
            fl_ref, _, _ = oracle.pattern(A, B, F, alpha)
            ok &= bool((fl == fl_ref).all())
        out_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_pattern_rows_partition():
    for L, B in ((64, 8), (1024, 32), (4096, 64), (96, 4)):
        for world in (1, 2, 3, 4, 8):
            r = [pattern_rows(L, B, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == L and all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            assert all(a % B == 0 and b % B == 0 for a, b in r)


def test_gloo_world2_pool_allreduce_pattern():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pool, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok in res), res
