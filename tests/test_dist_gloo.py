"""World-size-2 checks of the N>1 host logic on CPU (gloo): balanced contiguous sharding of the
(b, h, row-block) units, max-over-ranks timing, and the rank-ordered output gather."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_06095_b200.dist import gather_rows, max_over_ranks, mha_units, shard_range


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 48, 192 * 8, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    assert mha_units(1, 12, 512) == 48  # cfg1: 6 units per GPU at 8 GPUs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = max_over_ranks(1.5 + rank)
        local = torch.full((3, 4), float(rank))
        g = gather_rows(local)
        b, e = shard_range(mha_units(16, 12, 1024), world, rank)
        q.put((rank, t, g.tolist(), (b, e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_reduction_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [2.5, 2.5]  # max over ranks
    for r in res:
        rows = r[2]
        assert rows[:3] == [[0.0] * 4] * 3 and rows[3:] == [[1.0] * 4] * 3  # rank-ordered gather
    assert res[0][3] == (0, 768) and res[1][3] == (768, 1536)


def _layer_worker(rank, world, port, q):
    """bench.py's N > 1 data path on CPU: the global batch's sequences sharded by shard_range, a
    row-independent layer stand-in (GEMM + LayerNorm, the per-row math of the layer's templates)
    applied per shard, outputs gathered in rank order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bs, seq, hid = 6, 16, 32
        g = torch.Generator().manual_seed(7)
        x_global = torch.rand(bs * seq, hid, generator=g)
        w = torch.rand(hid, hid, generator=g)
        b0, b1 = shard_range(bs, world, rank)
        x = x_global[b0 * seq:b1 * seq]
        y = torch.nn.functional.layer_norm(x @ w, (hid,))
        # gather_rows needs equal shards (all_gather); 6 sequences over 2 or 3 ranks are equal
        full = gather_rows(y)
        ref = torch.nn.functional.layer_norm(x_global @ w, (hid,))
        q.put((rank, bool(torch.equal(full, ref)), (b0, b1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_layer_gather_equals_whole_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000 + world
    procs = [ctx.Process(target=_layer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert [r[2] for r in res] == [shard_range(6, world, r) for r in range(world)]
