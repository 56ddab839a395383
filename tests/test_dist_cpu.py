"""World-size-2 gloo tests of the multi-process plumbing (CPU, no GPU needed)."""

import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_06126_b200.dist import broadcast_bytes, max_over_ranks, row_shard, sum_over_ranks


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = bytes(range(128)) if rank == 0 else None
    got = broadcast_bytes(uid)
    mx = max_over_ranks(1.5 + rank)
    sm = sum_over_ranks(row_shard(8192, world, rank)[1])
    q.put((rank, got == bytes(range(128)), mx, sm))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_broadcast_and_reductions(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res)
    assert all(mx == 1.5 + world - 1 for _, _, mx, _ in res)
    assert all(sm == 8192 for _, _, _, sm in res)


def test_row_shard_partition_matches_oracle_schedule():
    from oracle.schedules import _shards
    for B in (1, 7, 256, 8192, 8193):
        for W in (1, 2, 3, 8):
            if B < W:
                continue
            mine = [row_shard(B, W, r) for r in range(W)]
            assert mine == _shards(B, W)
            assert sum(n for _, n in mine) == B
