"""torch.distributed plumbing for row-sharded learner groups (process groups only: no compute).

One process per GPU (torchrun).  Rank 0 draws the NCCL unique id through the C ABI
(spz_nccl_unique_id) and broadcasts its 128 bytes; timings are reduced as the max over ranks.
"""

import os

import torch
import torch.distributed as dist


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def row_shard(batch, world, rank):
    """(row0, rows) of `rank`: global rows [0, B) split contiguously, the first B % W ranks one row longer.

    Mirrors the learner's own partition (reading #17) for reporting and tests."""
    base, rem = divmod(batch, world)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def broadcast_bytes(payload, src=0, device=None):
    """Broadcast a bytes object (e.g. the 128-byte NCCL unique id) from `src` to every rank."""
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src, device=device)
    return obj[0]


def max_over_ranks(value, device=None):
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value, device=None):
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
