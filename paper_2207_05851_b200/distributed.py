"""Data-parallel translation across the GPUs of one box.

Translation is embarrassingly parallel: every rank holds a full weight
replica and decodes its own contiguous, length-balanced shard of the
inputs; the only exchange is gathering the finished records back to rank 0
in input order.  There is no collective inside the decode loop.

`shard_bounds` balances by source length (decode work ~ 2L+10 steps per
chunk at random init); `gather_records` moves the (small) records with
torch.distributed's object gather — NCCL on GPUs, gloo in the CPU tests.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(lengths, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, end) shards with roughly equal sum(2L + 10)."""
    n = len(lengths)
    work = np.cumsum([2 * int(x) + 10 for x in lengths]) if n else np.zeros(0)
    total = float(work[-1]) if n else 0.0
    bounds, start = [], 0
    for r in range(world):
        if r == world - 1:
            end = n
        else:
            target = total * (r + 1) / world
            end = int(np.searchsorted(work, target, side="left")) + 1 if n else 0
            end = max(start, min(end, n))
        bounds.append((start, end))
        start = end
    return bounds


def shard_inputs(inputs, rank: int, world: int):
    """This rank's slice of `inputs` (SentenceInput list) and its offset."""
    b = shard_bounds([len(i.tokens) for i in inputs], world)[rank]
    return inputs[b[0]:b[1]], b[0]


def gather_records(records, rank: int, world: int, group=None):
    """Gather per-rank record lists to rank 0, concatenated in rank order
    (= input order, shards are contiguous).  Returns None on other ranks."""
    import torch.distributed as dist
    if world == 1:
        return list(records)
    out = [None] * world if rank == 0 else None
    dist.gather_object(list(records), out, dst=0, group=group)
    if rank != 0:
        return None
    merged = []
    for part in out:
        merged.extend(part)
    return merged


def translate_distributed(model, vocabs, inputs, settings=None, rank: int = 0, world: int = 1):
    """translate() over a torch.distributed job: shard, decode locally,
    gather to rank 0 (which returns the full record list)."""
    from .search import translate
    mine, _ = shard_inputs(inputs, rank, world)
    recs = translate(model, vocabs, mine, settings) if mine else []
    return gather_records(recs, rank, world)
