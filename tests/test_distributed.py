"""Multi-process sharding + final gather of the data-parallel translation
path, on CPU with the gloo backend (world_size 2), as the GPU job does over
NCCL (no collective inside the decode loop, one gather)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2207_05851_b200.distributed import gather_records, shard_bounds, shard_inputs
from paper_2207_05851_b200.search import SentenceInput, TranslationRecord


def test_shard_bounds_cover_and_balance():
    lengths = [30] * 50 + [5] * 50 + [60] * 28
    for world in (1, 2, 4, 8):
        b = shard_bounds(lengths, world)
        assert b[0][0] == 0 and b[-1][1] == len(lengths)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        work = [sum(2 * x + 10 for x in lengths[s:e]) for s, e in b]
        assert max(work) - min(work) <= 2 * max(2 * x + 10 for x in lengths)
    assert shard_bounds([], 4) == [(0, 0)] * 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inputs = [SentenceInput(tokens=[f"w{i}"] * (1 + i % 7)) for i in range(n)]
    mine, off = shard_inputs(inputs, rank, world)
    # stand-in for the device translate(): echo the input position
    recs = [TranslationRecord(text=f"out{off + k}", score=-float(off + k), factors=[], chunks=1,
                              forced_eos=False) for k in range(len(mine))]
    merged = gather_records(recs, rank, world)
    if rank == 0:
        q.put([r.text for r in merged])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [13, 1, 0])
def test_gloo_world2_gather_restores_input_order(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [f"out{i}" for i in range(n)]
