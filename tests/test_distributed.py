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


def _device_worker(rank, world, port, case_names, q):
    """One rank of a real multi-process translation job: each rank decodes
    its shard on cuda:0 through the product translate(), rank 0 gathers."""
    import sys

    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(__file__))
    from fixture_models import product_model, product_vocabs
    from oracle.fixture_configs import SEARCH_CASES
    from paper_2207_05851_b200.distributed import translate_distributed
    from paper_2207_05851_b200.search import SearchSettings
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for name in case_names:
        case = next(c for c in SEARCH_CASES if c["name"] == name)
        inputs = [SentenceInput(**i) for i in case["inputs"]]
        settings = SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0))
        recs = translate_distributed(product_model(case["config"], "fp32"),
                                     product_vocabs(case["config"]), inputs, settings, rank, world)
        if rank == 0:
            out[name] = [(r.text, r.score, r.error) for r in recs]
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_translate_distributed_device_world2_matches_reference():
    """translate_distributed with the real device translate() on two ranks
    (both on cuda:0, gloo for the gather): the gathered records equal the
    reference's own records for the same inputs (tests/golden/search.json)."""
    import json

    from conftest import GOLDEN
    names = ["toy_beam3", "tiny_greedy_16x32", "ssru_beam4"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(r, 2, port, names, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    gold = {c["name"]: c["records"] for c in json.loads((GOLDEN / "search.json").read_text())["cases"]}
    for name in names:
        assert len(got[name]) == len(gold[name])
        for (text, score, err), g in zip(got[name], gold[name]):
            assert (err is None) == (g["error"] is None)
            assert text == g["text"]
            if err is None:
                assert abs(score - g["score"]) < 1e-4
