"""End-to-end translate() on the GPU vs the reference's own records
(tests/golden/search.json, produced by the reference) and vs the oracle.

fp32 mode: output token sequences identical on >= 99% of records and
scores within 1e-4 (north star: per-step log-probs within 1e-4 in fp32).
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from fixture_models import product_model, product_vocabs
from oracle.fixture_configs import SEARCH_CASES

pytestmark = pytest.mark.gpu

GOLD = {c["name"]: c["records"] for c in json.loads((GOLDEN / "search.json").read_text())["cases"]}


def _settings(case):
    from paper_2207_05851_b200.search import (NvsRestriction, SearchSettings,
                                              ShortlistRestriction)
    from paper_2207_05851_b200.shortlist import Shortlist
    restriction = None
    if case.get("shortlist"):
        restriction = ShortlistRestriction(Shortlist(
            {int(k): np.asarray(v, dtype=np.int64) for k, v in case["shortlist"].items()}))
    elif case.get("nvs") is not None:
        restriction = NvsRestriction(case["nvs"])
    return SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0),
                          restriction=restriction, use_greedy=case.get("use_greedy"))


def _run(case, precision):
    from paper_2207_05851_b200.search import SentenceInput, translate
    over = {"max_seq_len": case["max_seq_len"]} if case.get("max_seq_len") else {}
    m = product_model(case["config"], precision, **over)
    inputs = [SentenceInput(**inp) for inp in case["inputs"]]
    return translate(m, product_vocabs(case["config"]), inputs, _settings(case))


STATS = {"n": 0, "same": 0}


@pytest.mark.parametrize("case", SEARCH_CASES, ids=lambda c: c["name"])
def test_translate_fp32_matches_reference(case):
    recs = _run(case, "fp32")
    gold = GOLD[case["name"]]
    assert len(recs) == len(gold)
    mismatched = []
    for r, g in zip(recs, gold):
        assert (r.error is None) == (g["error"] is None), (r, g)
        if g["error"] is not None:
            assert r.text == "" and r.chunks == 0
            continue
        STATS["n"] += 1
        assert r.chunks == g["chunks"]
        if r.text == g["text"] and r.factors == g["factors"]:
            STATS["same"] += 1
            assert r.forced_eos == g["forced_eos"]
            assert abs(r.score - g["score"]) <= 1e-4, (r.score, g["score"])
        else:
            mismatched.append((r.text, g["text"]))
    # >= 99% identical overall; a small case may not lose a single record
    assert len(mismatched) <= len(recs) // 100, mismatched


def test_batch_equals_one_by_one():
    """test_search.py:400-405 on the device path (batch composition invariance)."""
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    case = next(c for c in SEARCH_CASES if c["name"] == "toy_beam3")
    m = product_model("toy", "bf16")
    v = product_vocabs("toy")
    inputs = [SentenceInput(**i) for i in case["inputs"]]
    together = translate(m, v, inputs, SearchSettings(beam=3))
    single = [translate(m, v, [i], SearchSettings(beam=3))[0] for i in inputs]
    assert together == single


def test_greedy_equals_beam_one_device():
    """test_search.py:170-177: bit-exact logprob and tokens."""
    from paper_2207_05851_b200.search import SentenceInput, beam_search, greedy_search
    m = product_model("toy", "bf16")
    v = product_vocabs("toy")
    for inp in next(c for c in SEARCH_CASES if c["name"] == "toy_greedy")["inputs"]:
        s = SentenceInput(**inp)
        g = greedy_search(m, v, s)
        b = beam_search(m, v, s, beam=1)
        assert g == b


def test_wider_beam_never_scores_worse():
    from paper_2207_05851_b200.search import SentenceInput, beam_search
    m = product_model("toy", "fp32")
    v = product_vocabs("toy")
    for inp in next(c for c in SEARCH_CASES if c["name"] == "toy_beam3")["inputs"]:
        s = SentenceInput(**inp)
        assert beam_search(m, v, s, 4).normalized(1.0) >= beam_search(m, v, s, 1).normalized(1.0)


def test_tiny_bf16_agreement_report():
    """bf16 tensor-core mode on BASELINE configs[0]: outputs are NOT required
    to be identical (random-init margins ~1e-3); per-step parity
    is checked teacher-forced in test_model_gpu.py.  Here: sanity + report."""
    case = next(c for c in SEARCH_CASES if c["name"] == "tiny_greedy_16x32")
    recs = _run(case, "bf16")
    gold = GOLD[case["name"]]
    same = sum(r.text == g["text"] for r, g in zip(recs, gold))
    tok_agree = np.mean([np.mean([a == b for a, b in zip(r.text.split(), g["text"].split())])
                         for r, g in zip(recs, gold)])
    print(f"bf16 tiny greedy: {same}/{len(gold)} identical, token agreement {tok_agree:.3f}")
    assert all(r.forced_eos == g["forced_eos"] for r, g in zip(recs, gold))
    assert tok_agree > 0.5


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_concurrent_stream_batches_identical(precision):
    """decode_jobs runs its batches concurrently on several CUDA streams, with
    GEMM tiles sized for the shared device (skb_epilogue.streams).  Tile sizes
    never change numerics, so the records are identical to one stream."""
    from paper_2207_05851_b200 import engine
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    m = product_model("toy", precision)
    vocabs = product_vocabs("toy")
    rng = np.random.default_rng(5)
    words = [vocabs.src_vocab.to_token(i) for i in range(4, len(vocabs.src_vocab))]
    inputs = [SentenceInput(tokens=[words[i] for i in rng.integers(0, len(words), rng.integers(3, 20))])
              for _ in range(40)]
    old = engine.DECODE_STREAMS
    try:
        out = {}
        for streams in (1, 3):
            engine.DECODE_STREAMS = streams
            out[streams] = translate(m, vocabs, inputs, SearchSettings(beam=3), max_rows=24)
    finally:
        engine.DECODE_STREAMS = old
    assert [(r.text, r.score) for r in out[1]] == [(r.text, r.score) for r in out[3]]


@pytest.mark.parametrize("gemm_split", ["throughput", "latency"])
def test_batch_invariance_at_scale(gemm_split):
    """test_search.py:400-405 at the benchmark model's size (bf16): a batch
    whose encoder sees > 2560 rows (B*L) and whose decoder runs several
    streams of R = 640 rows, against the same sentences one at a time
    (R = beam, prologue-LayerNorm GEMMs).  Every GEMM, the split-K FFN2 and
    the log-softmax partials must take the same reduction order — for the
    serving model and for the latency model (every projection K-split, the
    small-slice st.async reduction at R = 5, the bulk-copy one at R = 640)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    model, vocabs, _ = bench.build_model("big", gemm_split=gemm_split)
    rng = np.random.default_rng(7)
    sents = [[f"w{i}" for i in rng.integers(0, 31996, size=int(n))] for n in rng.integers(1, 121, size=160)]
    st = SearchSettings(beam=5, length_alpha=1.0)
    big = translate(model, vocabs, [SentenceInput(tokens=s) for s in sents], st, max_rows=640)
    for i in (0, 41, 97, 159):
        one = translate(model, vocabs, [SentenceInput(tokens=sents[i])], st)[0]
        assert one.text == big[i].text and one.score == big[i].score, (i, one.score, big[i].score)


@pytest.mark.parametrize("name", ["srcfac", "ssru", "factored"])
def test_translate_from_reference_written_model_dir(name):
    """Load a model directory the REFERENCE wrote (save_model_dir,
    checkpoint.py:316-330) with the product's load_model_dir and translate:
    the records equal the ones the reference produced from the same
    directory (tests/golden/refdir_records.json)."""
    from paper_2207_05851_b200.checkpoint import load_model_dir
    from paper_2207_05851_b200.search import SentenceInput, translate
    gold = json.loads((GOLDEN / "refdir_records.json").read_text())[name]
    case = next(c for c in SEARCH_CASES if c["name"] == gold["case"])
    md = load_model_dir(GOLDEN / f"refdir_{name}", precision="fp32")
    recs = translate(md.model, md, [SentenceInput(**i) for i in case["inputs"]], _settings(case))
    assert len(recs) == len(gold["records"])
    for r, g in zip(recs, gold["records"]):
        assert (r.error is None) == (g["error"] is None)
        assert r.text == g["text"] and r.factors == g["factors"] and r.chunks == g["chunks"]
        if g["error"] is None:
            assert abs(r.score - g["score"]) < 1e-4


def test_workspaces_released_with_model():
    """A released Model takes its cached decode workspaces (KV cache, graphs)
    with it: the per-model cache is weak in the model, and the workspaces
    hold only a weak reference back (cached workspaces kept old
    models alive)."""
    import gc
    import weakref

    from fixture_models import oracle_model, product_config
    from paper_2207_05851_b200 import engine
    from paper_2207_05851_b200.model import Model
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    case = next(c for c in SEARCH_CASES if c["name"] == "toy_beam3")
    m = Model(product_config("toy"), params=oracle_model("toy").p, precision="bf16")
    translate(m, product_vocabs("toy"), [SentenceInput(**i) for i in case["inputs"]],
              SearchSettings(beam=3))
    assert m in engine._WS_CACHE and len(engine._WS_CACHE[m]) > 0
    ref = weakref.ref(m)
    del m
    gc.collect()
    assert ref() is None
    assert all(k is not None for k in engine._WS_CACHE.keys())
    assert not any(ref() is k for k in engine._WS_CACHE.keys())
