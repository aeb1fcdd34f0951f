"""INT8 feed-forward path on the device (skiff quant.py) vs the reference.

The integer arithmetic is exact and the rescale is the reference's float32
sequence, so given the same float32 input rows the device quantization and
the int8 tcgen05 GEMM reproduce the reference BIT FOR BIT
(tests/golden/quant.npz, written by the reference).  End to end, models
swapped with quantize_model translate like the reference's quantized models
(tests/golden/quant_records.json): fp32 parity mode, >= 99 % identical
outputs, scores within 1e-4.
"""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from fixture_models import product_model, product_vocabs
from oracle import skiff_oracle as O
from oracle.fixture_configs import SEARCH_CASES

pytestmark = pytest.mark.gpu

G = np.load(GOLDEN / "quant.npz")


def _bits(a):
    return np.asarray(a, dtype=np.float32).view(np.int32)


def test_quantize_rows_bit_exact():
    from paper_2207_05851_b200 import kern
    for w, q, s in ((G["w1"], G["q1"], G["s1"]), (G["w2"], G["q2"], G["s2"]),
                    (G["x"], G["qx"], G["sx"])):
        wd = torch.as_tensor(w, device="cuda")
        qd = torch.empty(w.shape, dtype=torch.int8, device="cuda")
        sd = torch.empty(w.shape[0], device="cuda")
        kern.quantize_rows(wd, qd, sd)
        torch.cuda.synchronize()
        assert np.array_equal(qd.cpu().numpy(), q)
        assert np.array_equal(_bits(sd.cpu().numpy()), _bits(s))


@pytest.mark.parametrize("M,K,Nn", [(7, 256, 192), (640, 1024, 4096), (130, 4096, 1024),
                                    (1, 32, 64), (33, 48, 16)])
def test_gemm_i8_matches_oracle_bitwise(M, K, Nn):
    """Exact int32 accumulation + float32 rescale (+bias, ReLU / residual)."""
    from paper_2207_05851_b200 import _native as N
    from paper_2207_05851_b200 import kern
    rng = np.random.default_rng(M + K + Nn)
    x = rng.standard_normal((M, K)).astype(np.float32)
    w = (rng.standard_normal((Nn, K)) * 0.05).astype(np.float32)
    b = rng.standard_normal(Nn).astype(np.float32)
    qw, sw = O.quantize_rows(w)
    qx, sx = O.quantize_rows(x)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
    out = torch.zeros(M, Nn, device="cuda")
    kern.gemm_i8(dev(qx), dev(sx), dev(qw), dev(sw), out, N.EPI_RELU, dev(b))
    want = np.maximum(O.quantized_linear(x, qw, sw, b), 0).astype(np.float32)
    x0 = rng.standard_normal((M, Nn)).astype(np.float32)
    xr = dev(x0)
    kern.gemm_i8(dev(qx), dev(sx), dev(qw), dev(sw), xr, N.EPI_RESID, dev(b))
    torch.cuda.synchronize()
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(want))
    want_r = (x0 + O.quantized_linear(x, qw, sw, b)).astype(np.float32)
    assert np.array_equal(_bits(xr.cpu().numpy()), _bits(want_r))


def test_ffn_layer_reproduces_reference_outputs():
    """quantize(x) -> FFN1 (+b1, ReLU) -> quantize -> FFN2 (+b2) on the
    device from the reference's own quantized weights: bit-identical to the
    reference's QuantizedLinear outputs."""
    from paper_2207_05851_b200 import _native as N
    from paper_2207_05851_b200 import kern
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # noqa: E731
    M, K = G["x"].shape
    qa = torch.empty(M, K, dtype=torch.int8, device="cuda")
    sa = torch.empty(M, device="cuda")
    kern.quantize_rows(dev(G["x"]), qa, sa)
    f = torch.zeros(M, G["q1"].shape[0], device="cuda")
    kern.gemm_i8(qa, sa, dev(G["q1"]), dev(G["s1"]), f, N.EPI_STORE, dev(G["b1"]))
    f_relu = torch.zeros_like(f)
    kern.gemm_i8(qa, sa, dev(G["q1"]), dev(G["s1"]), f_relu, N.EPI_RELU, dev(G["b1"]))
    qf = torch.empty(M, f.shape[1], dtype=torch.int8, device="cuda")
    sf = torch.empty(M, device="cuda")
    kern.quantize_rows(f_relu, qf, sf)
    out2 = torch.zeros(M, G["q2"].shape[0], device="cuda")
    kern.gemm_i8(qf, sf, dev(G["q2"]), dev(G["s2"]), out2, N.EPI_STORE, dev(G["b2"]))
    torch.cuda.synchronize()
    assert np.array_equal(_bits(f.cpu().numpy()), _bits(G["out1"]))
    assert np.array_equal(_bits(out2.cpu().numpy()), _bits(G["out2"]))


def test_quantize_model_weights_match_reference():
    """quantize_model swaps exactly the feed-forward weights (quant.py:135-145)
    and their device int8 copies equal the reference quantizer's."""
    from paper_2207_05851_b200.model import Model
    from paper_2207_05851_b200.quant import quantize_model
    from fixture_models import oracle_model, product_config
    m = Model(product_config("tiny"), params=oracle_model("tiny").p, precision="fp32")
    names = quantize_model(m)
    assert names == [n for n in oracle_model("tiny").p if n.endswith((".ffn.w1", ".ffn.w2"))]
    for n in names:
        q, s = O.quantize_rows(oracle_model("tiny").p[n])
        assert np.array_equal(m.quantized[n].q.cpu().numpy(), q)
        assert np.array_equal(_bits(m.quantized[n].scales.cpu().numpy()), _bits(s))


GOLD = json.loads((GOLDEN / "quant_records.json").read_text())


@pytest.mark.parametrize("name", sorted(GOLD))
def test_quantized_translate_matches_reference(name):
    from paper_2207_05851_b200.model import Model
    from paper_2207_05851_b200.quant import quantize_model
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    from fixture_models import oracle_model, product_config
    case = next(c for c in SEARCH_CASES if c["name"] == name)
    m = Model(product_config(case["config"]), params=oracle_model(case["config"]).p,
              precision="fp32")
    quantize_model(m)
    recs = translate(m, product_vocabs(case["config"]),
                     [SentenceInput(**i) for i in case["inputs"]],
                     SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0)))
    gold = GOLD[name]
    assert len(recs) == len(gold)
    same = sum(r.text == g["text"] for r, g in zip(recs, gold))
    assert same >= 0.99 * len(gold), (same, len(gold))
    for r, g in zip(recs, gold):
        if r.text == g["text"]:
            assert abs(r.score - g["score"]) < 1e-4, (r.score, g["score"])


def test_quantized_bf16_model_runs_and_stays_close():
    """The int8 FFN inside a bf16 model (the bench precision): translation
    runs through the captured decode graphs and mostly agrees with fp32."""
    from paper_2207_05851_b200.model import Model
    from paper_2207_05851_b200.quant import quantize_model
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    from fixture_models import oracle_model, product_config
    case = next(c for c in SEARCH_CASES if c["name"] == "tiny_greedy_16x32")
    m = Model(product_config("tiny"), params=oracle_model("tiny").p, precision="bf16")
    quantize_model(m)
    recs = translate(m, product_vocabs("tiny"), [SentenceInput(**i) for i in case["inputs"]],
                     SearchSettings(beam=1))
    assert all(r.error is None for r in recs)
    same = sum(r.text == g["text"] for r, g in zip(recs, GOLD["tiny_greedy_16x32"]))
    assert same >= 0.5 * len(recs)
