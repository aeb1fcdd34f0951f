"""Teacher-forced decode_step parity (model.py:521-585) on the device model
protocol, against logits recorded from the REFERENCE (tests/golden/steps_*).

Tolerances (north star): per-step log-probs within 1e-4 in fp32 mode and
2e-2 in bf16 mode, along the reference's own token path and row reorders.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from fixture_models import oracle_model, product_model
from oracle import skiff_oracle as O
from oracle.fixture_configs import CONFIGS

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", [n for n, s in CONFIGS.items() if s.get("steps")])
def test_teacher_forced_steps(name, precision):
    g = np.load(GOLDEN / f"steps_{name}.npz")
    m = product_model(name, precision)
    nsf, ntf = len(m.config.source_factor_specs), len(m.config.target_factor_specs)
    st = m.decode_init(g["src"], [g[f"src_factor{i}"] for i in range(nsf)], g["lens"])
    worst = 0.0
    for t in range(g["fed"].shape[0]):
        out = m.decode_step(st, g["fed"][t], [g[f"fed_factor{k}"][t] for k in range(ntf)])
        lp = O.log_softmax(out.surface.data)
        ref = O.log_softmax(g["logits"][t])
        worst = max(worst, float(np.abs(lp - ref).max()))
        for k in range(ntf):
            assert np.abs(out.factors[k].data - g[f"factor_logits{k}"][t]).max() < 50 * TOL[precision]
        st.select_rows(g["reorders"][t])
    assert worst <= TOL[precision], worst


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_tiny_greedy_path_teacher_forced(precision):
    """BASELINE configs[0] (tiny 2-1, d256, V8k): follow the ORACLE's greedy
    path for 3 sentences and compare every step's full log-prob row."""
    om = oracle_model("tiny")
    m = product_model("tiny", precision)
    rng = np.random.default_rng(3)
    worst = 0.0
    for _ in range(3):
        src = [int(x) for x in rng.integers(4, 8000, size=12)]
        trace = []
        O.greedy(om, O.OChunk(src), trace=trace)
        st = m.decode_init(np.array([src]), [], np.array([len(src)]))
        for step in trace:
            out = m.decode_step(st, np.array(step["fed"]), [])
            lp = O.log_softmax(out.surface.data)[0]
            worst = max(worst, float(np.abs(lp - step["lp"][0]).max()))
    assert worst <= TOL[precision], worst


def test_restricted_logits_are_a_column_subset():
    """test_model.py:292-301 on the device."""
    m = product_model("toy", "fp32")
    src, lens = np.array([[4, 5, 6]]), np.array([3])
    active = np.array([1, 3, 5, 8])
    full = m.decode_step(m.decode_init(src, [], lens), np.array([2]), []).surface.data
    sub = m.decode_step(m.decode_init(src, [], lens, active_ids=active), np.array([2]),
                        []).surface.data
    np.testing.assert_allclose(sub, full[:, active], rtol=0, atol=1e-6)


def test_nvs_select_matches_reference():
    g = np.load(GOLDEN / "steps_toy.npz")
    m = product_model("toy", "fp32")
    st = m.decode_init(g["src"], [], g["lens"])
    ids = m.nvs_select(st.enc, g["lens"], 0.5, [0, 1, 3])
    np.testing.assert_array_equal(np.concatenate(ids), g["nvs_ids"])


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", [n for n, s in CONFIGS.items()
                                  if s.get("steps") and s["steps"].get("teacher")])
def test_forward_sequence_matches_reference(name, precision):
    """model.py:444-492 (teacher forced) on the device vs the REFERENCE's own
    forward_sequence logits (tests/golden/steps_*.npz 'teacher_logits')."""
    g = np.load(GOLDEN / f"steps_{name}.npz")
    m = product_model(name, precision)
    nsf, ntf = len(m.config.source_factor_specs), len(m.config.target_factor_specs)
    out = m.forward_sequence(g["src"][:1], [g[f"src_factor{i}"][:1] for i in range(nsf)],
                             g["lens"][:1], g["fed"].T[:1],
                             [g[f"fed_factor{k}"].T[:1] for k in range(ntf)])
    got = out.surface.data
    ref = g["teacher_logits"]
    assert got.shape == ref.shape
    worst = float(np.abs(O.log_softmax(got) - O.log_softmax(ref)).max())
    assert worst <= TOL[precision], worst
    assert len(out.factors) == ntf


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("name", ["toy", "ssru", "tiny", "factored", "srcfac"])
def test_batched_teacher_forced_pass(name, precision):
    """forward_sequence runs all B x T positions in one pass (causal
    self-attention kernel / SSRU scan, B*T-row GEMMs): a ragged batch of 3
    sentences vs the oracle's full-sequence restatement of model.py:444-492,
    and vs the stepwise incremental path (the reference invariant
    test_model.py:270-282)."""
    m = product_model(name, precision)
    om = oracle_model(name)
    c = m.config
    nsf, ntf = len(c.source_factor_specs), len(c.target_factor_specs)
    rng = np.random.default_rng(17)
    B, L, T = 3, 6, 7
    lens = np.array([6, 3, 5])
    src = rng.integers(4, c.src_vocab_size, size=(B, L)).astype(np.int64)
    src_f = [rng.integers(4, s.vocab_size, size=(B, L)).astype(np.int64) for s in c.source_factor_specs]
    trg = rng.integers(4, c.trg_vocab_size, size=(B, T)).astype(np.int64)
    trg[:, 0] = 2  # BOS
    trg_f = [rng.integers(5, s.vocab_size, size=(B, T)).astype(np.int64) for s in c.target_factor_specs]
    for f in trg_f:
        f[:, 0] = 4  # shift marker
    got = m.forward_sequence(src, src_f, lens, trg, trg_f).surface.data
    want = om.forward_sequence(src, src_f, lens, trg, trg_f)
    assert got.shape == (B, T, c.trg_vocab_size)
    worst = float(np.abs(O.log_softmax(got) - O.log_softmax(np.asarray(want, np.float32))).max())
    assert worst <= TOL[precision], worst
    step = m.forward_sequence_stepwise(src, src_f, lens, trg, trg_f).surface.data
    worst = float(np.abs(O.log_softmax(got) - O.log_softmax(step)).max())
    assert worst <= TOL[precision], worst
