"""Shared definitions of the golden-fixture models and search cases.

Used by oracle/make_golden.py (which runs the reference on them) and by the
tests (which rebuild the same models from the same seeds via the oracle's
init and the product's loader).  Pure data + a seeded input generator; no
reference code.
"""

from __future__ import annotations

import numpy as np


def make_words(n: int) -> list[str]:
    return [f"w{i}" for i in range(n)]


CONFIGS = {
    # test_search.py toy: untrained 1+1 layers with NVS head (seed 31)
    "toy": dict(seed=31, config=dict(src_vocab_size=14, trg_vocab_size=14, d_model=16, heads=2,
                                     ff_dim=32, encoder_layers=1, decoder_layers=1,
                                     nvs_enabled=True, max_seq_len=16),
                steps=dict(L=5, T=6, teacher=True),
                beam_trace=dict(beam=4, L=4)),
    # one target factor stream (test_search.py factored, seed 77)
    "factored": dict(seed=77, config=dict(src_vocab_size=14, trg_vocab_size=14, d_model=16,
                                          heads=2, ff_dim=32, encoder_layers=1, decoder_layers=1,
                                          target_factor_specs=[7], max_seq_len=16),
                     steps=dict(L=4, T=5)),
    # SSRU hybrid decoder
    "ssru": dict(seed=5, config=dict(src_vocab_size=40, trg_vocab_size=40, d_model=32, heads=4,
                                     ff_dim=64, encoder_layers=2, decoder_layers=2,
                                     decoder_kind="ssru", max_seq_len=32),
                 steps=dict(L=6, T=7, teacher=True),
                 beam_trace=dict(beam=3, L=5)),
    # source factors (sum + concat) and a target factor
    "srcfac": dict(seed=11, config=dict(src_vocab_size=30, trg_vocab_size=30, d_model=32, heads=4,
                                        ff_dim=48, encoder_layers=1, decoder_layers=1,
                                        source_factor_specs=[(8, 32, "sum"), (6, 8, "concat")],
                                        target_factor_specs=[9], max_seq_len=16),
                   steps=dict(L=5, T=4)),
    # BASELINE.json configs[0]: tiny transformer enc 2 / dec 1, d=256, vocab 8k
    "tiny": dict(seed=13, config=dict(src_vocab_size=8000, trg_vocab_size=8000, d_model=256,
                                      heads=4, ff_dim=1024, encoder_layers=2, decoder_layers=1,
                                      max_seq_len=128),
                 steps=dict(L=6, T=4),
                 beam_trace=dict(beam=5, L=5, keep_lp_steps=[1])),
}


def _sentences(seed, n, vocab_words, lo=1, hi=8):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        k = int(rng.integers(lo, hi + 1))
        out.append([str(w) for w in rng.choice(vocab_words, size=k)])
    return out


def _inputs(tokens_list, **kw):
    return [dict(tokens=t, **kw) for t in tokens_list]


def _shortlist_rows(seed, n_src, n_trg, k):
    rng = np.random.default_rng(seed)
    return {str(i): sorted(set(int(x) for x in rng.integers(4, n_trg, size=k)))
            for i in range(n_src)}


W10 = make_words(10)
W36 = make_words(36)
W26 = make_words(26)
W7996 = make_words(7996)

SEARCH_CASES = [
    dict(name="toy_greedy", config="toy", beam=1, inputs=_inputs(_sentences(5, 12, W10))),
    dict(name="toy_beam1_nogreedy", config="toy", beam=1, use_greedy=False,
         inputs=_inputs(_sentences(5, 12, W10))),
    dict(name="toy_beam3", config="toy", beam=3, inputs=_inputs(_sentences(7, 10, W10))),
    dict(name="toy_beam5_a06", config="toy", beam=5, alpha=0.6,
         inputs=_inputs(_sentences(8, 10, W10))),
    dict(name="toy_shortlist_beam2", config="toy", beam=2,
         shortlist=_shortlist_rows(9, 14, 14, 3), inputs=_inputs(_sentences(10, 10, W10))),
    dict(name="toy_nvs_greedy", config="toy", beam=1, nvs=0.5,
         inputs=_inputs(_sentences(6, 8, W10))),
    dict(name="toy_nvs_beam3", config="toy", beam=3, nvs=0.5,
         inputs=_inputs(_sentences(6, 8, W10))),
    dict(name="toy_prefix_greedy", config="toy", beam=1,
         inputs=_inputs(_sentences(11, 6, W10), target_prefix=["w3", "w1"])),
    dict(name="toy_prefix_beam3_strip", config="toy", beam=3,
         inputs=_inputs(_sentences(11, 6, W10), target_prefix=["w7", "w8"], strip_prefix=True)),
    dict(name="toy_prefix_oov_and_eos", config="toy", beam=2,
         inputs=[dict(tokens=["w1", "w2"], target_prefix=["nope", "w4"]),
                 dict(tokens=["w5"], target_prefix=["</s>"])]),
    dict(name="toy_chunked_beam2", config="toy", beam=2, max_seq_len=4,
         inputs=_inputs(_sentences(12, 5, W10, lo=5, hi=11), source_prefix=["w9"])
         + [dict(tokens=["w1"] * 9, target_prefix=["w2"], prefix_all_chunks=True)]),
    dict(name="toy_errors", config="toy", beam=2,
         inputs=[dict(tokens=["w1"]), dict(tokens=[]), dict(tokens=["w1"], source_factors=[["P"]]),
                 dict(tokens=["w1"], target_prefix=["w2"] * 12), dict(tokens=["w3", "w4"])]),
    dict(name="factored_greedy", config="factored", beam=1,
         inputs=[dict(tokens=["w1", "w2"], target_prefix=["w3", "w4", "w5"],
                      target_prefix_factors=[["F0_0", "F0_0", "F0_1"]])]
         + _inputs(_sentences(13, 5, W10))),
    dict(name="factored_beam3", config="factored", beam=3,
         inputs=[dict(tokens=["w1", "w2"], target_prefix=["w3"],
                      target_prefix_factors=[["F0_1"]])]
         + _inputs(_sentences(14, 5, W10))),
    # prefix-factor streams longer than the surface prefix (the factor of
    # output token j is emitted at step j + 1, search.py:261-272)
    dict(name="factored_long_factor_prefix", config="factored", beam=3,
         inputs=[dict(tokens=["w1", "w2", "w6"], target_prefix=["w3"],
                      target_prefix_factors=[["F0_0", "F0_1", "F0_0"]]),
                 dict(tokens=["w4"], target_prefix_factors=[["F0_1", "F0_1"]])]),
    dict(name="factored_long_factor_prefix_greedy", config="factored", beam=1,
         inputs=[dict(tokens=["w1", "w2", "w6"], target_prefix=["w3"],
                      target_prefix_factors=[["F0_0", "F0_1", "F0_0"]])]),
    dict(name="ssru_greedy", config="ssru", beam=1, inputs=_inputs(_sentences(15, 6, W36))),
    dict(name="ssru_beam4", config="ssru", beam=4, alpha=0.6,
         inputs=_inputs(_sentences(16, 6, W36))),
    dict(name="srcfac_beam2", config="srcfac", beam=2,
         inputs=[dict(tokens=["w1", "w2", "w3"],
                      source_factors=[["s0_1", "s0_2", "s0_3"], ["s1_0", "s1_1", "zzz"]],
                      source_prefix=["w4"])]),
    # BASELINE configs[0]: tiny, greedy, 16 sentences of length 32
    dict(name="tiny_greedy_16x32", config="tiny", beam=1,
         inputs=_inputs(_sentences(13, 16, W7996, lo=32, hi=32))),
    dict(name="tiny_beam5", config="tiny", beam=5,
         inputs=_inputs(_sentences(17, 2, W7996, lo=6, hi=10))),
]


# ----------------------------------------------------------------- scale
# The BASELINE.json configs the bench measures, for the
# reference-generated beam traces in tests/golden/scale_*.npz: the GPU tests
# teacher-force the product's bench kernels along these traces.
BIG66 = dict(src_vocab_size=32000, trg_vocab_size=32000, d_model=1024, heads=16, ff_dim=4096,
             encoder_layers=6, decoder_layers=6, decoder_kind="self_attention", max_seq_len=128)
BASE66 = dict(BIG66, d_model=512, heads=8, ff_dim=2048)
BIG_SSRU = dict(BIG66, encoder_layers=20, decoder_layers=2, decoder_kind="ssru")

SCALE_CONFIGS = {"big": dict(seed=13, config=BIG66),
                 "base": dict(seed=13, config=BASE66),
                 "big_ssru": dict(seed=13, config=BIG_SSRU)}

# (name, config, beam, alpha, source lengths, shortlist top-k or None)
SCALE_TRACES = [
    dict(name="big_beam5", config="big", beam=5, alpha=1.0, lengths=[30, 19], seed=101),
    dict(name="big_greedy", config="big", beam=1, alpha=1.0, lengths=[30], seed=102),
    dict(name="base_beam5", config="base", beam=5, alpha=1.0, lengths=[30, 13], seed=103),
    dict(name="big_ssru_beam5_sl200", config="big_ssru", beam=5, alpha=1.0, lengths=[30, 24],
         seed=104, shortlist=200),
    dict(name="big_ssru_greedy_sl200", config="big_ssru", beam=1, alpha=1.0, lengths=[30],
         seed=105, shortlist=200),
]
# log-prob rows kept per trace (the rest of the trace keeps only fed tokens
# and parents): early steps, the middle, and the last (forced-EOS) step
SCALE_KEEP_STEPS = (0, 1, 2, 7, 23, 41, "last")
SCALE_TOPN, SCALE_RANDN = 16, 256
# base 6-6 beam 5: whole-record fp32 parity subsample (north star: >= 99 %
# of output sequences identical in fp32 mode)
BASE_RECORDS = dict(config="base", beam=5, alpha=1.0, n=6, seed=106, lo=4, hi=30)


def scale_sentences(seed, lengths, V):
    """SURVEY §8d synthetic sources: ids uniform in 4..V-1, tokens w{id-4}."""
    rng = np.random.default_rng(seed)
    return [[f"w{int(i)}" for i in rng.integers(0, V - 4, size=n)] for n in lengths]


def synthetic_shortlist_rows(V: int, k: int = 200, seed: int = 7) -> dict:
    """every source id 4..V-1 gets k distinct target ids drawn
    from 4..V-1 with default_rng(seed) (first k distinct of an oversampled
    draw, kept in draw order, returned sorted as Shortlist rows are).
    Shared by the golden generator, the tests and bench.py."""
    rng = np.random.default_rng(seed)
    draw = rng.integers(4, V, size=(V - 4, k + k // 2 + 16))
    rows = {}
    for i in range(V - 4):
        u, first = np.unique(draw[i], return_index=True)
        pick = u[np.argsort(first)][:k]
        if pick.size < k:  # pragma: no cover - oversampling makes this vanishingly rare
            extra = np.setdiff1d(np.arange(4, V), pick)[: k - pick.size]
            pick = np.concatenate([pick, extra])
        rows[i + 4] = np.sort(pick).astype(np.int64)
    return rows
