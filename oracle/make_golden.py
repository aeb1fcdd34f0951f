"""Generate tests/golden/ fixtures by running the REFERENCE implementation.

Run in the build container only (it needs /root/reference):

    python oracle/make_golden.py

It copies /root/reference/pkg/src to a scratch dir (so nothing is written
into the read-only reference tree), imports `skiff` from there, and records
on seeded inputs:

  * kernels.npz   — matmul / layer_norm / softmax / log_softmax / sigmoid /
                    multi-head attention outputs (kernels.py:167-547)
  * params.json   — per-parameter float64 checksums of init_params for every
                    fixture config (model.py:244-265)
  * steps_<cfg>.npz — teacher-forced decode_step logits along a fixed token
                    path, plus select_rows reorders (model.py:521-585, 316-330)
  * search.json   — translate() records for greedy / beam / alpha / shortlist /
                    NVS / prefix / strip / chunking / error cases
                    (search.py:275-468)
  * beam_trace_<cfg>.npz — per-step lp, alive scores and picks of a beam run,
                    captured by wrapping Model.decode_step and
                    DecodeState.select_rows (never editing the reference)
  * scale_<trace>.npz — the same capture at the BENCH configs (big 6-6,
                    base 6-6, big 20-2 SSRU + top-200 shortlist; beam 5 and
                    greedy): every step's fed tokens and parents, and at a few
                    steps the log-probs of each row's top-16 columns plus 256
                    random active columns (the full rows would be MBs); the
                    final hypothesis.  `python oracle/make_golden.py scale`
  * records_base.json — translate() records of the base 6-6 beam-5
                    subsample (fp32 whole-sequence parity)
  * refdir_<cfg>/ + refdir_records.json — model directories written by the
                    reference's own save_model_dir (config, SKP1 params.bin,
                    vocab JSON incl. factor vocabularies) and the records the
                    reference's translate() produces after loading them back
                    with its load_model_dir (checkpoint.py:316-353): the
                    product must read these directories unchanged.
                    `python oracle/make_golden.py modeldirs`
  * quant.npz + quant_records.json — the int8 feed-forward path
                    (quant.py): quantize_rows / QuantizedLinear outputs on
                    seeded matrices, and translate() records of models
                    swapped with quantize_model.  `... make_golden.py quant`

The oracle (oracle/skiff_oracle.py) is then checked against these files by
tests/test_oracle_golden.py; the CUDA path is checked against the oracle and
against these files by the -m gpu tests.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
from oracle.fixture_configs import (BASE_RECORDS, CONFIGS, SCALE_CONFIGS,  # noqa: E402
                                    SCALE_KEEP_STEPS, SCALE_RANDN, SCALE_TOPN, SCALE_TRACES,
                                    SEARCH_CASES, make_words, scale_sentences,
                                    synthetic_shortlist_rows)


def import_reference():
    src = Path("/root/reference/pkg/src")
    if not src.is_dir():
        raise SystemExit("make_golden.py needs /root/reference (build container only)")
    tmp = Path(tempfile.mkdtemp(prefix="skiff_ref_"))
    shutil.copytree(src, tmp / "src")
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp / "numba"))
    sys.path.insert(0, str(tmp / "src"))
    import skiff  # noqa: F401
    return tmp


def ref_model(name):
    from skiff.model import Model, ModelConfig, SourceFactorSpec, TargetFactorSpec
    spec = CONFIGS[name] if name in CONFIGS else SCALE_CONFIGS[name]
    cfg = dict(spec["config"])
    cfg["source_factor_specs"] = [SourceFactorSpec(*s) for s in cfg.get("source_factor_specs", [])]
    cfg["target_factor_specs"] = [TargetFactorSpec(v) for v in cfg.get("target_factor_specs", [])]
    return Model(ModelConfig(**cfg), seed=spec["seed"])


def ref_vocabs(name):
    from skiff.vocab import FACTOR_SPECIALS, SPECIALS, Vocabulary
    spec = CONFIGS[name] if name in CONFIGS else SCALE_CONFIGS[name]
    cfg = spec["config"]
    src = Vocabulary(SPECIALS + make_words(cfg["src_vocab_size"] - 4))
    trg = Vocabulary(SPECIALS + make_words(cfg["trg_vocab_size"] - 4))
    sfv = [Vocabulary(SPECIALS + [f"s{i}_{j}" for j in range(v - 4)])
           for i, (v, _, _) in enumerate(cfg.get("source_factor_specs", []))]
    tfv = [Vocabulary(FACTOR_SPECIALS + [f"F{i}_{j}" for j in range(v - 5)])
           for i, v in enumerate(cfg.get("target_factor_specs", []))]
    return SimpleNamespace(src_vocab=src, trg_vocab=trg, src_factor_vocabs=sfv,
                           trg_factor_vocabs=tfv)


def gen_kernels():
    import skiff.kernels as K
    from skiff.kernels import Tensor
    rng = np.random.default_rng(1234)
    out = {}
    a = rng.normal(size=(5, 37)).astype(np.float32)
    b = rng.normal(size=(37, 11)).astype(np.float32)
    out["mm_a"], out["mm_b"] = a, b
    out["mm_out"] = K.matmul(Tensor(a), Tensor(b)).data
    x = rng.normal(size=(4, 3, 24)).astype(np.float32) * 3 + 1
    g = rng.normal(size=(24,)).astype(np.float32)
    bb = rng.normal(size=(24,)).astype(np.float32)
    out["ln_x"], out["ln_g"], out["ln_b"] = x, g, bb
    out["ln_out"] = K.layer_norm(Tensor(x), Tensor(g), Tensor(bb)).data
    s = (rng.normal(size=(6, 50)) * 5).astype(np.float32)
    out["sm_x"] = s
    out["sm_out"] = K.softmax(Tensor(s)).data
    out["lsm_out"] = K.log_softmax(Tensor(s)).data
    out["sig_out"] = K.sigmoid(Tensor(s)).data
    q = rng.normal(size=(2, 5, 16)).astype(np.float32)
    kv = rng.normal(size=(2, 7, 16)).astype(np.float32)
    ws = [rng.normal(size=(16, 16)).astype(np.float32) * 0.3 for _ in range(4)]
    mask = np.where(np.arange(7)[None, :] >= np.array([5, 7])[:, None], -1e9, 0.0
                    ).astype(np.float32)[:, None, None, :]
    out["mha_q"], out["mha_kv"], out["mha_mask"] = q, kv, mask
    for i, n in enumerate(("wq", "wk", "wv", "wo")):
        out["mha_" + n] = ws[i]
    out["mha_out"] = K.multi_head_attention(Tensor(q), Tensor(kv), Tensor(kv), 4,
                                            *[Tensor(w) for w in ws], mask=mask).data
    np.savez_compressed(GOLDEN / "kernels.npz", **out)


def gen_params():
    out = {}
    for name in CONFIGS:
        m = ref_model(name)
        out[name] = {n: [float(t.data.astype(np.float64).sum()),
                         float(np.abs(t.data.astype(np.float64)).sum()),
                         float(t.data.ravel()[0]), float(t.data.ravel()[-1])]
                     for n, t in m.params.items()}
    (GOLDEN / "params.json").write_text(json.dumps(out, indent=0, sort_keys=True))


def gen_steps():
    """Teacher-forced decode along fixed paths, with a beam-style reorder."""
    for name, spec in CONFIGS.items():
        if not spec.get("steps"):
            continue
        m = ref_model(name)
        cfg = m.config
        rng = np.random.default_rng(99)
        B, L, T = 3, spec["steps"]["L"], spec["steps"]["T"]
        lens = np.array([L, max(1, L - 2), max(1, L // 2)])
        src = rng.integers(4, cfg.src_vocab_size, size=(B, L))
        for i, n in enumerate(lens):
            src[i, n:] = 0
        sf = [rng.integers(4, v.vocab_size, size=(B, L)) for v in cfg.source_factor_specs]
        fed = rng.integers(4, cfg.trg_vocab_size, size=(T, B))
        fed[0] = 2
        fedf = [rng.integers(4, v.vocab_size, size=(T, B)) for v in cfg.target_factor_specs]
        for f in fedf:
            f[0] = 4
        reorders = rng.integers(0, B, size=(T, B))
        st = m.decode_init(src, sf, lens)
        logits, facs = [], []
        for t in range(T):
            o = m.decode_step(st, fed[t], [f[t] for f in fedf])
            logits.append(o.surface.data)
            facs.append([f.data for f in o.factors])
            st.select_rows(reorders[t])
        out = dict(src=src, lens=lens, fed=fed, reorders=reorders,
                   logits=np.stack(logits).astype(np.float32))
        for i, s in enumerate(sf):
            out[f"src_factor{i}"] = s
        for k, f in enumerate(fedf):
            out[f"fed_factor{k}"] = f
            out[f"factor_logits{k}"] = np.stack([x[k] for x in facs]).astype(np.float32)
        if spec["steps"].get("teacher"):
            trg_in = fed.T[:1].repeat(1, 0)
            full = m.forward_sequence(src[:1], [s[:1] for s in sf], lens[:1],
                                      fed.T[:1], [f.T[:1] for f in fedf]).surface.data
            out["teacher_logits"] = full.astype(np.float32)
            del trg_in
        if len(cfg.source_factor_specs) == 0 and cfg.nvs_enabled:
            nvs = m.nvs_select(m.encode(src, sf, lens)[0], lens, 0.5, [0, 1, 3])
            out["nvs_ids"] = np.concatenate(nvs)
            out["nvs_counts"] = np.array([len(x) for x in nvs])
        np.savez_compressed(GOLDEN / f"steps_{name}.npz", **out)


def _records_to_json(records):
    return [dict(text=r.text, score=r.score, factors=r.factors, chunks=r.chunks,
                 forced_eos=r.forced_eos, error=r.error) for r in records]


def gen_search():
    from skiff.model import Model, ModelConfig
    from skiff.search import (NvsRestriction, SearchSettings, SentenceInput,
                              ShortlistRestriction, translate, chunk_input,
                              parse_input_line)
    from skiff.shortlist import Shortlist
    results = []
    for case in SEARCH_CASES:
        m = ref_model(case["config"])
        vocabs = ref_vocabs(case["config"])
        if case.get("max_seq_len"):
            cfg = ModelConfig(**{**vars(m.config), "max_seq_len": case["max_seq_len"]})
            m = Model(cfg, params=m.params)
        restriction = None
        if case.get("shortlist"):
            rows = {int(k): np.asarray(v, dtype=np.int64) for k, v in case["shortlist"].items()}
            restriction = ShortlistRestriction(Shortlist(rows))
        elif case.get("nvs") is not None:
            restriction = NvsRestriction(case["nvs"])
        settings = SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0),
                                  restriction=restriction, use_greedy=case.get("use_greedy"))
        inputs = [SentenceInput(**inp) for inp in case["inputs"]]
        records = translate(m, vocabs, inputs, settings)
        results.append(dict(name=case["name"], records=_records_to_json(records)))
    # host-logic goldens: parsing and chunking
    lines = ['a b   c', '{"text": "a b", "source_prefix": "<t>", "target_prefix": "x y", '
             '"target_prefix_factors": ["O O B"], "source_factors": ["P Q"]}',
             '{"text": "a", "extra": 1}', '{bad json', '{"text": 3}']
    parsed = []
    for ln in lines:
        try:
            s = parse_input_line(ln)
            parsed.append(dict(ok=True, tokens=s.tokens, source_factors=s.source_factors,
                               source_prefix=s.source_prefix, target_prefix=s.target_prefix,
                               target_prefix_factors=s.target_prefix_factors))
        except Exception as e:  # noqa: BLE001
            parsed.append(dict(ok=False, error=type(e).__name__))
    chunks = [[c.tokens for c in chunk_input(SentenceInput(tokens=list("abcdefghij"),
                                                           source_prefix=["<p>"]), 4)]]
    (GOLDEN / "search.json").write_text(json.dumps(
        dict(cases=results, parsed=parsed, chunks=chunks), indent=0))


def gen_beam_traces():
    """Wrap decode_step/select_rows to record what beam_search saw and chose."""
    import skiff.kernels as K
    from skiff.model import DecodeState, Model
    from skiff.search import SentenceInput, beam_search
    for name, spec in CONFIGS.items():
        bt = spec.get("beam_trace")
        if not bt:
            continue
        m = ref_model(name)
        vocabs = ref_vocabs(name)
        rng = np.random.default_rng(5)
        words = vocabs.src_vocab.tokens[4:]
        rec = {"lp": [], "parents": [], "fed": []}
        orig_step, orig_sel = Model.decode_step, DecodeState.select_rows

        def step(self, state, prev_ids, prev_factor_ids):
            out = orig_step(self, state, prev_ids, prev_factor_ids)
            rec["lp"].append(K.log_softmax(out.surface).data.copy())
            rec["fed"].append(np.asarray(prev_ids).copy())
            return out

        def sel(self, idx):
            rec["parents"].append(np.asarray(idx).copy())
            return orig_sel(self, idx)

        Model.decode_step, DecodeState.select_rows = step, sel
        try:
            toks = list(rng.choice(words, size=bt["L"]))
            hyp = beam_search(m, vocabs, SentenceInput(tokens=toks), bt["beam"],
                              length_alpha=bt.get("alpha", 1.0))
        finally:
            Model.decode_step, DecodeState.select_rows = orig_step, orig_sel
        keep = bt.get("keep_lp_steps")
        out = dict(src=np.array(vocabs.src_vocab.encode(toks)),
                   hyp_tokens=np.array(hyp.tokens, dtype=np.int64),
                   hyp_logprob=np.array(hyp.logprob), hyp_steps=np.array(hyp.steps),
                   hyp_forced=np.array(hyp.forced_eos),
                   n_steps=np.array(len(rec["lp"])))
        for t, (lp, fed) in enumerate(zip(rec["lp"], rec["fed"])):
            out[f"fed{t}"] = fed
            if keep is None or t in keep or t == len(rec["lp"]) - 1:
                out[f"lp{t}"] = lp
        for t, p in enumerate(rec["parents"]):
            out[f"parents{t}"] = p
        np.savez_compressed(GOLDEN / f"beam_trace_{name}.npz", **out)


def _capture(m, vocabs, inp, beam, alpha, restriction):
    """Run the reference's own greedy_search / beam_search on one sentence,
    recording every decode_step's fed tokens and log-probs and every
    select_rows' parents (wrapping, never editing, the reference)."""
    import skiff.kernels as K
    from skiff.model import DecodeState, Model
    from skiff.search import beam_search, greedy_search
    rec = {"lp": [], "fed": [], "parents": [], "active": None}
    orig_step, orig_sel = Model.decode_step, DecodeState.select_rows

    def step(self, state, prev_ids, prev_factor_ids):
        out = orig_step(self, state, prev_ids, prev_factor_ids)
        rec["lp"].append(K.log_softmax(out.surface).data.copy())
        rec["fed"].append(np.asarray(prev_ids).copy())
        rec["active"] = out.active_ids
        return out

    def sel(self, idx):
        rec["parents"].append(np.asarray(idx).copy())
        return orig_sel(self, idx)

    Model.decode_step, DecodeState.select_rows = step, sel
    try:
        if beam == 1:
            hyp = greedy_search(m, vocabs, inp, restriction, alpha)
        else:
            hyp = beam_search(m, vocabs, inp, beam, restriction, alpha)
    finally:
        Model.decode_step, DecodeState.select_rows = orig_step, orig_sel
    return hyp, rec


def gen_scale(only=None):
    """Beam traces at the bench configs, subset-compressed."""
    import time
    from skiff.search import SentenceInput, ShortlistRestriction
    from skiff.shortlist import Shortlist
    models = {}
    for tr in SCALE_TRACES:
        if only and tr["name"] not in only:
            continue
        t0 = time.time()
        if tr["config"] not in models:
            models.clear()
            models[tr["config"]] = (ref_model(tr["config"]), ref_vocabs(tr["config"]))
        m, vocabs = models[tr["config"]]
        V = m.config.trg_vocab_size
        K = tr["beam"]
        restriction = None
        if tr.get("shortlist"):
            restriction = ShortlistRestriction(Shortlist(synthetic_shortlist_rows(V, tr["shortlist"])))
        out = {}
        for s, toks in enumerate(scale_sentences(tr["seed"], tr["lengths"], V)):
            hyp, rec = _capture(m, vocabs, SentenceInput(tokens=toks), K, tr["alpha"], restriction)
            T = len(rec["lp"])
            active = rec["active"]
            fed = np.full((T, K), -1, np.int32)
            par = np.full((T, K), -1, np.int32)
            nrows = np.zeros(T, np.int32)
            for t in range(T):
                f = rec["fed"][t]
                fed[t, :len(f)] = f
                nrows[t] = len(f)
                if t < len(rec["parents"]):
                    par[t, :len(rec["parents"][t])] = rec["parents"][t]
            keep = sorted({T - 1 if k == "last" else k for k in SCALE_KEEP_STEPS if k == "last" or k < T})
            rng = np.random.default_rng(tr["seed"] * 1000 + s)
            A = rec["lp"][0].shape[1]
            top_col = np.zeros((len(keep), K, SCALE_TOPN), np.int32)
            top_lp = np.zeros((len(keep), K, SCALE_TOPN), np.float32)
            rnd_col = np.zeros((len(keep), SCALE_RANDN), np.int32)
            rnd_lp = np.zeros((len(keep), K, SCALE_RANDN), np.float32)
            for i, t in enumerate(keep):
                lp = rec["lp"][t]
                cols = np.sort(rng.choice(A, size=SCALE_RANDN, replace=False))
                rnd_col[i] = cols
                for r in range(lp.shape[0]):
                    # top-N by (lp desc, column asc): stable on ties
                    o = np.lexsort((np.arange(A), -lp[r]))[:SCALE_TOPN]
                    top_col[i, r], top_lp[i, r] = o, lp[r, o]
                    rnd_lp[i, r] = lp[r, cols]
            tok_of = (lambda c: active[c]) if active is not None else (lambda c: c)
            pre = f"s{s}_"
            out.update({pre + "src": np.array(vocabs.src_vocab.encode(toks), np.int32),
                        pre + "fed": fed, pre + "parents": par, pre + "nrows": nrows,
                        pre + "keep": np.array(keep, np.int32),
                        pre + "top_tok": tok_of(top_col).astype(np.int32), pre + "top_lp": top_lp,
                        pre + "rnd_tok": tok_of(rnd_col).astype(np.int32), pre + "rnd_lp": rnd_lp,
                        pre + "hyp_tokens": np.array(hyp.tokens, np.int32),
                        pre + "hyp_logprob": np.array(hyp.logprob),
                        pre + "hyp_steps": np.array(hyp.steps),
                        pre + "hyp_forced": np.array(hyp.forced_eos)})
            if active is not None:
                out[pre + "active"] = np.asarray(active, np.int32)
        out["n_sentences"] = np.array(len(tr["lengths"]))
        np.savez_compressed(GOLDEN / f"scale_{tr['name']}.npz", **out)
        print(f"scale {tr['name']}: {time.time() - t0:.1f} s", flush=True)


def gen_base_records():
    """translate() records, base 6-6 beam 5, for whole-sequence fp32 parity."""
    from skiff.search import SearchSettings, SentenceInput, translate
    br = BASE_RECORDS
    m, vocabs = ref_model(br["config"]), ref_vocabs(br["config"])
    V = m.config.trg_vocab_size
    rng = np.random.default_rng(br["seed"])
    lengths = [int(x) for x in rng.integers(br["lo"], br["hi"] + 1, size=br["n"])]
    sents = scale_sentences(br["seed"], lengths, V)
    recs = translate(m, vocabs, [SentenceInput(tokens=t) for t in sents],
                     SearchSettings(beam=br["beam"], length_alpha=br["alpha"]))
    (GOLDEN / "records_base.json").write_text(json.dumps(
        dict(inputs=sents, records=_records_to_json(recs)), indent=0))


REFDIR_CASES = [("srcfac", "srcfac_beam2"), ("ssru", "ssru_beam4"), ("factored", "factored_beam3")]


def gen_model_dirs():
    """Model directories saved by the reference + its records after reload."""
    from skiff.checkpoint import load_model_dir, save_model_dir
    from skiff.search import SearchSettings, SentenceInput, translate
    out = {}
    for cfg_name, case_name in REFDIR_CASES:
        d = GOLDEN / f"refdir_{cfg_name}"
        shutil.rmtree(d, ignore_errors=True)
        v = ref_vocabs(cfg_name)
        save_model_dir(d, ref_model(cfg_name), v.src_vocab, v.trg_vocab, v.src_factor_vocabs,
                       v.trg_factor_vocabs)
        md = load_model_dir(d)
        case = next(c for c in SEARCH_CASES if c["name"] == case_name)
        settings = SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0))
        recs = translate(md.model, md, [SentenceInput(**i) for i in case["inputs"]], settings)
        out[cfg_name] = dict(case=case_name, records=_records_to_json(recs))
    (GOLDEN / "refdir_records.json").write_text(json.dumps(out, indent=0))


QUANT_CASES = ["toy_beam3", "tiny_greedy_16x32", "ssru_greedy", "tiny_beam5"]


def gen_quant():
    """quant.py on seeded matrices + translate records of quantized models."""
    from skiff.kernels import Tensor
    from skiff.quant import QuantizedLinear, quantize_model, quantize_rows
    from skiff.search import SearchSettings, SentenceInput, translate
    rng = np.random.default_rng(2024)
    M, K1, N1 = 7, 256, 192
    x = rng.standard_normal((M, K1)).astype(np.float32)
    x[3] = 0.0                                      # all-zero row: scale 1
    x[4, :5] = [0.5, -0.5, 1.5, -2.5, 127.0]        # ties at the rounding boundary
    w1 = (rng.standard_normal((N1, K1)) * 0.05).astype(np.float32)
    b1 = rng.standard_normal(N1).astype(np.float32)
    w2 = (rng.standard_normal((K1, N1)) * 0.05).astype(np.float32)
    b2 = rng.standard_normal(K1).astype(np.float32)
    q1, s1 = quantize_rows(w1)
    q2, s2 = quantize_rows(w2)
    out1 = QuantizedLinear(q1, s1)(Tensor(x), Tensor(b1)).data
    h2 = np.maximum(out1, 0).astype(np.float32)
    out2 = QuantizedLinear(q2, s2)(Tensor(h2), Tensor(b2)).data
    qx, sx = quantize_rows(x)
    np.savez_compressed(GOLDEN / "quant.npz", x=x, w1=w1, b1=b1, w2=w2, b2=b2, q1=q1, s1=s1,
                        q2=q2, s2=s2, out1=out1, out2=out2, qx=qx, sx=sx)
    recs = {}
    for name in QUANT_CASES:
        case = next(c for c in SEARCH_CASES if c["name"] == name)
        m, vocabs = ref_model(case["config"]), ref_vocabs(case["config"])
        quantize_model(m)
        settings = SearchSettings(beam=case.get("beam", 1), length_alpha=case.get("alpha", 1.0))
        recs[name] = _records_to_json(translate(m, vocabs, [SentenceInput(**i) for i in case["inputs"]],
                                                settings))
    (GOLDEN / "quant_records.json").write_text(json.dumps(recs, indent=0))


def main():
    GOLDEN.mkdir(parents=True, exist_ok=True)
    tmp = import_reference()
    try:
        if len(sys.argv) > 1 and sys.argv[1] == "quant":
            gen_quant()
        elif len(sys.argv) > 1 and sys.argv[1] == "modeldirs":
            gen_model_dirs()
        elif len(sys.argv) > 1 and sys.argv[1] == "scale":
            gen_scale(set(sys.argv[2:]) or None)
            if len(sys.argv) == 2:
                gen_base_records()
        else:
            gen_kernels()
            gen_params()
            gen_steps()
            gen_search()
            gen_beam_traces()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    for p in sorted(GOLDEN.iterdir()):
        print(f"{p.name:32s} {p.stat().st_size:>9d} B")


if __name__ == "__main__":
    main()
