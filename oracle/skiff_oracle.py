"""CPU oracle for the translation hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference (`skiff`, mounted at
/root/reference/pkg/src/skiff) decode path: parameter init, encoder,
incremental decoder step (self-attention or SSRU), restricted output
projection, log-softmax, greedy and beam search with prefix forcing,
forced EOS and length-normalised final pick.  It exists only to CHECK the
CUDA product path: the only legal importers are `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs
of `bench.py`.  The product (`paper_2207_05851_b200`) never imports it.

Numerics follow the reference conventions exactly:
  * every matrix product accumulates in float64 and rounds once to float32
    (kernels.py:167-176);
  * layer norm: population variance, eps 1e-5 (kernels.py:298-324);
  * (log-)softmax max-shifted in float32 (kernels.py:273-295);
  * attention scale 1/sqrt(d_h) applied after QK^T, additive -1e9 masks
    (kernels.py:510-517, 23);
  * beam hypothesis scores are float64 sums of float32 log-probs
    (search.py:353-358, 373).

Parity pinning: `oracle/make_golden.py` runs the reference itself (in the
build container, where /root/reference exists) on seeded inputs and
commits the outputs under `tests/golden/`; `tests/test_oracle_golden.py`
checks this oracle against those vectors bit-for-bit (integer outputs) and
to 1e-6 (float outputs).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
F64 = np.float64

# vocab.py:17-21 — pinned special ids
PAD_ID, UNK_ID, BOS_ID, EOS_ID, SHIFT_ID = 0, 1, 2, 3, 4
# kernels.py:23
NEG_INF = -1.0e9


class OracleError(Exception):
    """Raised where the reference raises one of its SkiffError subclasses.
    `kind` names the reference class (InputError, ConfigError, ShapeError)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ------------------------------------------------------------------ numerics

def mm64(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """float64-accumulated product rounded once to float32 (kernels.py:167-176).
    The reference casts both operands on every call; so do we (same cost
    profile for the CPU baseline)."""
    return np.matmul(a.astype(F64), b.astype(F64)).astype(F32)


def linear(x, w, b=None):
    """x @ w.T (+ b), w stored (out, in) (kernels.py:479-484)."""
    y = mm64(x, w.T)
    if b is not None:
        y = y + b
    return y


def layer_norm(x, gain, bias, eps=1e-5):
    """kernels.py:298-324 — population variance, eps rounded to x.dtype."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = np.mean(xc * xc, axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + np.asarray(eps, dtype=x.dtype))
    return (xc * inv) * gain + bias


def softmax(x):
    """kernels.py:273-284."""
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def log_softmax(x):
    """kernels.py:287-295."""
    s = x - x.max(axis=-1, keepdims=True)
    return s - np.log(np.exp(s).sum(axis=-1, keepdims=True))


def sigmoid(x):
    """Sign-split logistic (kernels.py:253-260)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def heads_split(x, h):
    """(B, L, d) -> (B, h, L, d/h) (kernels.py:494-500)."""
    b, n, d = x.shape
    return x.reshape(b, n, h, d // h).transpose(0, 2, 1, 3)


def heads_merge(x):
    """(B, h, L, dh) -> (B, L, h*dh) (kernels.py:503-507)."""
    b, h, n, dh = x.shape
    return x.transpose(0, 2, 1, 3).reshape(b, n, h * dh)


def attend(qh, kh, vh, mask):
    """Scaled dot-product attention (kernels.py:510-517)."""
    scale = np.asarray(1.0 / math.sqrt(qh.shape[-1]), dtype=qh.dtype)
    s = mm64(qh, kh.transpose(0, 1, 3, 2)) * scale
    if mask is not None:
        s = s + mask.astype(s.dtype)
    return mm64(softmax(s), vh)


def causal(n):
    """kernels.py:487-491."""
    m = np.zeros((n, n), dtype=F32)
    m[np.triu_indices(n, k=1)] = NEG_INF
    return m


def posenc(length, dim, offset=0):
    """Interleaved sin/cos codes computed in float64, cast to float32
    (model.py:161-171)."""
    pos = np.arange(offset, offset + length, dtype=F64)[:, None]
    half = (dim + 1) // 2
    freq = np.exp(-math.log(10000.0) * (2.0 * np.arange(half) / dim))[None, :]
    ang = pos * freq
    pe = np.zeros((length, 2 * half), dtype=F64)
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang)
    return pe[:, :dim].astype(F32)


def pad_bias(lengths, width):
    """(B,1,1,L) additive -1e9 past each length (model.py:174-179)."""
    pad = np.arange(width)[None, :] >= np.asarray(lengths)[:, None]
    return np.where(pad, NEG_INF, 0.0).astype(F32)[:, None, None, :]


# -------------------------------------------------------------------- config

@dataclass
class OConfig:
    """Mirror of ModelConfig (model.py:53-101).  source_factor_specs is a
    list of (vocab_size, dim, combine); target_factor_specs a list of vocab
    sizes."""
    src_vocab_size: int
    trg_vocab_size: int
    d_model: int = 512
    heads: int = 8
    ff_dim: int = 2048
    encoder_layers: int = 6
    decoder_layers: int = 6
    decoder_kind: str = "self_attention"
    source_factor_specs: list = field(default_factory=list)
    target_factor_specs: list = field(default_factory=list)
    nvs_enabled: bool = False
    max_seq_len: int = 128

    @classmethod
    def of(cls, cfg) -> "OConfig":
        """Accept any ModelConfig-shaped object (duck-typed)."""
        if isinstance(cfg, OConfig):
            return cfg
        sf = [(int(s.vocab_size), int(s.dim), str(s.combine)) if not isinstance(s, tuple)
              else tuple(s) for s in cfg.source_factor_specs]
        tf = [int(s.vocab_size) if not isinstance(s, int) else s
              for s in cfg.target_factor_specs]
        return cls(cfg.src_vocab_size, cfg.trg_vocab_size, cfg.d_model, cfg.heads,
                   cfg.ff_dim, cfg.encoder_layers, cfg.decoder_layers, cfg.decoder_kind,
                   sf, tf, bool(cfg.nvs_enabled), cfg.max_seq_len)

    @property
    def surface_dim(self) -> int:
        return self.d_model - sum(d for _, d, c in self.source_factor_specs if c == "concat")


def param_layout(cfg: OConfig) -> list[tuple[str, str, tuple]]:
    """(name, init kind, shape) in the reference's draw order
    (model.py:182-241).  Kinds: mat / emb / one / zero."""
    d, ff = cfg.d_model, cfg.ff_dim
    out: list[tuple[str, str, tuple]] = []

    def ln(p):
        out.append((p + ".gain", "one", (d,)))
        out.append((p + ".bias", "zero", (d,)))

    def att(p):
        out.extend((f"{p}.{w}", "mat", (d, d)) for w in ("wq", "wk", "wv", "wo"))

    def ffn(p):
        out.extend([(p + ".w1", "mat", (ff, d)), (p + ".b1", "zero", (ff,)),
                    (p + ".w2", "mat", (d, ff)), (p + ".b2", "zero", (d,))])

    out.append(("embed.src.surface", "emb", (cfg.src_vocab_size, cfg.surface_dim)))
    for i, (v, dim, _) in enumerate(cfg.source_factor_specs):
        out.append((f"embed.src.factor{i}", "emb", (v, dim)))
    out.append(("embed.trg.surface", "emb", (cfg.trg_vocab_size, d)))
    for i, v in enumerate(cfg.target_factor_specs):
        out.append((f"embed.trg.factor{i}", "emb", (v, d)))
    for i in range(cfg.encoder_layers):
        p = f"encoder.layer{i}"
        att(p + ".self_attn"); ln(p + ".self_attn_norm")
        ffn(p + ".ffn"); ln(p + ".ffn_norm")
    for i in range(cfg.decoder_layers):
        p = f"decoder.layer{i}"
        if cfg.decoder_kind == "ssru":
            out.extend([(p + ".ssru.wf", "mat", (d, d)), (p + ".ssru.bf", "zero", (d,)),
                        (p + ".ssru.w", "mat", (d, d))])
            ln(p + ".ssru_norm")
        else:
            att(p + ".self_attn"); ln(p + ".self_attn_norm")
        att(p + ".cross_attn"); ln(p + ".cross_attn_norm")
        ffn(p + ".ffn"); ln(p + ".ffn_norm")
    ln("decoder.final_norm")
    for i, v in enumerate(cfg.target_factor_specs):
        out.append((f"output.factor{i}.w", "mat", (v, d)))
        out.append((f"output.factor{i}.b", "zero", (v,)))
    if cfg.nvs_enabled:
        out.append(("nvs.w", "mat", (cfg.trg_vocab_size, d)))
        out.append(("nvs.b", "zero", (cfg.trg_vocab_size,)))
    return out


def init_params(cfg: OConfig, seed: int = 13) -> dict[str, np.ndarray]:
    """Deterministic init from one default_rng(seed) stream (model.py:244-265):
    Xavier-uniform matrices, N(0, 0.3/sqrt(dim)) embeddings, ones/zeros."""
    rng = np.random.default_rng(seed)
    params = {}
    for name, kind, shape in param_layout(cfg):
        if kind == "mat":
            lim = math.sqrt(6.0 / (shape[0] + shape[1]))
            a = rng.uniform(-lim, lim, size=shape)
        elif kind == "emb":
            a = rng.normal(0.0, 0.3 / math.sqrt(shape[1]), size=shape)
        elif kind == "one":
            a = np.ones(shape)
        else:
            a = np.zeros(shape)
        params[name] = np.asarray(a, dtype=F32)
    return params


# --------------------------------------------------------------------- model

class OState:
    """Per-batch incremental decoder state (model.py:290-330)."""

    def __init__(self, enc, bias, cross, active_ids):
        self.enc = enc
        self.bias = bias
        self.cross = cross          # list of (kh, vh) per decoder layer
        self.kv = [None] * len(cross)    # (kh, vh) self-attn caches
        self.cell = [None] * len(cross)  # SSRU cells
        self.active_ids = active_ids
        self.step = 0

    def select_rows(self, idx):
        """Gather every per-row state by index (model.py:316-330)."""
        idx = np.asarray(idx, dtype=np.int64)
        self.enc = self.enc[idx]
        self.bias = self.bias[idx]
        self.cross = [(k[idx], v[idx]) for k, v in self.cross]
        self.kv = [None if c is None else (c[0][idx], c[1][idx]) for c in self.kv]
        self.cell = [None if c is None else c[idx] for c in self.cell]


def ssru_step(h, c_prev, wf, bf, w):
    """model.py:268-272: f = sigmoid(Wf h + bf); c = f*c + (1-f)*(W h);
    returns (relu(c), c)."""
    f = sigmoid(linear(h, wf, bf))
    c = f * c_prev + (np.asarray(1.0, dtype=F32) - f) * linear(h, w)
    return np.maximum(c, 0), c


class OracleModel:
    """Encoder/decoder forward in the reference's numerics (model.py:343-585)."""

    def __init__(self, cfg, params: dict[str, np.ndarray]):
        self.cfg = OConfig.of(cfg)
        self.p = params

    # model.py:370-397
    def embed_src(self, ids, factor_ids):
        c, p = self.cfg, self.p
        x = p["embed.src.surface"][ids] + posenc(ids.shape[1], c.surface_dim)[None]
        concat = [p[f"embed.src.factor{i}"][factor_ids[i]]
                  for i, (_, _, comb) in enumerate(c.source_factor_specs) if comb == "concat"]
        if concat:
            x = np.concatenate([x] + concat, axis=-1)
        for i, (_, _, comb) in enumerate(c.source_factor_specs):
            if comb == "sum":
                x = x + p[f"embed.src.factor{i}"][factor_ids[i]]
        return x

    # model.py:399-410
    def embed_trg(self, ids, factor_ids, offset=0):
        p = self.p
        x = p["embed.trg.surface"][ids] + posenc(ids.shape[1], self.cfg.d_model, offset)[None]
        for i in range(len(self.cfg.target_factor_specs)):
            x = x + p[f"embed.trg.factor{i}"][factor_ids[i]]
        return x

    def _mha(self, q_in, kv_in, base, mask):
        p, h = self.p, self.cfg.heads
        qh = heads_split(linear(q_in, p[base + ".wq"]), h)
        kh = heads_split(linear(kv_in, p[base + ".wk"]), h)
        vh = heads_split(linear(kv_in, p[base + ".wv"]), h)
        return linear(heads_merge(attend(qh, kh, vh, mask)), p[base + ".wo"])

    def _ffn(self, x, base):
        # model.py:432-440
        p = self.p
        h = layer_norm(x, p[base + "_norm.gain"], p[base + "_norm.bias"])
        h = np.maximum(linear(h, p[base + ".w1"], p[base + ".b1"]), 0)
        return linear(h, p[base + ".w2"], p[base + ".b2"])

    # model.py:414-430 — pre-norm, no final encoder LN
    def encode(self, ids, factor_ids, lengths):
        p = self.p
        x = self.embed_src(ids, factor_ids)
        bias = pad_bias(lengths, ids.shape[1])
        for i in range(self.cfg.encoder_layers):
            b = f"encoder.layer{i}"
            h = layer_norm(x, p[b + ".self_attn_norm.gain"], p[b + ".self_attn_norm.bias"])
            x = x + self._mha(h, h, b + ".self_attn", bias)
            x = x + self._ffn(x, b + ".ffn")
        return x, bias

    # model.py:496-517
    def nvs_select(self, enc, lengths, threshold, always_include):
        keep = np.arange(enc.shape[1])[None, :] < np.asarray(lengths)[:, None]
        pooled = np.where(keep[:, :, None], enc, -np.inf).max(axis=1)
        probs = sigmoid(linear(pooled, self.p["nvs.w"], self.p["nvs.b"]))
        forced = np.asarray(sorted(set(int(i) for i in always_include)), dtype=np.int64)
        return [np.union1d(np.flatnonzero(r > threshold), forced).astype(np.int64)
                for r in probs]

    # model.py:521-534
    def decode_init(self, ids, factor_ids, lengths, active_ids=None):
        enc, bias = self.encode(ids, factor_ids, lengths)
        cross = []
        for i in range(self.cfg.decoder_layers):
            b = f"decoder.layer{i}.cross_attn"
            cross.append((heads_split(linear(enc, self.p[b + ".wk"]), self.cfg.heads),
                          heads_split(linear(enc, self.p[b + ".wv"]), self.cfg.heads)))
        return OState(enc, bias, cross, active_ids)

    # model.py:536-585 — returns (surface logits (B, A) f32, factor logits)
    def decode_step(self, st: OState, prev_ids, prev_factor_ids):
        c, p = self.cfg, self.p
        if st.step >= 2 * c.max_seq_len + 10:
            raise OracleError("ShapeError", "decode ran past the hard position limit")
        x = self.embed_trg(np.asarray(prev_ids)[:, None],
                           [np.asarray(f)[:, None] for f in prev_factor_ids], st.step)
        for i in range(c.decoder_layers):
            b = f"decoder.layer{i}"
            if c.decoder_kind == "ssru":
                h = layer_norm(x, p[b + ".ssru_norm.gain"], p[b + ".ssru_norm.bias"])
                if st.cell[i] is None:
                    st.cell[i] = np.zeros_like(h)
                out, st.cell[i] = ssru_step(h, st.cell[i], p[b + ".ssru.wf"],
                                            p[b + ".ssru.bf"], p[b + ".ssru.w"])
                x = x + out
            else:
                h = layer_norm(x, p[b + ".self_attn_norm.gain"], p[b + ".self_attn_norm.bias"])
                qh = heads_split(linear(h, p[b + ".self_attn.wq"]), c.heads)
                kh = heads_split(linear(h, p[b + ".self_attn.wk"]), c.heads)
                vh = heads_split(linear(h, p[b + ".self_attn.wv"]), c.heads)
                if st.kv[i] is not None:
                    kh = np.concatenate([st.kv[i][0], kh], axis=2)
                    vh = np.concatenate([st.kv[i][1], vh], axis=2)
                st.kv[i] = (kh, vh)
                x = x + linear(heads_merge(attend(qh, kh, vh, None)), p[b + ".self_attn.wo"])
            h = layer_norm(x, p[b + ".cross_attn_norm.gain"], p[b + ".cross_attn_norm.bias"])
            qh = heads_split(linear(h, p[b + ".cross_attn.wq"]), c.heads)
            ck, cv = st.cross[i]
            x = x + linear(heads_merge(attend(qh, ck, cv, st.bias)), p[b + ".cross_attn.wo"])
            x = x + self._ffn(x, b + ".ffn")
        h = layer_norm(x, p["decoder.final_norm.gain"], p["decoder.final_norm.bias"])
        h = h.reshape(h.shape[0], h.shape[2])
        emb = p["embed.trg.surface"]
        rows = emb if st.active_ids is None else emb[st.active_ids]
        surface = mm64(h, rows.T)
        factors = [linear(h, p[f"output.factor{k}.w"], p[f"output.factor{k}.b"])
                   for k in range(len(c.target_factor_specs))]
        st.step += 1
        return surface, factors

    # model.py:444-492 (teacher forced; second oracle for step parity)
    def forward_sequence(self, src, src_f, lens, trg_in, trg_f):
        c, p = self.cfg, self.p
        enc, bias = self.encode(src, src_f, lens)
        x = self.embed_trg(trg_in, trg_f)
        for i in range(c.decoder_layers):
            b = f"decoder.layer{i}"
            if c.decoder_kind == "ssru":
                h = layer_norm(x, p[b + ".ssru_norm.gain"], p[b + ".ssru_norm.bias"])
                cell = np.zeros((h.shape[0], 1, h.shape[2]), dtype=F32)
                outs = []
                for t in range(h.shape[1]):
                    o, cell = ssru_step(h[:, t:t + 1], cell, p[b + ".ssru.wf"],
                                        p[b + ".ssru.bf"], p[b + ".ssru.w"])
                    outs.append(o)
                x = x + np.concatenate(outs, axis=1)
            else:
                h = layer_norm(x, p[b + ".self_attn_norm.gain"], p[b + ".self_attn_norm.bias"])
                x = x + self._mha(h, h, b + ".self_attn", causal(h.shape[1]))
            h = layer_norm(x, p[b + ".cross_attn_norm.gain"], p[b + ".cross_attn_norm.bias"])
            x = x + self._mha(h, enc, b + ".cross_attn", bias)
            x = x + self._ffn(x, b + ".ffn")
        h = layer_norm(x, p["decoder.final_norm.gain"], p["decoder.final_norm.bias"])
        return mm64(h, p["embed.trg.surface"].T)


# -------------------------------------------------------------------- search

@dataclass
class OHyp:
    """Finished hypothesis (search.py:62-75)."""
    tokens: list
    factors: list
    logprob: float
    steps: int
    forced_eos: bool

    def normalized(self, alpha):
        return self.logprob / (self.steps ** alpha)


@dataclass
class OChunk:
    """Id-encoded chunk: everything the search needs from one SentenceInput
    chunk after vocabulary lookup (search.py:194-226)."""
    src_ids: list
    src_factor_ids: list = field(default_factory=list)   # per stream, padded under the prefix
    prefix_ids: list = field(default_factory=list)
    prefix_factor_ids: list = field(default_factory=list)


def max_output_len(src_len):
    """search.py:231-232."""
    return 2 * src_len + 10


def column_of(active, token):
    """search.py:245-251."""
    if active is None:
        return token
    col = int(np.searchsorted(active, token))
    if col >= active.size or active[col] != token:
        raise OracleError("ConfigError", f"token id {token} missing from the restricted vocabulary")
    return col


def resolve_active(model: OracleModel, state: OState, chunk: OChunk, restriction):
    """search.py:235-242 + ShortlistRestriction/NvsRestriction.resolve
    (search.py:88-110) + validate_active_ids (model.py:333-340).
    restriction is None, ("shortlist", rows_dict) or ("nvs", threshold)."""
    if restriction is None:
        return None
    extra = np.array([PAD_ID, UNK_ID, EOS_ID] + list(chunk.prefix_ids), dtype=np.int64)
    kind, arg = restriction
    if kind == "shortlist":
        parts = [arg[i] for i in set(int(i) for i in chunk.src_ids) if i in arg]
        ids = np.unique(np.concatenate(parts)) if parts else np.empty(0, np.int64)
        ids = np.union1d(ids, extra)
    else:
        (ids,) = model.nvs_select(state.enc, np.array([len(chunk.src_ids)]), arg, extra)
    ids = np.unique(np.asarray(ids, dtype=np.int64))
    if ids.size == 0:
        raise OracleError("ConfigError", "restricted output vocabulary is empty")
    if ids[0] < 0 or ids[-1] >= model.cfg.trg_vocab_size:
        raise OracleError("ConfigError", "restricted vocabulary ids out of range")
    return ids


def _factor_pick(fac_logits, row, t, prefix_factor_ids, n):
    """search.py:261-272 — greedy factor per stream, prefix override at t-1."""
    out = []
    for k in range(n):
        if t >= 1 and k < len(prefix_factor_ids) and t - 1 < len(prefix_factor_ids[k]):
            out.append(int(prefix_factor_ids[k][t - 1]))
        else:
            out.append(int(np.argmax(fac_logits[k][row])))
    return out


def _start(model, chunk, restriction):
    ids = np.array([chunk.src_ids], dtype=np.int64)
    fids = [np.array([f], dtype=np.int64) for f in chunk.src_factor_ids]
    lengths = np.array([len(chunk.src_ids)], dtype=np.int64)
    max_len = max_output_len(len(chunk.src_ids))
    if len(chunk.prefix_ids) > max_len - 1:
        raise OracleError("InputError", "target prefix does not fit the output budget")
    st = model.decode_init(ids, fids, lengths)
    st.active_ids = resolve_active(model, st, chunk, restriction)
    return st, max_len


def greedy(model: OracleModel, chunk: OChunk, restriction=None, trace=None) -> OHyp:
    """search.py:275-313.  trace, if a list, receives one dict per step."""
    st, max_len = _start(model, chunk, restriction)
    nf = len(model.cfg.target_factor_specs)
    prev, prev_f = [BOS_ID], [[SHIFT_ID] for _ in range(nf)]
    tokens, factors, logprob, forced = [], [[] for _ in range(nf)], 0.0, False
    for t in range(max_len):
        surface, fac = model.decode_step(st, np.array(prev), [np.array(f) for f in prev_f])
        lp = log_softmax(surface)[0]
        if t < len(chunk.prefix_ids):
            col = column_of(st.active_ids, chunk.prefix_ids[t])
        else:
            col = int(np.argmax(lp))
            if t == max_len - 1:
                eos = column_of(st.active_ids, EOS_ID)
                forced = col != eos
                col = eos
        token = int(st.active_ids[col]) if st.active_ids is not None else col
        if trace is not None:
            trace.append({"fed": list(prev), "lp": lp[None].copy(), "col": col})
        logprob += float(lp[col])
        ch = _factor_pick(fac, 0, t, chunk.prefix_factor_ids, nf)
        for k in range(nf):
            factors[k].append(ch[k])
        if token == EOS_ID:
            return OHyp(tokens, factors, logprob, t + 1, forced)
        tokens.append(token)
        prev, prev_f = [token], [[c] for c in ch]
    raise AssertionError("final step always emits EOS")


def beam_select(lp, alive_scores, beam, active, forced_col=None):
    """One beam selection (search.py:345-369): candidates (parent, col) with
    float64 score alive[parent] + lp[parent, col], ordered by
    (score desc, token asc, parent asc); returns the first `beam` as
    (parent, col, score) triples.  forced_col restricts each row to one
    column (prefix or final forced EOS)."""
    n_rows, n_cols = lp.shape
    if forced_col is not None:
        sc = np.array([alive_scores[b] + lp[b, forced_col] for b in range(n_rows)])
        par = np.arange(n_rows)
        cols = np.full(n_rows, forced_col)
    else:
        sc = (np.asarray(alive_scores, dtype=F64)[:, None] + lp).ravel()
        par = np.repeat(np.arange(n_rows), n_cols)
        cols = np.tile(np.arange(n_cols), n_rows)
    tok = active[cols] if active is not None else cols
    order = np.lexsort((par, tok, -sc))[:beam]
    return [(int(par[i]), int(cols[i]), float(alive_scores[par[i]]) + float(lp[par[i], cols[i]]))
            for i in order]


def beam(model: OracleModel, chunk: OChunk, beam_size: int, restriction=None,
         alpha: float = 1.0, trace=None, normalize=log_softmax, max_steps=None,
         timings=None) -> OHyp:
    """search.py:325-394.  trace, if a list, receives per step the fed
    tokens, the fp32 log-prob matrix, alive scores and the selection.
    `normalize` maps the step's surface logits to log-probs (identity when a
    test feeds log-probs directly, as the kernel's lp_in mode does).
    max_steps / timings bound the run for CPU-baseline sampling: timings
    receives the wall time of decode_init and of every executed step."""
    import time as _time
    t_start = _time.perf_counter()
    if beam_size < 1:
        raise OracleError("ConfigError", f"beam size must be at least 1, got {beam_size}")
    st, max_len = _start(model, chunk, restriction)
    nf = len(model.cfg.target_factor_specs)
    active = st.active_ids
    alive = [([], [[] for _ in range(nf)], 0.0)]
    finished: list[OHyp] = []
    prev, prev_f = [BOS_ID], [[SHIFT_ID] for _ in range(nf)]
    npre = len(chunk.prefix_ids)
    if timings is not None:
        timings.append(_time.perf_counter() - t_start)
    for t in range(max_len):
        if max_steps is not None and t >= max_steps:
            return None
        t0 = _time.perf_counter()
        surface, fac = model.decode_step(st, np.array(prev), [np.array(f) for f in prev_f])
        lp = normalize(surface)
        final_force = t == max_len - 1 and t >= npre
        forced_col = None
        if t < npre or final_force:
            forced_col = column_of(active, EOS_ID if final_force else chunk.prefix_ids[t])
        scores = [h[2] for h in alive]
        picks = beam_select(lp, scores, beam_size, active, forced_col)
        if trace is not None:
            trace.append({"fed": list(prev), "lp": lp.copy(), "scores": list(scores),
                          "forced_col": forced_col, "picks": picks})
        new_alive, parents, nxt, nxt_f = [], [], [], []
        for parent, col, score in picks:
            token = int(active[col]) if active is not None else col
            ch = _factor_pick(fac, parent, t, chunk.prefix_factor_ids, nf)
            toks, facs, _ = alive[parent]
            facs = [facs[k] + [ch[k]] for k in range(nf)]
            if token == EOS_ID:
                forced = final_force and int(np.argmax(lp[parent])) != col
                finished.append(OHyp(list(toks), facs, score, t + 1, forced))
            else:
                new_alive.append((toks + [token], facs, score))
                parents.append(parent)
                nxt.append(token)
                nxt_f.append(ch)
        if not new_alive:
            break
        st.select_rows(parents)
        if timings is not None:
            timings.append(_time.perf_counter() - t0)
        alive = new_alive
        prev = nxt
        prev_f = [[c[k] for c in nxt_f] for k in range(nf)]
    best = finished[0]
    for h in finished[1:]:
        if h.normalized(alpha) > best.normalized(alpha):
            best = h
    return best


def run_chunk(model, chunk, beam_size=1, restriction=None, alpha=1.0, use_greedy=None):
    """search.py:399-409."""
    g = use_greedy if use_greedy is not None else beam_size == 1
    if g:
        if beam_size != 1:
            raise OracleError("ConfigError", "greedy decoding is incompatible with beam > 1")
        return greedy(model, chunk, restriction)
    return beam(model, chunk, beam_size, restriction, alpha)


def translate_ids(model, chunks_per_sentence, beam_size=1, restriction=None, alpha=1.0,
                  use_greedy=None):
    """search.py:412-451 at the id level: per sentence, decode every chunk
    independently and combine: tokens concatenated, score =
    sum(logprob) / sum(steps)^alpha.  Returns (tokens, score, forced, hyps)."""
    out = []
    for chunks in chunks_per_sentence:
        hyps = [run_chunk(model, c, beam_size, restriction, alpha, use_greedy) for c in chunks]
        tokens = [t for h in hyps for t in h.tokens]
        lp = sum(h.logprob for h in hyps)
        steps = sum(h.steps for h in hyps)
        out.append((tokens, lp / (steps ** alpha), any(h.forced_eos for h in hyps), hyps))
    return out


# ---------------------------------------------------------------- cost model

def decoder_step_macs(cfg, step, src_len, out_cols=None):
    """model.py:590-606 (V replaced by the active width when restricted)."""
    c = OConfig.of(cfg)
    d, ff = c.d_model, c.ff_dim
    inner = 2 * d * d if c.decoder_kind == "ssru" else 4 * d * d + 2 * (step + 1) * d
    cross = 2 * d * d + 2 * src_len * d
    v = c.trg_vocab_size if out_cols is None else out_cols
    return c.decoder_layers * (inner + cross + 2 * d * ff) + d * v + \
        sum(d * s for s in c.target_factor_specs)


def encoder_macs(cfg, src_len):
    """model.py:609-613."""
    c = OConfig.of(cfg)
    d, ff = c.d_model, c.ff_dim
    return c.encoder_layers * (4 * src_len * d * d + 2 * src_len * src_len * d
                               + 2 * src_len * d * ff)


def sentence_flops(cfg, src_len, rows_per_step, out_cols=None):
    """Algorithmic FLOPs of one translated chunk: 2 x MACs of encode, cross
    K/V once, and sum over steps of rows_t x decoder_step_cost
    (model.py:616-621)."""
    c = OConfig.of(cfg)
    macs = encoder_macs(c, src_len) + c.decoder_layers * 2 * src_len * c.d_model ** 2
    macs += sum(r * decoder_step_macs(c, t, src_len, out_cols)
                for t, r in enumerate(rows_per_step))
    return 2 * macs


def dumps_hyp(h: OHyp) -> str:
    return json.dumps({"tokens": h.tokens, "factors": h.factors, "logprob": h.logprob,
                       "steps": h.steps, "forced_eos": h.forced_eos})


# ----------------------------------------------------------- text-level glue

class OVocab:
    """Token<->id map with the pinned specials first (vocab.py:33-78)."""

    def __init__(self, tokens):
        self.tokens = list(tokens)
        self.ids = {t: i for i, t in enumerate(self.tokens)}

    def encode(self, toks):
        return [self.ids.get(t, UNK_ID) for t in toks]

    def decode(self, ids):
        return [self.tokens[i] for i in ids]


def chunk_sentence(inp: dict, max_seq_len: int) -> list[dict]:
    """search.py:164-191 on plain dicts (keys as SentenceInput fields)."""
    toks = inp.get("tokens", [])
    if not toks:
        raise OracleError("InputError", "empty input")
    sp = inp.get("source_prefix", [])
    if max_seq_len <= len(sp):
        raise OracleError("InputError", "source prefix leaves no room")
    budget = max_seq_len - len(sp)
    out = []
    for start in range(0, len(toks), budget):
        with_target = start == 0 or inp.get("prefix_all_chunks", False)
        out.append(dict(tokens=toks[start:start + budget],
                        source_factors=[s[start:start + budget] for s in inp.get("source_factors", [])],
                        source_prefix=list(sp),
                        target_prefix=list(inp.get("target_prefix", [])) if with_target else [],
                        target_prefix_factors=[list(s) for s in inp.get("target_prefix_factors", [])]
                        if with_target else []))
    return out


def encode_text_chunk(ch: dict, vocabs) -> OChunk:
    """search.py:194-226: ids of src prefix + body; factor streams PAD-padded
    under the prefix; target prefix (and its factors) through the target
    vocabularies (unknown -> UNK)."""
    npre = len(ch["source_prefix"])
    src = vocabs["src"].encode(ch["source_prefix"] + ch["tokens"])
    sf = [[PAD_ID] * npre + v.encode(s) for s, v in zip(ch["source_factors"], vocabs["src_f"])]
    pre = vocabs["trg"].encode(ch["target_prefix"])
    pref = [v.encode(s) for s, v in zip(ch["target_prefix_factors"], vocabs["trg_f"])]
    return OChunk(src, sf, pre, pref)


def translate_text(model: OracleModel, vocabs: dict, inputs: list[dict], beam_size=1,
                   alpha=1.0, restriction=None, use_greedy=None) -> list[dict]:
    """search.py:412-468: per-sentence records with in-band InputError."""
    cfg = model.cfg
    nf = len(cfg.target_factor_specs)
    recs = []
    for inp in inputs:
        try:
            for i, s in enumerate(inp.get("source_factors", [])):
                if len(s) != len(inp.get("tokens", [])):
                    raise OracleError("InputError", f"source factor stream {i} length mismatch")
            if len(inp.get("source_factors", [])) != len(cfg.source_factor_specs):
                raise OracleError("InputError", "model expects a different number of "
                                                "source factor streams")
            if len(inp.get("target_prefix_factors", [])) > nf:
                raise OracleError("InputError", "too many target prefix factor streams")
            chunks = chunk_sentence(inp, cfg.max_seq_len)
            words, facs = [], [[] for _ in range(nf)]
            lp_sum, steps, forced = 0.0, 0, False
            for ch in chunks:
                h = run_chunk(model, encode_text_chunk(ch, vocabs), beam_size, restriction,
                              alpha, use_greedy)
                w = vocabs["trg"].decode(h.tokens)
                al = [vocabs["trg_f"][k].decode(h.factors[k][1:]) for k in range(nf)]
                if inp.get("strip_prefix") and ch["target_prefix"]:
                    drop = min(len(ch["target_prefix"]), len(w))
                    w = w[drop:]
                    al = [a[drop:] for a in al]
                words.extend(w)
                for k in range(nf):
                    facs[k].extend(al[k])
                lp_sum += h.logprob
                steps += h.steps
                forced = forced or h.forced_eos
            recs.append(dict(text=" ".join(words), score=lp_sum / (steps ** alpha),
                             factors=[" ".join(f) for f in facs], chunks=len(chunks),
                             forced_eos=forced, error=None))
        except OracleError as e:
            if e.kind != "InputError":
                raise
            recs.append(dict(text="", score=0.0, factors=[], chunks=0, forced_eos=False,
                             error=str(e)))
    return recs


# ------------------------------------------------------------------ int8
# quant.py:33-132 — dynamic int8 feed-forward.  The integer product is exact,
# the rescale is (float32(acc) * a_scale) * w_scale, each product rounded in
# float32, then + bias.

def round_half_away(x):
    """quant.py:33-37: ties away from zero, in the input's float32."""
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def quantize_rows(w):
    """quant.py:40-53 (weights) / 99-104 (activations, same rule)."""
    w = np.asarray(w, dtype=F32)
    maxabs = np.abs(w).max(axis=1)
    scales = np.where(maxabs > 0, maxabs / 127.0, 1.0).astype(F32)
    q = np.clip(round_half_away(w / scales[:, None]), -127, 127).astype(np.int8)
    return q, scales


def gemm_i8(qx, qw):
    """quant.py:60-78: (m, k) int8 . (n, k)^T int8 -> (m, n) int32, exact."""
    return qx.astype(np.int32) @ qw.astype(np.int32).T


def quantized_linear(x, q, scales, bias=None):
    """quant.py:121-132: QuantizedLinear.__call__ on float32 rows."""
    flat = np.ascontiguousarray(np.asarray(x, dtype=F32).reshape(-1, x.shape[-1]))
    qx, a_scales = quantize_rows(flat)
    out = gemm_i8(qx, q).astype(F32) * a_scales[:, None] * np.asarray(scales, F32)[None, :]
    if bias is not None:
        out = out + np.asarray(bias, F32)
    return out.reshape(x.shape[:-1] + (q.shape[0],))
