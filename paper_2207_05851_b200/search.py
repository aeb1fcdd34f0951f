"""Drop-in translation API (mirrors skiff search.py:43-468).

Same dataclasses, same input protocol (plain or JSON lines), same chunking,
prefix forcing, restriction, error isolation and scoring as the reference.
What changes is where the search runs: `translate` id-encodes every chunk of
every input on the host, then decodes ALL chunks together in length-sorted
device batches (engine.decode_jobs) — encoder, decoder steps and the beam
bookkeeping are CUDA kernels, captured as one CUDA graph per step.  The
reference's sequential per-sentence loop (search.py:459-467) becomes one
batched device run; outputs do not depend on batch composition
(test_search.py:400-405).

`greedy_search` / `beam_search` accept either a device `Model` or any object
implementing the reference's model protocol (decode_init / decode_step /
select_rows, e.g. test_search.py's StubModel).  For the latter the model's
logits are uploaded each step and the SAME device beam kernel picks the
candidates (ProtocolSearch).
"""

from __future__ import annotations

import json
import logging
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kern
from . import _native as N
from .checkpoint import Vocabulary
from .engine import ChunkJob, ChunkResult, LazyJobs, decode_jobs
from .errors import ConfigError, InputError
from .shortlist import sorted_union
from .model import (BOS_ID, EOS_ID, PAD_ID, SHIFT_ID, UNK_ID, Model, validate_active_ids)

logger = logging.getLogger(__name__)

INPUT_KEYS = ("text", "source_prefix", "target_prefix", "target_prefix_factors",
              "source_factors")


@dataclass
class SentenceInput:
    """One sentence to translate, with optional factors and prefixes (search.py:43-59)."""
    tokens: list[str]
    source_factors: list[list[str]] = field(default_factory=list)
    source_prefix: list[str] = field(default_factory=list)
    target_prefix: list[str] = field(default_factory=list)
    target_prefix_factors: list[list[str]] = field(default_factory=list)
    prefix_all_chunks: bool = False
    strip_prefix: bool = False

    def validate(self) -> None:
        for i, stream in enumerate(self.source_factors):
            if len(stream) != len(self.tokens):
                raise InputError(f"source factor stream {i} has {len(stream)} tokens, "
                                 f"text has {len(self.tokens)}")


@dataclass
class Hypothesis:
    """Finished hypothesis (search.py:62-75): tokens exclude EOS; factors hold
    one entry per step including the EOS step."""
    tokens: list[int]
    factors: list[list[int]]
    logprob: float
    steps: int
    forced_eos: bool
    finished: bool = True

    def normalized(self, length_alpha: float) -> float:
        return self.logprob / (self.steps ** length_alpha)


@dataclass
class TranslationRecord:
    text: str
    score: float
    factors: list[str]
    chunks: int
    forced_eos: bool
    error: str | None = None


class ShortlistRestriction:
    """Union of the shortlist rows of the chunk's source ids (search.py:88-97)."""

    def __init__(self, shortlist):
        self.shortlist = shortlist

    def resolve(self, model, state, src_ids, lengths, extra_ids) -> np.ndarray:
        return sorted_union(self.shortlist.lookup(src_ids), extra_ids)


class NvsRestriction:
    """Encoder-side vocabulary selection at a threshold (search.py:100-110)."""

    def __init__(self, threshold: float):
        self.threshold = threshold

    def resolve(self, model, state, src_ids, lengths, extra_ids) -> np.ndarray:
        (ids,) = model.nvs_select(state.enc, lengths, self.threshold, always_include=extra_ids)
        return ids


@dataclass
class SearchSettings:
    beam: int = 1
    length_alpha: float = 1.0
    restriction: ShortlistRestriction | NvsRestriction | None = None
    use_greedy: bool | None = None


# ------------------------------------------------------------------- input
def parse_input_line(line: str) -> SentenceInput:
    """search.py:124-161."""
    stripped = line.strip()
    if not stripped.startswith("{"):
        return SentenceInput(tokens=line.split())
    try:
        obj = json.loads(stripped)
    except json.JSONDecodeError as e:
        raise InputError(f"invalid JSON input: {e}") from None
    if not isinstance(obj, dict):
        raise InputError("JSON input must be an object")
    unknown = set(obj) - set(INPUT_KEYS)
    if unknown:
        raise InputError(f"unknown input keys: {sorted(unknown)}")
    if "text" not in obj:
        raise InputError("JSON input is missing \"text\"")

    def tokens(key):
        v = obj.get(key, "")
        if not isinstance(v, str):
            raise InputError(f"\"{key}\" must be a string")
        return v.split()

    def streams(key):
        v = obj.get(key, [])
        if not isinstance(v, list) or not all(isinstance(x, str) for x in v):
            raise InputError(f"\"{key}\" must be a sequence of strings")
        return [x.split() for x in v]

    inp = SentenceInput(tokens=tokens("text"), source_factors=streams("source_factors"),
                        source_prefix=tokens("source_prefix"),
                        target_prefix=tokens("target_prefix"),
                        target_prefix_factors=streams("target_prefix_factors"))
    inp.validate()
    return inp


def chunk_input(inp: SentenceInput, max_seq_len: int) -> list[SentenceInput]:
    """search.py:164-191."""
    if not inp.tokens:
        raise InputError("empty input")
    plen = len(inp.source_prefix)
    if max_seq_len <= plen:
        raise InputError(f"source prefix ({plen} tokens) leaves no room in a window of "
                         f"{max_seq_len}")
    budget = max_seq_len - plen
    if len(inp.tokens) <= budget:
        return [inp]  # one window: the chunk is the input itself (never mutated)
    out = []
    for start in range(0, len(inp.tokens), budget):
        with_target = start == 0 or inp.prefix_all_chunks
        out.append(SentenceInput(
            tokens=inp.tokens[start:start + budget],
            source_factors=[s[start:start + budget] for s in inp.source_factors],
            source_prefix=list(inp.source_prefix),
            target_prefix=list(inp.target_prefix) if with_target else [],
            target_prefix_factors=[list(s) for s in inp.target_prefix_factors]
            if with_target else [],
            prefix_all_chunks=inp.prefix_all_chunks, strip_prefix=inp.strip_prefix))
    return out


def encode_chunk(chunk: SentenceInput, vocabs):
    """search.py:194-207: (src_ids (1, L), factor ids list of (1, L), lengths (1,))."""
    ids = vocabs.src_vocab.encode(chunk.source_prefix + chunk.tokens)
    plen = len(chunk.source_prefix)
    fids = [np.array([[PAD_ID] * plen + v.encode(s)], dtype=np.int64)
            for s, v in zip(chunk.source_factors, vocabs.src_factor_vocabs)]
    return np.array([ids], dtype=np.int64), fids, np.array([len(ids)], dtype=np.int64)


def _encode_with_warning(tokens, vocab: Vocabulary, what: str) -> list[int]:
    out = []
    for tok in tokens:
        if tok not in vocab:
            logger.warning("%s token %r is not in the vocabulary; using UNK", what, tok)
        out.append(vocab.to_id(tok))
    return out


def encode_target_prefix(chunk: SentenceInput, vocabs):
    """search.py:219-226."""
    pre = _encode_with_warning(chunk.target_prefix, vocabs.trg_vocab, "target prefix")
    fac = [_encode_with_warning(s, v, f"target prefix factor {i}")
           for i, (s, v) in enumerate(zip(chunk.target_prefix_factors, vocabs.trg_factor_vocabs))]
    return pre, fac


def _max_output_len(src_len: int) -> int:
    return 2 * src_len + 10


def _check_prefix_budget(prefix_ids, max_len) -> None:
    if len(prefix_ids) > max_len - 1:
        raise InputError(f"target prefix ({len(prefix_ids)} tokens) does not fit the "
                         f"output budget of {max_len}")


def _chunk_job(model, chunk: SentenceInput, vocabs, restriction) -> tuple[ChunkJob, float | None]:
    """Host half of _start_state (search.py:235-242): ids, prefix, active ids
    (encode_chunk's ids as plain lists: no numpy round trip per sentence)."""
    ids = vocabs.src_vocab.encode(chunk.source_prefix + chunk.tokens)
    plen = len(chunk.source_prefix)
    fids = [[PAD_ID] * plen + v.encode(s) for s, v in zip(chunk.source_factors, vocabs.src_factor_vocabs)]
    pre, pre_f = encode_target_prefix(chunk, vocabs)
    _check_prefix_budget(pre, _max_output_len(len(ids)))
    job = ChunkJob(ids, fids, pre, pre_f)
    nvs = None
    if isinstance(restriction, NvsRestriction):
        nvs = restriction.threshold
    elif restriction is not None:
        extra = np.array([PAD_ID, UNK_ID, EOS_ID] + list(pre), dtype=np.int64)
        ids_a = np.asarray(ids, dtype=np.int64)
        a = restriction.resolve(model, None, ids_a, np.array([ids_a.size], dtype=np.int64), extra)
        job.active_ids = validate_active_ids(model.config, a)
    return job, nvs


def _hyp(r: ChunkResult) -> Hypothesis:
    return Hypothesis(r.tokens, r.factors, r.logprob, r.steps, r.forced_eos)


def _decide(settings: SearchSettings) -> int:
    """search.py:399-409: beam width K of the device run (1 = greedy)."""
    greedy = settings.use_greedy if settings.use_greedy is not None else settings.beam == 1
    if greedy:
        if settings.beam != 1:
            raise ConfigError("greedy decoding is incompatible with beam > 1")
        return 1
    if settings.beam < 1:
        raise ConfigError(f"beam size must be at least 1, got {settings.beam}")
    return settings.beam


# ------------------------------------------------------------------ search
def greedy_search(model, vocabs, chunk: SentenceInput, restriction=None,
                  length_alpha: float = 1.0) -> Hypothesis:
    """search.py:275-313 (device beam kernel with K = 1, bit-identical)."""
    return _search_one(model, vocabs, chunk, 1, restriction, length_alpha)


def beam_search(model, vocabs, chunk: SentenceInput, beam: int, restriction=None,
                length_alpha: float = 1.0) -> Hypothesis:
    """search.py:325-394."""
    if beam < 1:
        raise ConfigError(f"beam size must be at least 1, got {beam}")
    return _search_one(model, vocabs, chunk, beam, restriction, length_alpha)


def _search_one(model, vocabs, chunk, beam, restriction, alpha) -> Hypothesis:
    if not isinstance(model, Model):
        return ProtocolSearch(model, vocabs, chunk, beam, restriction, alpha).run()
    job, nvs = _chunk_job(model, chunk, vocabs, restriction)
    (r,) = decode_jobs(model, [job], beam, alpha, nvs)
    return _hyp(r)


def translate(model, vocabs, inputs, settings: SearchSettings | None = None,
              max_rows: int = 2560) -> list[TranslationRecord]:
    """search.py:454-468: every input independently; a malformed record
    yields an error record.  All chunks of all inputs decode together."""
    settings = settings or SearchSettings()
    cfg = model.config
    nf = len(cfg.target_factor_specs)
    plans: list = []
    all_chunks: list[SentenceInput] = []
    lens: list[int] = []
    nvs_thr = settings.restriction.threshold if isinstance(settings.restriction, NvsRestriction) else None
    for inp in inputs:
        try:
            inp.validate()
            if len(inp.source_factors) != len(cfg.source_factor_specs):
                raise InputError(f"model expects {len(cfg.source_factor_specs)} source factor "
                                 f"streams, input has {len(inp.source_factors)}")
            if len(inp.target_prefix_factors) > nf:
                raise InputError(f"model has {nf} target factor streams, prefix factors name "
                                 f"{len(inp.target_prefix_factors)}")
            chunks = chunk_input(inp, cfg.max_seq_len)
            n_src = [len(ch.source_prefix) + len(ch.tokens) for ch in chunks]
            for ch, n in zip(chunks, n_src):  # _chunk_job's only input check, from lengths
                _check_prefix_budget(ch.target_prefix, _max_output_len(n))
            plans.append((inp, chunks, len(all_chunks)))
            all_chunks.extend(chunks)
            lens.extend(n_src)
        except InputError as e:
            logger.warning("input skipped: %s", e)
            plans.append(str(e))
    # the chunks' ids are encoded when their device batch is launched
    jobs = LazyJobs(lens, lambda i: _chunk_job(model, all_chunks[i], vocabs, settings.restriction)[0])
    texts: dict = {}  # chunk index -> (surface tokens, factor tokens), built while the GPU decodes

    def detok(i, r):
        texts[i] = (vocabs.trg_vocab.decode(r.tokens),
                    [vocabs.trg_factor_vocabs[q].decode(r.factors[q][1:]) for q in range(nf)])

    if jobs:
        K = _decide(settings)
        if isinstance(model, Model):
            results = [_hyp(r) for r in decode_jobs(model, jobs, K, settings.length_alpha,
                                                    nvs_thr, max_rows, on_done=detok)]
        else:
            results = [ProtocolSearch.from_job(model, jobs[i], K, settings.restriction,
                                               settings.length_alpha).run() for i in range(len(jobs))]
    records = []
    for plan in plans:
        if isinstance(plan, str):
            records.append(TranslationRecord("", 0.0, [], 0, False, plan))
            continue
        inp, chunks, first = plan
        words: list[str] = []
        facs: list[list[str]] = [[] for _ in range(nf)]
        lp, steps, forced = 0.0, 0, False
        for k, ch in enumerate(chunks):
            h = results[first + k]
            if first + k in texts:
                toks, aligned = texts[first + k]
            else:
                toks = vocabs.trg_vocab.decode(h.tokens)
                aligned = [vocabs.trg_factor_vocabs[q].decode(h.factors[q][1:]) for q in range(nf)]
            if inp.strip_prefix and ch.target_prefix:
                drop = min(len(ch.target_prefix), len(toks))
                toks = toks[drop:]
                aligned = [a[drop:] for a in aligned]
            words.extend(toks)
            for q in range(nf):
                facs[q].extend(aligned[q])
            lp += h.logprob
            steps += h.steps
            forced = forced or h.forced_eos
        records.append(TranslationRecord(" ".join(words), lp / (steps ** settings.length_alpha),
                                         [" ".join(f) for f in facs], len(chunks), forced))
    return records


# ================================================ protocol-model search
class ProtocolSearch:
    """Search over any reference-protocol model: the model produces logits
    on its own (host or device); candidate selection, EOS routing and
    history run in the device beam kernel (skb_beam_step)."""

    def __init__(self, model, vocabs, chunk, beam, restriction, alpha, job=None,
                 logits_are_logprobs=False):
        self.model, self.beam, self.alpha, self.restriction = model, beam, alpha, restriction
        self.lp_in = logits_are_logprobs
        if job is None:
            src_ids, src_f, lengths = encode_chunk(chunk, vocabs)
            pre, pre_f = encode_target_prefix(chunk, vocabs)
            job = ChunkJob([int(x) for x in src_ids[0]], [[int(x) for x in f[0]] for f in src_f],
                           pre, pre_f)
        self.job = job

    @classmethod
    def from_job(cls, model, job, beam, restriction, alpha):
        return cls(model, None, None, beam, restriction, alpha, job)

    def run(self) -> Hypothesis:
        m, job, K = self.model, self.job, self.beam
        if K < 1:
            raise ConfigError(f"beam size must be at least 1, got {K}")
        cfg = m.config
        nf = len(cfg.target_factor_specs)
        src = np.array([job.src_ids], dtype=np.int64)
        sf = [np.array([f], dtype=np.int64) for f in job.src_factor_ids]
        lengths = np.array([len(job.src_ids)], dtype=np.int64)
        max_len = _max_output_len(len(job.src_ids))
        _check_prefix_budget(job.prefix_ids, max_len)
        state = m.decode_init(src, sf, lengths)
        if self.restriction is not None:
            extra = np.array([PAD_ID, UNK_ID, EOS_ID] + list(job.prefix_ids), dtype=np.int64)
            state.active_ids = validate_active_ids(
                cfg, self.restriction.resolve(m, state, src[0], lengths, extra))
        active = getattr(state, "active_ids", None)
        dev = torch.device("cuda")
        V = cfg.trg_vocab_size if active is None else active.size

        def col_of(tok):
            if active is None:
                return tok
            c = int(np.searchsorted(active, tok))
            if c >= active.size or active[c] != tok:
                raise ConfigError(f"token id {tok} missing from the restricted vocabulary")
            return c

        # the prefix tables hold the surface prefix and every factor stream
        P = max([1, len(job.prefix_ids)] + [len(f) for f in job.prefix_factor_ids[:nf]])
        z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt, device=dev)  # noqa: E731
        bufs = dict(
            len_pen=torch.tensor([float(s) ** self.alpha if s else 1.0 for s in range(max_len + 1)],
                                 dtype=torch.float64, device=dev),
            step=z(1), col_token=None if active is None else
            torch.from_numpy(active.astype(np.int32)).to(dev),
            max_len=torch.tensor([max_len], dtype=torch.int32, device=dev),
            prefix_len=torch.tensor([len(job.prefix_ids)], dtype=torch.int32, device=dev),
            prefix_col=torch.tensor([col_of(t) for t in job.prefix_ids] or [-1],
                                    dtype=torch.int32, device=dev),
            prefix_fac=torch.full((max(nf, 1), P), -1, dtype=torch.int32, device=dev),
            n_alive=torch.ones(1, dtype=torch.int32, device=dev), done=z(1),
            score=z(K, torch.float64), tok=z(K), ftok=z(max(nf, 1) * K), parent=z(K),
            tok_hist=z(max_len * K), par_hist=z(max_len * K), fac_hist=z(max_len * max(nf, 1) * K),
            cand_score=z(K * K, torch.float64), cand_lp=z(K * K, torch.float32), cand_col=z(K * K),
            cand_cnt=z(K), row_argmax=z(K), fac_choice=z(K * max(nf, 1)), counter=z(1),
            best_norm=z(1, torch.float64), best_logprob=z(1, torch.float64), best_steps=z(1),
            best_forced=z(1), best_parent=z(1), best_fac=z(max(nf, 1)), n_done=z(1))
        for k, stream in enumerate(job.prefix_factor_ids[:nf]):
            if stream:
                bufs["prefix_fac"][k, :len(stream)] = torch.tensor(stream, dtype=torch.int32)
        fac_w = [s.vocab_size for s in cfg.target_factor_specs]
        off_h = [int(x) for x in np.cumsum([0] + fac_w)]
        fac_off = torch.tensor(off_h, dtype=torch.int32, device=dev)
        logits = torch.zeros(K, V, device=dev)
        facl = torch.zeros(K, max(1, sum(fac_w)), device=dev)
        b = bufs
        st = N.BeamState(1, K, V, max_len, nf, b["len_pen"].data_ptr(), b["step"].data_ptr(),
                         N.ptr(b["col_token"]), None, col_of(EOS_ID), b["max_len"].data_ptr(),
                         b["prefix_len"].data_ptr(), b["prefix_col"].data_ptr(), P,
                         b["prefix_fac"].data_ptr() if nf else None, b["n_alive"].data_ptr(),
                         b["done"].data_ptr(), b["score"].data_ptr(), b["tok"].data_ptr(),
                         b["ftok"].data_ptr(), b["parent"].data_ptr(), b["tok_hist"].data_ptr(),
                         b["par_hist"].data_ptr(), b["fac_hist"].data_ptr(),
                         facl.data_ptr() if nf else None, facl.stride(0), fac_off.data_ptr(),
                         None, 0, 0, 0, b["cand_score"].data_ptr(), b["cand_lp"].data_ptr(),
                         b["cand_col"].data_ptr(), b["cand_cnt"].data_ptr(),
                         b["row_argmax"].data_ptr(), b["fac_choice"].data_ptr(),
                         b["counter"].data_ptr(), b["best_norm"].data_ptr(),
                         b["best_logprob"].data_ptr(), b["best_steps"].data_ptr(),
                         b["best_forced"].data_ptr(), b["best_parent"].data_ptr(),
                         b["best_fac"].data_ptr(), b["n_done"].data_ptr())
        prev = np.array([BOS_ID])
        prev_f = [np.array([SHIFT_ID]) for _ in range(nf)]
        for t in range(max_len):
            out = m.decode_step(state, prev, prev_f)
            surf = np.asarray(out.surface.data, dtype=np.float32)
            n_rows = surf.shape[0]
            logits[:n_rows].copy_(torch.from_numpy(surf))
            for k in range(nf):
                facl[:n_rows, off_h[k]:off_h[k + 1]].copy_(
                    torch.from_numpy(np.asarray(out.factors[k].data, dtype=np.float32)))
            kern.beam_step(logits, st, self.lp_in)
            n_alive = int(b["n_alive"].item())
            if int(b["done"].item()):
                break
            parents = b["parent"][:n_alive].cpu().numpy()
            state.select_rows([int(p) for p in parents])
            prev = b["tok"][:n_alive].cpu().numpy().astype(np.int64)
            fk = b["ftok"].view(max(nf, 1), K)[:, :n_alive].cpu().numpy()
            prev_f = [fk[k].astype(np.int64) for k in range(nf)]
            b["step"].add_(1)
        toks = torch.zeros(1, max_len, dtype=torch.int32, device=dev)
        facs = torch.zeros(1, max(nf, 1), max_len, dtype=torch.int32, device=dev)
        kern.beam_finalize(st, toks, facs)
        s = int(b["best_steps"].item())
        return Hypothesis([int(x) for x in toks[0, :s - 1].cpu()],
                          [[int(x) for x in facs[0, k, :s].cpu()] for k in range(nf)],
                          float(b["best_logprob"].item()), s, bool(b["best_forced"].item()))
