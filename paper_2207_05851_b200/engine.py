"""Batched device decoder: the hot path behind translate() (search.py:275-468).

One "row" is one hypothesis slot.  A batch of B chunks decoded with beam K
owns R = B*K row slots (slot b*K+i = beam position i of chunk b).  Every step
runs, for all R rows, the decoder forward (model.py:536-585) and then the
beam bookkeeping kernel (search.py:345-393) entirely on the GPU:

  embed -> [LN -> QKV GEMM -> self-attn (KV cache, ancestor table) -> Wo GEMM
  (+residual) | LN -> SSRU GEMM with fused cell epilogue] -> LN -> cross-Q
  GEMM -> cross-attn -> Wo GEMM -> LN -> FFN1 (+bias, ReLU) -> FFN2 (+bias,
  +residual) ... -> final LN -> output-projection GEMM over the (restricted)
  vocabulary -> beam step (masked log-softmax, float64 scores, exact top-K,
  EOS routing) -> reorder (ancestor table) -> step += 1

The step is captured once into a CUDA graph and replayed; the host only
polls a "sentences done" counter every few steps.  KV-cache bytes never
move: beam reorders rewrite the [2, R, S] int32 ancestor table instead.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kern
from . import _native as N
from .config import SSRU
from .errors import ConfigError, ShapeError
from .model import BOS_ID, EOS_ID, PAD_ID, SHIFT_ID, UNK_ID, Model, validate_active_ids

I32 = torch.int32


class StepBuffers:
    """Every device buffer a decode step touches (stable for graph capture)."""

    def __init__(self, model: Model, R: int, B: int, L: int, S_max: int, U: int,
                 E_out: torch.Tensor, ckv: torch.Tensor, lengths: torch.Tensor,
                 row_sent: torch.Tensor, cache_rows: int | None = None):
        c = model.config
        d, D, dev, cdt = c.d_model, c.decoder_layers, model.device, model.cdt
        nf = len(c.target_factor_specs)
        self.R, self.B, self.L, self.S_max, self.U = R, B, L, S_max, U
        self.step = torch.zeros(1, dtype=I32, device=dev)
        self.tok = torch.full((R,), BOS_ID, dtype=I32, device=dev)
        self.ftok = torch.full((max(nf, 1), R), SHIFT_ID, dtype=I32, device=dev)
        self.parent = torch.arange(R, dtype=I32, device=dev)
        self.row_sent = row_sent
        self.lengths = lengths
        self.ckv = ckv
        self.E_out = E_out
        self.x = torch.zeros(R, d, device=dev)
        self.h = torch.zeros(R, d, device=dev, dtype=cdt)
        self.ctx = torch.zeros(R, d, device=dev, dtype=cdt)
        self.q = torch.zeros(R, d, device=dev, dtype=cdt)
        self.f = torch.zeros(R, c.ff_dim, device=dev, dtype=cdt)
        self.logits = torch.zeros(R, U, device=dev)
        # fused log-softmax partials: (max, sum exp) per 32-column group
        G = (U + 31) // 32
        self.lse_part = torch.zeros(R, 2 * (G + (G & 1)), device=dev)  # rows 16-byte aligned
        self.mask = None          # [B, words] active-column bits (restricted vocab)
        self.group = 1            # rows per sentence group (beam size)
        self.fac = torch.zeros(R, int(model.fac_off[-1].item()) if nf else 1, device=dev)
        if c.decoder_kind == SSRU:
            self.cell = torch.zeros(D, 2, R, d, device=dev)
            self.qkv = self.kc = self.vc = None
        else:
            self.cell = None
            self.qkv = torch.zeros(R, 3 * d, device=dev, dtype=cdt)
            cap = R if cache_rows is None else cache_rows
            self.kc = torch.zeros(D, cap, S_max, d, device=dev, dtype=cdt)
            self.vc = torch.zeros(D, cap, S_max, d, device=dev, dtype=cdt)
        self.anc = torch.zeros(2, R, S_max, dtype=I32, device=dev)


def step_forward(model: Model, sb: StepBuffers) -> None:
    """Enqueue one decoder step for all rows (model.py:536-585)."""
    c = model.config
    d, H, dh = c.d_model, c.heads, c.head_dim
    R = sb.R
    nf = len(c.target_factor_specs)
    kern.embed_target(sb.tok, model.E_trg, model.pe_trg, sb.step, sb.ftok if nf else None,
                      model.trg_ftab_ptrs if nf else None, sb.x)
    for li, Ly in enumerate(model.dec):
        kern.layernorm(sb.x, *Ly.ln_self, sb.h)
        if c.decoder_kind == SSRU:
            kern.gemm(sb.h, Ly.w_ssru, sb.x, N.EPI_SSRU, Ly.b_ssru, c_state=sb.cell[li],
                      src_row=sb.parent, step=sb.step, state_stride=R * d)
        else:
            kern.gemm(sb.h, Ly.wqkv, sb.qkv)
            kern.self_attention_step(sb.qkv, sb.kc[li], sb.vc[li], sb.anc, sb.step, sb.ctx,
                                     R, H, dh, sb.S_max, sb.group)
            kern.gemm(sb.ctx, Ly.wo, sb.x, N.EPI_RESID)
        kern.layernorm(sb.x, *Ly.ln_cross, sb.h)
        kern.gemm(sb.h, Ly.wq_c, sb.q)
        kern.cross_attention_step(sb.q, sb.ckv, li * 2 * d, li * 2 * d + d, sb.L, sb.row_sent,
                                  sb.lengths, sb.ctx, R, H, dh, sb.group)
        kern.gemm(sb.ctx, Ly.wo_c, sb.x, N.EPI_RESID)
        kern.layernorm(sb.x, *Ly.ln_ffn, sb.h)
        kern.gemm(sb.h, Ly.w1, sb.f, N.EPI_RELU, Ly.b1)
        kern.gemm(sb.f, Ly.w2, sb.x, N.EPI_RESID, Ly.b2)
    kern.layernorm(sb.x, *model.ln_final, sb.h)
    kern.gemm(sb.h, sb.E_out, sb.logits, N.EPI_LOGITS, lse_part=sb.lse_part, mask=sb.mask,
              rows_per_group=sb.group)
    if nf:
        kern.gemm(sb.h, model.w_fac, sb.fac, N.EPI_STORE, model.b_fac)


# ====================================================================== jobs
@dataclass
class ChunkJob:
    """One id-encoded chunk (search.py:194-226)."""
    src_ids: list
    src_factor_ids: list = field(default_factory=list)
    prefix_ids: list = field(default_factory=list)
    prefix_factor_ids: list = field(default_factory=list)
    active_ids: np.ndarray | None = None


@dataclass
class ChunkResult:
    tokens: list
    factors: list
    logprob: float
    steps: int
    forced_eos: bool


def _encode_batch(model: Model, jobs: list[ChunkJob]):
    c = model.config
    B = len(jobs)
    L = max(len(j.src_ids) for j in jobs)
    ids = np.zeros((B, L), dtype=np.int32)
    nsf = len(c.source_factor_specs)
    fids = np.zeros((max(nsf, 1), B, L), dtype=np.int32)
    lengths = np.zeros(B, dtype=np.int32)
    for b, j in enumerate(jobs):
        n = len(j.src_ids)
        ids[b, :n] = j.src_ids
        lengths[b] = n
        for k in range(nsf):
            fids[k, b, :n] = j.src_factor_ids[k]
    dev = model.device
    ids_d = torch.from_numpy(ids.reshape(-1)).to(dev)
    fids_d = torch.from_numpy(fids.reshape(max(nsf, 1), -1)).to(dev)
    len_d = torch.from_numpy(lengths).to(dev)
    if (ids < 0).any() or (ids >= c.src_vocab_size).any():
        raise ShapeError(f"ids out of range [0, {c.src_vocab_size}) for embedding table")
    enc = model.encode_device(ids_d, fids_d if nsf else None, len_d, B, L)
    return enc, len_d, B, L


def nvs_active_sets(model: Model, enc, len_d, B, L, threshold, jobs) -> list[np.ndarray]:
    """NvsRestriction.resolve (search.py:100-110) for a batch of chunks."""
    if not model.config.nvs_enabled:
        raise ConfigError("model was built without vocabulary selection")
    if not (0.0 <= threshold <= 1.0):
        raise ConfigError(f"nvs threshold {threshold} outside [0, 1]")
    from .model import mask_to_ids
    mask = model.nvs_mask_device(enc, len_d, B, L, threshold).cpu().numpy()
    out = []
    for b, j in enumerate(jobs):
        extra = np.array([PAD_ID, UNK_ID, EOS_ID] + list(j.prefix_ids), dtype=np.int64)
        ids = np.union1d(mask_to_ids(mask[b], model.config.trg_vocab_size),
                         np.unique(extra))
        out.append(validate_active_ids(model.config, ids))
    return out


class BeamBatch:
    """Device state of one batched beam (or greedy, K=1) run.

    Construction does the host work and stages every input on the device
    (ids, lengths, prefixes, restriction masks, buffers); `run()` is pure
    device work: encoder, cross K/V, the captured decode loop, finalize."""

    GRAPH_POLL = 8

    def __init__(self, model: Model, jobs: list[ChunkJob], beam: int, alpha: float,
                 nvs_threshold: float | None = None, use_graph: bool = True):
        if beam < 1:
            raise ConfigError(f"beam size must be at least 1, got {beam}")
        if beam > 32:
            raise ConfigError(f"beam size {beam} exceeds the device limit of 32")
        self.model, self.jobs, self.K, self.alpha = model, jobs, beam, alpha
        self.use_graph = use_graph
        self.nvs_threshold = nvs_threshold
        c = model.config
        dev = model.device
        nf = len(c.target_factor_specs)
        self.nf = nf
        B = len(jobs)
        L = max(len(j.src_ids) for j in jobs)
        self.B, self.L = B, L
        # ---- source ids (padded), staged on the device
        ids = np.zeros((B, L), dtype=np.int32)
        nsf = len(c.source_factor_specs)
        fids = np.zeros((max(nsf, 1), B, L), dtype=np.int32)
        lengths = np.zeros(B, dtype=np.int32)
        for b, j in enumerate(jobs):
            n = len(j.src_ids)
            ids[b, :n] = j.src_ids
            lengths[b] = n
            for k in range(nsf):
                fids[k, b, :n] = j.src_factor_ids[k]
        if (ids < 0).any() or (ids >= c.src_vocab_size).any():
            raise ShapeError(f"ids out of range [0, {c.src_vocab_size}) for embedding table")
        self.h2d_bytes = ids.nbytes + lengths.nbytes + (fids.nbytes if nsf else 0)
        self.ids_d = torch.from_numpy(ids.reshape(-1)).to(dev)
        self.fids_d = torch.from_numpy(fids.reshape(max(nsf, 1), -1)).to(dev) if nsf else None
        self.len_d = torch.from_numpy(lengths).to(dev)
        # ---- per-chunk limits
        max_len = np.array([2 * len(j.src_ids) + 10 for j in jobs], dtype=np.int32)
        self.S_max = int(max_len.max())
        self.max_len = torch.from_numpy(max_len).to(dev)
        self.prefix_len = torch.tensor([len(j.prefix_ids) for j in jobs], dtype=I32, device=dev)
        self.R = B * beam
        self.row_sent = torch.arange(self.R, dtype=I32, device=dev) // beam
        self.len_pen = torch.tensor([float(s) ** alpha if s > 0 else 1.0
                                     for s in range(self.S_max + 1)],
                                    dtype=torch.float64, device=dev)
        self.sb = None
        if nvs_threshold is None:
            self._setup_vocab([j.active_ids for j in jobs])
        self.graph = None
        self.steps_run = 0
        self.launches_per_step = 0

    def _setup_vocab(self, actives):
        """Restricted output vocabulary (search.py:235-242) as the union U of
        the chunks' active sets plus a per-chunk column bitmask; then every
        buffer of the decode loop."""
        model, c, dev = self.model, self.model.config, self.model.device
        B, K, nf, jobs = self.B, self.K, self.nf, self.jobs
        restricted = any(a is not None for a in actives)
        V = c.trg_vocab_size
        if restricted:
            actives = [a if a is not None else np.arange(V, dtype=np.int64) for a in actives]
            U_ids = np.unique(np.concatenate(actives)).astype(np.int64)
            U = int(U_ids.size)
            mask = np.zeros((B, (U + 31) // 32), dtype=np.uint32)
            for b, a in enumerate(actives):
                cols = np.searchsorted(U_ids, a)
                np.bitwise_or.at(mask[b], cols >> 5,
                                 (np.uint32(1) << (cols & 31).astype(np.uint32)))
            self.col_token = torch.from_numpy(U_ids.astype(np.int32)).to(dev)
            self.mask = torch.from_numpy(mask.view(np.int32)).to(dev)
            E_out = torch.empty(U, c.d_model, device=dev, dtype=model.cdt)
            self._gather_E = True
            col_of = {int(t): i for i, t in enumerate(U_ids)}
        else:
            U = V
            self.col_token = self.mask = None
            E_out = model.E_trg_c
            self._gather_E = False
            col_of = None
        self.U = U
        eos_col = col_of[EOS_ID] if restricted else EOS_ID
        P = max(1, max(len(j.prefix_ids) for j in jobs))
        prefix_col = np.full((B, P), -1, dtype=np.int32)
        prefix_fac = np.full((B, max(nf, 1), P), -1, dtype=np.int32)
        for b, j in enumerate(jobs):
            for t, tok in enumerate(j.prefix_ids):
                if restricted:
                    if tok not in col_of:
                        raise ConfigError(f"token id {tok} missing from the restricted vocabulary")
                    prefix_col[b, t] = col_of[tok]
                else:
                    prefix_col[b, t] = tok
            for k, stream in enumerate(j.prefix_factor_ids[:nf]):
                prefix_fac[b, k, :len(stream)] = stream
        R, S_max = self.R, self.S_max
        D2 = 2 * c.d_model * c.decoder_layers
        ckv = torch.empty(B * self.L, max(D2, 1), device=dev, dtype=model.cdt)
        self.sb = StepBuffers(model, R, B, self.L, S_max, U, E_out, ckv, self.len_d,
                              self.row_sent)
        sb = self.sb
        sb.group = K
        sb.mask = self.mask

        def z(n, dt=I32):
            return torch.zeros(n, dtype=dt, device=dev)

        self.prefix_col = torch.from_numpy(prefix_col).to(dev)
        self.prefix_fac = torch.from_numpy(prefix_fac).to(dev)
        self.n_alive = torch.ones(B, dtype=I32, device=dev)
        self.done = z(B)
        self.score = z(R, torch.float64)
        self.tok_hist = z(S_max * R)
        self.par_hist = z(S_max * R)
        self.fac_hist = z(S_max * max(nf, 1) * R)
        self.cand_score = z(R * K, torch.float64)
        self.cand_lp = z(R * K, torch.float32)
        self.cand_col = z(R * K)
        self.cand_cnt = z(R)
        self.row_argmax = z(R)
        self.fac_choice = z(R * max(nf, 1))
        self.counter = z(B)
        self.best_norm = z(B, torch.float64)
        self.best_logprob = z(B, torch.float64)
        self.best_steps = z(B)
        self.best_forced = z(B)
        self.best_parent = z(B)
        self.best_fac = z(B * max(nf, 1))
        self.n_done = z(1)
        self.tokens_out = z(B * S_max).view(B, S_max)
        self.factors_out = z(B * max(nf, 1) * S_max).view(B, max(nf, 1), S_max)
        self.state = N.BeamState(
            B, K, U, S_max, nf, self.len_pen.data_ptr(), sb.step.data_ptr(),
            N.ptr(self.col_token), N.ptr(self.mask), eos_col, self.max_len.data_ptr(),
            self.prefix_len.data_ptr(), self.prefix_col.data_ptr(), P,
            self.prefix_fac.data_ptr() if nf else None, self.n_alive.data_ptr(),
            self.done.data_ptr(), self.score.data_ptr(), sb.tok.data_ptr(), sb.ftok.data_ptr(),
            sb.parent.data_ptr(), self.tok_hist.data_ptr(), self.par_hist.data_ptr(),
            self.fac_hist.data_ptr(), sb.fac.data_ptr() if nf else None, sb.fac.stride(0),
            model.fac_off.data_ptr(), sb.lse_part.data_ptr(), sb.lse_part.shape[1] // 2, 1, 0,
            self.cand_score.data_ptr(), self.cand_lp.data_ptr(),
            self.cand_col.data_ptr(), self.cand_cnt.data_ptr(), self.row_argmax.data_ptr(),
            self.fac_choice.data_ptr(), self.counter.data_ptr(), self.best_norm.data_ptr(),
            self.best_logprob.data_ptr(), self.best_steps.data_ptr(),
            self.best_forced.data_ptr(), self.best_parent.data_ptr(), self.best_fac.data_ptr(),
            self.n_done.data_ptr())

    def _encode(self):
        """Encoder + all layers' cross K/V (model.py:414-430, 527-531)."""
        m = self.model
        nsf = len(m.config.source_factor_specs)
        enc = m.encode_device(self.ids_d, self.fids_d if nsf else None, self.len_d,
                              self.B, self.L)
        if self.nvs_threshold is not None:
            self._setup_vocab(nvs_active_sets(m, enc, self.len_d, self.B, self.L,
                                              self.nvs_threshold, self.jobs))
        if m.config.decoder_layers:
            m.cross_kv_device(enc, out=self.sb.ckv)
        if self._gather_E:
            kern.gather_rows(m.E_trg_c, self.col_token, self.sb.E_out)

    # ------------------------------------------------------------- stepping
    def _one_step(self):
        step_forward(self.model, self.sb)
        kern.beam_step(self.sb.logits, self.state)
        kern.beam_reorder(self.sb.anc, self.sb.parent, self.sb.step, self.R, self.S_max)

    def run(self) -> list[ChunkResult]:
        self._encode()
        before = kern.launches
        self._one_step()                      # step 0 eagerly (also warms every kernel)
        self.launches_per_step = kern.launches - before
        self.steps_run = 1
        remaining = self.S_max - 1
        host_done = torch.zeros(1, dtype=I32, pin_memory=True)
        if remaining > 0 and self.use_graph:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._one_step()
            kern.launches -= self.launches_per_step  # capture does not launch
        while remaining > 0:
            n = min(self.GRAPH_POLL, remaining)
            for _ in range(n):
                if self.graph is not None:
                    self.graph.replay()
                    kern.launches += self.launches_per_step
                else:
                    self._one_step()
            remaining -= n
            self.steps_run += n
            if remaining > 0:
                host_done.copy_(self.n_done, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                if int(host_done[0]) >= self.B:
                    break
        return self.collect()

    def collect(self) -> list[ChunkResult]:
        c = self.model.config
        nf = len(c.target_factor_specs)
        B = self.B
        kern.beam_finalize(self.state, self.tokens_out, self.factors_out)
        toks, facs = self.tokens_out.cpu().numpy(), self.factors_out.cpu().numpy()
        steps = self.best_steps.cpu().numpy()
        lp = self.best_logprob.cpu().numpy()
        forced = self.best_forced.cpu().numpy()
        out = []
        for b in range(B):
            s = int(steps[b])
            if s <= 0:
                raise RuntimeError("device search finished without a hypothesis")
            out.append(ChunkResult([int(x) for x in toks[b, :s - 1]],
                                   [[int(x) for x in facs[b, k, :s]] for k in range(nf)],
                                   float(lp[b]), s, bool(forced[b])))
        return out


def decode_jobs(model: Model, jobs: list[ChunkJob], beam: int, alpha: float,
                nvs_threshold: float | None = None, max_rows: int = 2560,
                use_graph: bool = True) -> list[ChunkResult]:
    """Decode chunks in length-sorted device batches of <= max_rows rows.
    Results are independent of batch composition (row-wise kernels with a
    fixed reduction order), so sorting never changes outputs."""
    if not jobs:
        return []
    order = sorted(range(len(jobs)), key=lambda i: -len(jobs[i].src_ids))
    per_batch = max(1, max_rows // beam)
    results: list[ChunkResult | None] = [None] * len(jobs)
    for s in range(0, len(order), per_batch):
        idx = order[s:s + per_batch]
        bb = BeamBatch(model, [jobs[i] for i in idx], beam, alpha, nvs_threshold, use_graph)
        for i, r in zip(idx, bb.run()):
            results[i] = r
    return results


# =========================================================== model protocol
class _HostView:
    """Tensor-like wrapper: `.data` gives the numpy array (host copy)."""

    def __init__(self, t: torch.Tensor):
        self.device_tensor = t
        self._np = None

    @property
    def data(self) -> np.ndarray:
        if self._np is None:
            self._np = self.device_tensor.cpu().numpy()
        return self._np

    @property
    def shape(self):
        return tuple(self.device_tensor.shape)


@dataclass
class StepOutput:
    """model.py:275-280."""
    surface: _HostView
    factors: list
    active_ids: np.ndarray | None


class ProtocolState:
    """DecodeState of the reference protocol (model.py:302-330) on the GPU:
    decode_step / select_rows in arbitrary order, as cli bench and the
    teacher-forced parity tests drive them."""

    @classmethod
    def create(cls, model: Model, src_ids, src_factor_ids, lengths, active_ids=None):
        src_ids = np.asarray(src_ids)
        lengths = np.asarray(lengths)
        B = src_ids.shape[0]
        jobs = []
        for b in range(B):
            n = int(lengths[b])
            jobs.append(ChunkJob([int(x) for x in src_ids[b, :n]],
                                 [[int(x) for x in np.asarray(f)[b, :n]] for f in src_factor_ids]))
        if len(src_factor_ids) != len(model.config.source_factor_specs):
            raise ShapeError(f"model wants {len(model.config.source_factor_specs)} source factor "
                             f"streams, got {len(src_factor_ids)}")
        self = cls()
        self.model = model
        from .model import DeviceEncoding
        enc, len_d, B, L = _encode_batch(model, jobs)
        # the reference encodes the padded width it is given; the pad bias
        # hides positions >= length, so the tight width gives the same rows
        self.enc = DeviceEncoding(enc, len_d, B, L)
        self.B, self.L, self.len_d = B, L, len_d
        self.ckv = model.cross_kv_device(enc) if model.config.decoder_layers else None
        if active_ids is not None:
            active_ids = validate_active_ids(model.config, active_ids)
        self.active_ids = active_ids
        self.step = 0
        self._alloc(B, torch.arange(B, dtype=I32, device=model.device))
        return self

    @property
    def batch(self) -> int:
        return self.R

    def _out_matrix(self):
        m = self.model
        if self.active_ids is None:
            return m.E_trg_c, m.config.trg_vocab_size
        idx = torch.from_numpy(self.active_ids.astype(np.int32)).to(m.device)
        E = torch.empty(idx.numel(), m.config.d_model, device=m.device, dtype=m.cdt)
        kern.gather_rows(m.E_trg_c, idx, E)
        return E, idx.numel()

    def _alloc(self, R, row_sent, old: StepBuffers | None = None):
        """(Re)build the step buffers for R rows.  The KV-cache capacity only
        grows: ancestor entries keep pointing at physical slots of earlier
        rows, which must stay addressable."""
        m = self.model
        S = m.max_steps
        E, U = self._E if hasattr(self, "_E") else self._out_matrix()
        self._E = (E, U)
        cap = max(R, old.kc.shape[1] if old is not None and old.kc is not None else 0)
        sb = StepBuffers(m, R, self.B, self.L, S, U, E, self.ckv, self.len_d, row_sent, cap)
        if old is not None:
            sb.step.copy_(old.step)
            if old.kc is not None:
                sb.kc[:, :old.kc.shape[1]].copy_(old.kc)
                sb.vc[:, :old.vc.shape[1]].copy_(old.vc)
        self.sb, self.R = sb, R

    def step_forward(self, prev_ids, prev_factor_ids) -> StepOutput:
        m = self.model
        c = m.config
        if self.step >= 2 * c.max_seq_len + 10:
            raise ShapeError("decode ran past the hard position limit")
        prev = np.asarray(prev_ids).reshape(-1).astype(np.int32)
        if prev.size != self.R:
            raise ShapeError(f"prev_ids has {prev.size} rows, state has {self.R}")
        if len(prev_factor_ids) != len(c.target_factor_specs):
            raise ShapeError(f"model wants {len(c.target_factor_specs)} target factor streams, "
                             f"got {len(prev_factor_ids)}")
        if (prev < 0).any() or (prev >= c.trg_vocab_size).any():
            raise ShapeError("ids out of range for embedding table")
        sb = self.sb
        sb.tok.copy_(torch.from_numpy(prev))
        for k, f in enumerate(prev_factor_ids):
            sb.ftok[k].copy_(torch.from_numpy(np.asarray(f).reshape(-1).astype(np.int32)))
        step_forward(m, sb)
        logits = sb.logits.clone()
        nf = len(c.target_factor_specs)
        facs = []
        off = m.fac_off.cpu().numpy()
        for k in range(nf):
            facs.append(_HostView(sb.fac[:, off[k]:off[k + 1]].clone()))
        # identity reorder: row r keeps its own history (anc parity + step++)
        sb.parent.copy_(torch.arange(self.R, dtype=I32, device=m.device))
        kern.beam_reorder(sb.anc, sb.parent, sb.step, self.R, sb.S_max)
        self.step += 1
        return StepOutput(_HostView(logits), facs, self.active_ids)

    def select_rows(self, indices) -> None:
        """model.py:316-330: keep/repeat rows.  Gathers the ancestor table
        and SSRU cells; the KV cache stays in place."""
        m = self.model
        idx_np = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx_np.size and (idx_np.min() < 0 or idx_np.max() >= self.R):
            raise ShapeError("select_rows index out of range")
        n = int(idx_np.size)
        idx = torch.from_numpy(idx_np.astype(np.int32)).to(m.device)
        old = self.sb
        t = self.step
        row_sent = torch.empty(n, dtype=I32, device=m.device)
        kern.gather_rows(old.row_sent.view(-1, 1), idx, row_sent.view(-1, 1))
        anc_cur = old.anc[t & 1]
        anc_new = torch.empty(n, old.S_max, dtype=I32, device=m.device)
        kern.gather_rows(anc_cur, idx, anc_new)
        cells = None
        if old.cell is not None and t > 0:
            prev = (t - 1) & 1
            cells = [torch.empty(n, m.config.d_model, device=m.device) for _ in m.dec]
            for li in range(len(m.dec)):
                kern.gather_rows(old.cell[li, prev], idx, cells[li])
        self._alloc(n, row_sent, old)
        sb = self.sb
        sb.anc[t & 1, :n].copy_(anc_new)
        if cells is not None:
            prev = (t - 1) & 1
            for li in range(len(m.dec)):
                sb.cell[li, prev, :n].copy_(cells[li])
