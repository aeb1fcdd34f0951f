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

import os
import weakref
from collections import OrderedDict

import numpy as np
import torch

from . import kern
from . import _native as N
from .config import SSRU
from .errors import ConfigError, ShapeError
from .model import BOS_ID, EOS_ID, PAD_ID, SHIFT_ID, UNK_ID, Model, validate_active_ids
from .shortlist import sorted_union

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
        # LayerNorm fused into the residual GEMMs (bf16 path, SKB_FUSE_LN=1):
        # arrival tickets per (call site, 16-row tile), monotonic, never reset.
        # Off by default: measured on B200 the separate LayerNorm launch is
        # faster once several decode streams overlap (4510 vs 3510 sent/s).
        self.fuse_ln = (cdt == torch.bfloat16 and d % 128 == 0 and d <= 1024 and D > 0
                        and os.environ.get("SKB_FUSE_LN", "0") == "1" and not model.quantized)
        # int8 feed-forward scratch (quant.quantize_model)
        self.int8 = None
        if model.quantized:
            from .quant import Int8Scratch
            self.int8 = Int8Scratch(R, d, c.ff_dim, dev)
        self.ln_ctr = torch.zeros(3 * max(D, 1), (R + 15) // 16 + 1, dtype=I32, device=dev)
        # per-step self-attention plan (skb_attn_plan), allocated on the first
        # (eager) step once the group size is known
        self.plan = None
        self.plan_key = None
        self.use_plan = (c.decoder_kind != SSRU and cdt == torch.bfloat16 and c.head_dim == 64
                         and os.environ.get("SKB_ATTN_PLAN", "1") != "0"
                         and os.environ.get("SKB_ATTN_TC", "1") != "0")


def step_forward(model: Model, sb: StepBuffers) -> None:
    """Enqueue one decoder step for all rows (model.py:536-585)."""
    c = model.config
    d, H, dh = c.d_model, c.heads, c.head_dim
    R = sb.R
    nf = len(c.target_factor_specs)
    kern.embed_target(sb.tok, model.E_trg, model.pe_trg, sb.step, sb.ftok if nf else None,
                      model.trg_ftab_ptrs if nf else None, sb.x)
    fuse = sb.fuse_ln
    D = len(model.dec)

    def resid(A, W, bias, site, ln):
        """x += A.W^T (+bias); with SKB_FUSE_LN the epilogue also writes h = LN(x)."""
        if fuse:
            kern.gemm(A, W, sb.x, N.EPI_RESID, bias, ln=ln, ln_out=sb.h, ln_counter=sb.ln_ctr[site])
        else:
            kern.gemm(A, W, sb.x, N.EPI_RESID, bias)

    def on_h(W, out, kind, bias, ln, h_ready, **kw):
        """GEMM over h = LN(x) (model.py:562-581).  Unless the fused residual
        epilogue already wrote h, the LayerNorm runs in the GEMM's prologue
        (small batches) or as a launch right before it (identical bits)."""
        kern.gemm(sb.h, W, out, kind, bias, ln_in=None if h_ready else (sb.x, *ln), **kw)

    plan = None
    if sb.use_plan and D > 0 and 1 <= sb.group <= 16:
        key = (R, sb.group, sb.S_max)
        if sb.plan_key != key:
            sb.plan = torch.empty(kern.attn_plan_bytes(R, sb.group, sb.S_max), dtype=torch.uint8,
                                  device=sb.x.device)
            sb.plan_key = key
        kern.attn_plan(sb.anc, sb.step, sb.plan, R, sb.S_max, sb.group)
        plan = sb.plan
    for li, Ly in enumerate(model.dec):
        nxt = model.dec[li + 1].ln_self if li + 1 < D else model.ln_final
        if c.decoder_kind == SSRU:
            if li == 0 or not fuse:  # the SSRU epilogue updates x: LN first
                kern.layernorm(sb.x, *Ly.ln_self, sb.h)
            kern.gemm(sb.h, Ly.w_ssru, sb.x, N.EPI_SSRU, Ly.b_ssru, c_state=sb.cell[li],
                      src_row=sb.parent, step=sb.step, state_stride=R * d)
            on_h(Ly.wq_c, sb.q, N.EPI_STORE, None, Ly.ln_cross, False)
        else:
            on_h(Ly.wqkv, sb.qkv, N.EPI_STORE, None, Ly.ln_self, fuse and li > 0)
            kern.self_attention_step(sb.qkv, sb.kc[li], sb.vc[li], sb.anc, sb.step, sb.ctx,
                                     R, H, dh, sb.S_max, sb.group, plan=plan)
            resid(sb.ctx, Ly.wo, None, 3 * li, Ly.ln_cross)
            on_h(Ly.wq_c, sb.q, N.EPI_STORE, None, Ly.ln_cross, fuse)
        kern.cross_attention_step(sb.q, sb.ckv, li * 2 * d, li * 2 * d + d, sb.L, sb.row_sent,
                                  sb.lengths, sb.ctx, R, H, dh, sb.group)
        resid(sb.ctx, Ly.wo_c, None, 3 * li + 1, Ly.ln_ffn)
        if getattr(Ly, "q1", None) is not None:  # int8 feed-forward (quant.py)
            from .quant import ffn_int8
            ffn_int8(Ly, sb.x, sb.int8, R)
            continue
        on_h(Ly.w1, sb.f, N.EPI_RELU, Ly.b1, Ly.ln_ffn, fuse)
        resid(sb.f, Ly.w2, Ly.b2, 3 * li + 2, nxt)
    h_ready = fuse and D > 0
    on_h(sb.E_out, sb.logits, N.EPI_LOGITS, None, model.ln_final, h_ready, lse_part=sb.lse_part,
         mask=sb.mask, rows_per_group=sb.group)
    if nf:
        on_h(model.w_fac, sb.fac, N.EPI_STORE, model.b_fac, model.ln_final, h_ready)


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


def _check_source_ids(c, ids: np.ndarray, fids: np.ndarray) -> None:
    """Embedding lookups are unchecked on the device: range-check the
    surface ids and every source-factor stream against its table."""
    if (ids < 0).any() or (ids >= c.src_vocab_size).any():
        raise ShapeError(f"ids out of range [0, {c.src_vocab_size}) for embedding table")
    for k, spec in enumerate(c.source_factor_specs):
        if (fids[k] < 0).any() or (fids[k] >= spec.vocab_size).any():
            raise ShapeError(f"source factor {k} ids out of range [0, {spec.vocab_size})")


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
    _check_source_ids(c, ids, fids)
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


class DecodeWorkspace:
    """Every device buffer, the initial-state image and the captured CUDA
    graphs (encoder; 1 and CHUNK decode steps) for one batch shape.  Reused
    by every BeamBatch of the same shape: a new batch costs one pinned H2D
    copy of its inputs, two D2D state resets and graph replays."""

    CHUNK = int(os.environ.get("SKB_GRAPH_CHUNK", "8"))  # decode steps per captured graph

    @property
    def model(self) -> Model:
        m = self._model()
        if m is None:
            raise RuntimeError("the workspace's model was released")
        return m

    def __init__(self, model: Model, B: int, L: int, S_max: int, K: int, P: int, U: int,
                 alpha: float, restricted: bool):
        c = model.config
        dev = model.device
        nf, nsf = len(c.target_factor_specs), len(c.source_factor_specs)
        # weak: the per-model workspace cache is a WeakKeyDictionary, whose
        # values must not keep their key (the model) alive
        self._model = weakref.ref(model)
        self.B, self.L, self.S_max, self.K, self.P, self.U = B, L, S_max, K, P, U
        self.nf, self.nsf, self.restricted = nf, nsf, restricted
        R = B * K
        self.R = R
        nf1 = max(nf, 1)
        # ---- per-batch inputs: one int32 arena filled by one H2D copy
        self.in_sizes = dict(ids=B * L, fids=max(nsf, 1) * B * L, lengths=B, max_len=B,
                             prefix_len=B, prefix_col=B * P, prefix_fac=B * nf1 * P,
                             col_token=U if restricted else 1,
                             mask=B * ((U + 31) // 32) if restricted else 1)
        tot = sum(self.in_sizes.values())
        self.in_host = torch.zeros(tot, dtype=I32, pin_memory=True)
        self.in_dev = torch.zeros(tot, dtype=I32, device=dev)
        self.inp = {}
        off = 0
        for k, n in self.in_sizes.items():
            self.inp[k] = self.in_dev[off:off + n]
            off += n
        self.inp_host = {}
        off = 0
        for k, n in self.in_sizes.items():
            self.inp_host[k] = self.in_host[off:off + n]
            off += n
        # ---- decode state: int32 / float64 arenas reset from init images
        st_sizes = dict(n_alive=B, done=B, counter=B, best_steps=B, best_forced=B, best_parent=B,
                        best_fac=B * nf1, n_done=1, step=1, tok=R, ftok=nf1 * R, parent=R)
        self.st = {}
        tot = sum(st_sizes.values())
        self.st_i32 = torch.zeros(tot, dtype=I32, device=dev)
        off = 0
        for k, n in st_sizes.items():
            self.st[k] = self.st_i32[off:off + n]
            off += n
        self.st_f64 = torch.zeros(R + 2 * B, dtype=torch.float64, device=dev)
        self.st["score"] = self.st_f64[:R]
        self.st["best_norm"] = self.st_f64[R:R + B]
        self.st["best_logprob"] = self.st_f64[R + B:]
        self.st["n_alive"].fill_(1)
        self.st["tok"].fill_(BOS_ID)
        self.st["ftok"].fill_(SHIFT_ID)
        self.st["parent"].copy_(torch.arange(R, dtype=I32, device=dev))
        self.init_i32 = self.st_i32.clone()
        self.init_f64 = self.st_f64.clone()
        # ---- step buffers (tok/ftok/parent/step alias the state arena)
        self.row_sent = torch.arange(R, dtype=I32, device=dev) // K
        D2 = 2 * c.d_model * c.decoder_layers
        ckv = torch.empty(B * L, max(D2, 1), device=dev, dtype=model.cdt)
        E_out = torch.empty(U, c.d_model, device=dev, dtype=model.cdt) if restricted \
            else model.E_trg_c
        self.sb = StepBuffers(model, R, B, L, S_max, U, E_out, ckv, self.inp["lengths"],
                              self.row_sent)
        sb = self.sb
        sb.step, sb.tok, sb.parent = self.st["step"], self.st["tok"], self.st["parent"]
        sb.ftok = self.st["ftok"].view(nf1, R)
        sb.group = K
        sb.mask = self.inp["mask"].view(B, -1) if restricted else None
        self.enc_bufs = model.encoder_buffers(B * L)
        self.len_pen = torch.tensor([float(s) ** alpha if s > 0 else 1.0 for s in range(S_max + 1)],
                                    dtype=torch.float64, device=dev)

        def z(n, dt=I32):
            return torch.zeros(n, dtype=dt, device=dev)

        self.tok_hist = z(S_max * R)
        self.par_hist = z(S_max * R)
        self.fac_hist = z(S_max * nf1 * R)
        self.cand_score = z(R * K, torch.float64)
        self.cand_lp = z(R * K, torch.float32)
        self.cand_col = z(R * K)
        self.cand_cnt = z(R)
        self.row_argmax = z(R)
        self.fac_choice = z(R * nf1)
        self.tokens_out = z(B * S_max).view(B, S_max)
        self.factors_out = z(B * nf1 * S_max).view(B, nf1, S_max)
        self.out_host = torch.zeros(B * S_max + B * nf1 * S_max + 2 * B, dtype=I32,
                                    pin_memory=True)
        self.lp_host = torch.zeros(B, dtype=torch.float64, pin_memory=True)
        self.out_ready = None
        self.eos_col = None
        self.state = None
        self.graph_enc = self.graph_1 = self.graph_n = None
        self.launches_enc = self.launches_step = 0

    def bind_state(self, eos_col: int) -> None:
        model, sb, st, nf = self.model, self.sb, self.st, self.nf
        self.eos_col = eos_col
        self.state = N.BeamState(
            self.B, self.K, self.U, self.S_max, nf, self.len_pen.data_ptr(), st["step"].data_ptr(),
            N.ptr(self.inp["col_token"]) if self.restricted else None,
            N.ptr(self.inp["mask"]) if self.restricted else None, eos_col,
            self.inp["max_len"].data_ptr(), self.inp["prefix_len"].data_ptr(),
            self.inp["prefix_col"].data_ptr(), self.P,
            self.inp["prefix_fac"].data_ptr() if nf else None, st["n_alive"].data_ptr(),
            st["done"].data_ptr(), st["score"].data_ptr(), st["tok"].data_ptr(),
            st["ftok"].data_ptr(), st["parent"].data_ptr(), self.tok_hist.data_ptr(),
            self.par_hist.data_ptr(), self.fac_hist.data_ptr(),
            sb.fac.data_ptr() if nf else None, sb.fac.stride(0), model.fac_off.data_ptr(),
            sb.lse_part.data_ptr(), sb.lse_part.shape[1] // 2, 1, 0,
            self.cand_score.data_ptr(), self.cand_lp.data_ptr(), self.cand_col.data_ptr(),
            self.cand_cnt.data_ptr(), self.row_argmax.data_ptr(), self.fac_choice.data_ptr(),
            st["counter"].data_ptr(), st["best_norm"].data_ptr(), st["best_logprob"].data_ptr(),
            st["best_steps"].data_ptr(), st["best_forced"].data_ptr(),
            st["best_parent"].data_ptr(), st["best_fac"].data_ptr(), st["n_done"].data_ptr())

    # ---------------------------------------------------------------- work
    def encode(self):
        """Encoder + all layers' cross K/V (model.py:414-430, 527-531)."""
        m = self.model
        enc = m.encode_device(self.inp["ids"], self.inp["fids"].view(max(self.nsf, 1), -1)
                              if self.nsf else None, self.inp["lengths"], self.B, self.L,
                              self.enc_bufs)
        if m.config.decoder_layers:
            m.cross_kv_device(enc, out=self.sb.ckv, tmp=self.enc_bufs["xc"])
        if self.restricted:
            kern.gather_rows(m.E_trg_c, self.inp["col_token"], self.sb.E_out)
        return enc

    def one_step(self):
        step_forward(self.model, self.sb)
        kern.beam_step(self.sb.logits, self.state)
        kern.beam_reorder(self.sb.anc, self.sb.parent, self.sb.step, self.R, self.S_max)

    def reset(self):
        self.st_i32.copy_(self.init_i32, non_blocking=True)
        self.st_f64.copy_(self.init_f64, non_blocking=True)

    def _capture(self, fn, launches_attr):
        STATS["captures"] += 1
        g = torch.cuda.CUDAGraph()
        before = kern.launches
        with torch.cuda.graph(g):
            fn()
        setattr(self, launches_attr, kern.launches - before)
        kern.launches = before  # capture does not launch
        return g

    def run(self, S_run: int, use_graph: bool = True, poll: bool = True) -> int:
        """Encode + decode S_run <= S_max steps (stopping early, one chunk
        late, once every sentence is done).  Returns the number of steps run."""
        if not use_graph:
            self.encode()
            steps = 0
            while steps < S_run:
                self.one_step()
                steps += 1
            return steps
        if self.graph_enc is None:
            self.encode()                      # eager once: warms every kernel
            self.graph_enc = self._capture(self.encode, "launches_enc")
        else:
            self.graph_enc.replay()
            kern.launches += self.launches_enc
            _mark("encoder graph launched")
        steps = 0
        if self.graph_1 is None:
            self.one_step()                    # step 0 eagerly, then capture
            steps = 1
            self.graph_1 = self._capture(self.one_step, "launches_step")
            if self.S_max >= self.CHUNK:
                self.graph_n = self._capture(lambda: [self.one_step() for _ in range(self.CHUNK)],
                                             "launches_chunk")
        done_host = torch.zeros(1, dtype=I32, pin_memory=True)
        ev = None
        while steps < S_run:
            if self.graph_n is not None and S_run - steps >= self.CHUNK:
                if steps == 0:
                    _mark("first decode graph: launch")
                self.graph_n.replay()
                kern.launches += self.launches_chunk
                steps += self.CHUNK
            else:
                self.graph_1.replay()
                kern.launches += self.launches_step
                steps += 1
            if poll and steps < S_run:
                # early exit for finished batches, checked one chunk late so the
                # host never stalls the GPU pipeline; the counter is copied on a
                # side stream, so the decode stream runs the next graph at once
                # (a copy on the decode stream would sit between the graphs)
                if ev is not None and ev.query() and int(done_host[0]) >= self.B:
                    break
                main = torch.cuda.current_stream()
                side = _poll_stream(main)
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    done_host.copy_(self.st["n_done"], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record()
        return steps

    def enqueue_collect(self) -> None:
        """Backtrack the best hypotheses and start one asynchronous D2H copy
        of everything into pinned memory (stream-ordered right after this
        batch's decode, so a following batch can be launched before the
        results are read)."""
        B, S, nf1 = self.B, self.S_max, max(self.nf, 1)
        kern.beam_finalize(self.state, self.tokens_out, self.factors_out)
        h = self.out_host
        h[:B * S].copy_(self.tokens_out.view(-1), non_blocking=True)
        h[B * S:B * S + B * nf1 * S].copy_(self.factors_out.view(-1), non_blocking=True)
        h[B * S + B * nf1 * S:B * S + B * nf1 * S + B].copy_(self.st["best_steps"],
                                                              non_blocking=True)
        h[B * S + B * nf1 * S + B:].copy_(self.st["best_forced"], non_blocking=True)
        self.lp_host.copy_(self.st["best_logprob"], non_blocking=True)
        self.out_ready = torch.cuda.Event()
        self.out_ready.record()

    def collect(self) -> tuple:
        """Wait for the D2H copy of enqueue_collect() and unpack it."""
        if getattr(self, "out_ready", None) is None:
            self.enqueue_collect()
        self.out_ready.synchronize()
        self.out_ready = None
        B, S, nf1 = self.B, self.S_max, max(self.nf, 1)
        h = self.out_host
        lp = self.lp_host.clone()
        arr = h.numpy()
        toks = arr[:B * S].reshape(B, S)
        facs = arr[B * S:B * S + B * nf1 * S].reshape(B, nf1, S)
        steps = arr[B * S + B * nf1 * S:B * S + B * nf1 * S + B]
        forced = arr[B * S + B * nf1 * S + B:]
        return toks, facs, steps, forced, lp.numpy()


_POLL_STREAMS: dict = {}


def _poll_stream(main: torch.cuda.Stream) -> torch.cuda.Stream:
    """Side stream (one per decode stream) for the early-exit counter copies."""
    key = (main.device, main.cuda_stream)
    if key not in _POLL_STREAMS:
        _POLL_STREAMS[key] = torch.cuda.Stream(device=main.device)
    return _POLL_STREAMS[key]


STATS = {"workspaces": 0, "captures": 0}  # cache misses (diagnostics: tools/e2e_var.py)
HOST_TRACE = os.environ.get("SKB_HOST_TRACE", "0") == "1"
HOST_MARKS: list = []  # (label, perf_counter) when SKB_HOST_TRACE=1 (tools/host_timeline.py)


def _mark(label: str) -> None:
    if HOST_TRACE:
        import time
        HOST_MARKS.append((label, time.perf_counter()))


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# Workspaces per model (dropped with the model), least recently used first,
# bounded by device bytes (SKB_WS_BYTES, default 64 GB of the 180 GB: 5 decode
# streams x 2 slots of the big model plus the latency workspaces stay cached).
_WS_CACHE: "weakref.WeakKeyDictionary[Model, OrderedDict]" = weakref.WeakKeyDictionary()
_WS_BYTES = int(float(os.environ.get("SKB_WS_BYTES", 64e9)))


def _ws_bytes(ws) -> int:
    seen, tot = set(), 0
    for v in list(vars(ws).values()) + list(vars(ws.sb).values()) + list(ws.enc_bufs.values()):
        if isinstance(v, torch.Tensor) and v.is_cuda and v.data_ptr() not in seen:
            seen.add(v.data_ptr())
            tot += v.numel() * v.element_size()
    return tot


def _workspace(model, key, *args):
    per = _WS_CACHE.setdefault(model, OrderedDict())
    ws = per.get(key)
    if ws is not None:
        per.move_to_end(key)
        return ws
    ws = DecodeWorkspace(model, *args)
    STATS["workspaces"] += 1
    ws.nbytes = _ws_bytes(ws)
    per[key] = ws
    total = sum(w.nbytes for p in _WS_CACHE.values() for w in p.values())
    while total > _WS_BYTES and len(per) > 1:
        _, old = per.popitem(last=False)  # an in-flight batch keeps its own reference
        total -= old.nbytes
    return ws


def clear_workspaces() -> None:
    _WS_CACHE.clear()


class BeamBatch:
    """One batched beam (or greedy, K=1) run over a cached DecodeWorkspace.

    Construction does the host work and stages every input on the device;
    `run()` is device work: encoder, cross K/V, the captured decode loop,
    finalize, one D2H copy of the results."""

    def __init__(self, model: Model, jobs: list[ChunkJob], beam: int, alpha: float,
                 nvs_threshold: float | None = None, use_graph: bool = True, slot: int = 0):
        _mark("BeamBatch")
        if beam < 1:
            raise ConfigError(f"beam size must be at least 1, got {beam}")
        if beam > 32:
            raise ConfigError(f"beam size {beam} exceeds the device limit of 32")
        self.model, self.jobs, self.K, self.alpha = model, jobs, beam, alpha
        self.use_graph = use_graph
        self.nvs_threshold = nvs_threshold
        self.slot = slot  # workspace slot: consecutive batches alternate (pipelining)
        c = model.config
        nf, nsf = len(c.target_factor_specs), len(c.source_factor_specs)
        self.nf = nf
        B = len(jobs)
        L = max(len(j.src_ids) for j in jobs)
        self.B, self.L, self.R = B, L, B * beam
        max_len = np.array([2 * len(j.src_ids) + 10 for j in jobs], dtype=np.int32)
        # steps this batch runs (the longest chunk's 2L+10 cap, search.py:231-232)
        self.S_run = int(max_len.max())
        # the prefix tables hold the surface prefix AND every prefix-factor
        # stream (a factor stream may reach past the surface prefix)
        P = max([1] + [len(j.prefix_ids) for j in jobs]
                + [len(f) for j in jobs for f in j.prefix_factor_ids[:nf]])
        # Workspace shape buckets (reused across batches of similar shape):
        # padded source width to a multiple of 8 (the encoder's pad bias
        # hides the extra positions; pe rows cover it, Model.pe_rows), prefix
        # width to a multiple of 8; step capacity follows the padded width.
        self.L_ws = min(_round_up(L, 8), model.pe_rows)
        self.P = _round_up(P, 8)
        self.S_max = 2 * self.L_ws + 10
        self._max_len = max_len
        self.ws = None
        self.steps_run = 0
        if nvs_threshold is None:
            self._prepare([j.active_ids for j in jobs])

    # restricted vocabulary (search.py:235-242): union U + per-chunk bitmask
    def _prepare(self, actives):
        model, c = self.model, self.model.config
        B, L, K, P, nf, jobs = self.B, self.L, self.K, self.P, self.nf, self.jobs
        nsf = len(c.source_factor_specs)
        restricted = any(a is not None for a in actives)
        V = c.trg_vocab_size
        if restricted:
            actives = [a if a is not None else np.arange(V, dtype=np.int64) for a in actives]
            U_ids = sorted_union(*actives)
            U_real = int(U_ids.size)
            # union width bucketed to 1024 columns (a batch-1 shortlist run
            # has a different union per sentence; coarse buckets let calls
            # share a workspace and its captured graphs): the padding columns
            # repeat the last id and are never set in any sentence's mask
            U = min(_round_up(U_real, 1024), max(V, U_real))
        else:
            U = V
        Lw = self.L_ws
        key = (B, Lw, K, P, U, self.alpha, restricted, self.slot, kern.concurrency)
        ws = _workspace(model, key, B, Lw, self.S_max, K, P, U, self.alpha, restricted)
        self.ws = ws
        # this batch's inputs: own pinned staging + own device copy (several
        # batches of one shape can be staged before any of them runs)
        self.in_host = torch.zeros_like(ws.in_host, pin_memory=True)
        h = {}
        off = 0
        for k, n in ws.in_sizes.items():
            h[k] = self.in_host[off:off + n]
            off += n
        ids = h["ids"].numpy().reshape(B, Lw)
        ids[:] = 0
        fids = h["fids"].numpy().reshape(max(nsf, 1), B, Lw)
        fids[:] = 0
        lengths = h["lengths"].numpy()
        for b, j in enumerate(jobs):
            n = len(j.src_ids)
            ids[b, :n] = j.src_ids
            lengths[b] = n
            for k in range(nsf):
                fids[k, b, :n] = j.src_factor_ids[k]
        _check_source_ids(c, ids, fids)
        h["max_len"].numpy()[:] = self._max_len
        h["prefix_len"].numpy()[:] = [len(j.prefix_ids) for j in jobs]
        pcol = h["prefix_col"].numpy().reshape(B, P)
        pcol[:] = -1
        pfac = h["prefix_fac"].numpy().reshape(B, max(nf, 1), P)
        pfac[:] = -1
        col_of = None
        if restricted:
            ct = h["col_token"].numpy()
            ct[:U_real] = U_ids.astype(np.int32)
            ct[U_real:] = U_ids[-1]
            mask = h["mask"].numpy().view(np.uint32).reshape(B, -1)
            nbits = mask.shape[1] * 32
            for b, a in enumerate(actives):
                # bit c of row b set for every active column c (little-endian
                # words: column c is bit c & 31 of word c >> 5)
                bits = np.zeros(nbits, dtype=bool)
                bits[np.searchsorted(U_ids, a)] = True
                mask[b] = np.packbits(bits, bitorder="little").view(np.uint32)

            def col_of(tok):
                i = int(np.searchsorted(U_ids, tok))
                if i >= U_real or int(U_ids[i]) != tok:
                    raise ConfigError(f"token id {tok} missing from the restricted vocabulary")
                return i
        for b, j in enumerate(jobs):
            for t, tok in enumerate(j.prefix_ids):
                pcol[b, t] = col_of(tok) if restricted else tok
            for k, stream in enumerate(j.prefix_factor_ids[:nf]):
                pfac[b, k, :len(stream)] = stream
        eos_col = col_of(EOS_ID) if restricted else EOS_ID
        self.eos_col = eos_col
        self.h2d_bytes = self.in_host.numel() * 4
        _mark("inputs packed")
        self.in_dev = self.in_host.to(model.device, non_blocking=True)
        # start() may run on another stream: it waits for this copy
        self.in_ready = torch.cuda.Event()
        self.in_ready.record()

    # the attributes bench.py / tests read
    @property
    def sb(self):
        return self.ws.sb

    @property
    def state(self):
        return self.ws.state

    @property
    def done(self):
        return self.ws.st["done"]

    @property
    def n_alive(self):
        return self.ws.st["n_alive"]

    @property
    def n_done(self):
        return self.ws.st["n_done"]

    @property
    def tokens_out(self):
        return self.ws.tokens_out

    def start(self) -> None:
        """Launch encoder + decode + finalize + the D2H copy; returns without
        waiting (the host can prepare and launch the next batch)."""
        if self.ws is None:  # NVS: the active sets come from the encoder output
            m, c = self.model, self.model.config
            nsf = len(c.source_factor_specs)
            ids = np.zeros((self.B, self.L), dtype=np.int32)
            fids = np.zeros((max(nsf, 1), self.B, self.L), dtype=np.int32)
            lengths = np.zeros(self.B, dtype=np.int32)
            for b, j in enumerate(self.jobs):
                ids[b, :len(j.src_ids)] = j.src_ids
                lengths[b] = len(j.src_ids)
                for k in range(nsf):
                    fids[k, b, :len(j.src_ids)] = j.src_factor_ids[k]
            dev = m.device
            len_d = torch.from_numpy(lengths).to(dev)
            enc = m.encode_device(torch.from_numpy(ids.reshape(-1)).to(dev),
                                  torch.from_numpy(fids.reshape(max(nsf, 1), -1)).to(dev)
                                  if nsf else None, len_d, self.B, self.L)
            self._prepare(nvs_active_sets(m, enc, len_d, self.B, self.L, self.nvs_threshold,
                                          self.jobs))
        _mark("start")
        ws = self.ws
        if ws.state is None or ws.eos_col != self.eos_col:
            ws.bind_state(self.eos_col)
            ws.graph_1 = ws.graph_n = None  # the step graph bakes eos_col in
        torch.cuda.current_stream().wait_event(self.in_ready)
        ws.in_dev.copy_(self.in_dev, non_blocking=True)   # device-resident inputs
        ws.reset()
        _mark("inputs copied, state reset")
        self.steps_run = ws.run(self.S_run, self.use_graph)
        _mark("decode graphs launched")
        ws.enqueue_collect()
        _mark("collect enqueued")

    def finish(self) -> list[ChunkResult]:
        """Wait for this batch's results (launched by start())."""
        return self.collect()

    def run(self) -> list[ChunkResult]:
        self.start()
        return self.finish()

    def collect(self) -> list[ChunkResult]:
        toks, facs, steps, forced, lp = self.ws.collect()
        nf = self.nf
        out = []
        for b in range(self.B):
            s = int(steps[b])
            if s <= 0:
                raise RuntimeError("device search finished without a hypothesis")
            out.append(ChunkResult(toks[b, :s - 1].tolist(),
                                   [facs[b, k, :s].tolist() for k in range(nf)],
                                   float(lp[b]), s, bool(forced[b])))
        return out


class LazyJobs:
    """Chunk jobs built on first access, with their source lengths known up
    front for the length sort: decode_jobs builds a batch's jobs (the host's
    vocabulary encoding) right before launching it, so only the first batch
    waits for host preprocessing and the rest overlaps the GPU work of the
    batches launched before it."""

    def __init__(self, lengths: list[int], make):
        self.lengths = lengths
        self._make = make
        self._jobs: list = [None] * len(lengths)

    def __len__(self) -> int:
        return len(self.lengths)

    def __getitem__(self, i: int) -> ChunkJob:
        j = self._jobs[i]
        if j is None:
            j = self._jobs[i] = self._make(i)
        return j


def decode_jobs(model: Model, jobs, beam: int, alpha: float,
                nvs_threshold: float | None = None, max_rows: int = 2560,
                use_graph: bool = True, on_done=None) -> list[ChunkResult]:
    """Decode chunks (a list of ChunkJob, or LazyJobs) in length-sorted
    device batches of <= max_rows rows.  Results are independent of batch composition (row-wise kernels with a
    fixed reduction order), so sorting never changes outputs.  on_done(i, r)
    is called for every chunk as soon as its batch is read back, while the
    later batches still decode (host post-processing overlaps the GPU)."""
    if not jobs:
        return []
    lens = jobs.lengths if isinstance(jobs, LazyJobs) else [len(j.src_ids) for j in jobs]
    order = sorted(range(len(jobs)), key=lambda i: -lens[i])
    per_batch = max(1, max_rows // beam)
    # Batches run concurrently on DECODE_STREAMS CUDA streams (batch n on
    # stream n % S); on each stream batch n+S is prepared and launched before
    # batch n is read back, so a stream alternates two workspaces.
    with torch.cuda.device(model.device):
        return _decode_jobs(model, jobs, beam, alpha, nvs_threshold, order, per_batch, use_graph,
                            on_done)


def _decode_jobs(model, jobs, beam, alpha, nvs_threshold, order, per_batch, use_graph, on_done=None):
    results: list[ChunkResult | None] = [None] * len(jobs)

    def take(idx, bb):
        _mark("finish: wait")
        rs = bb.finish()
        _mark("finish: done")
        for i, r in zip(idx, rs):
            results[i] = r
            if on_done is not None:
                on_done(i, r)

    n_batches = (len(order) + per_batch - 1) // per_batch
    S = max(1, min(DECODE_STREAMS, n_batches))
    kern.set_concurrency(S)
    pool = _STREAMS.setdefault(model.device.index if model.device.index is not None
                               else torch.cuda.current_device(), [])
    if len(pool) < S:
        pool.extend(torch.cuda.Stream() for _ in range(S - len(pool)))
    main = torch.cuda.current_stream()
    streams = [main] + pool[1:S]
    for st in streams[1:]:
        st.wait_stream(main)
    pending = []
    for n, s in enumerate(range(0, len(order), per_batch)):
        idx = order[s:s + per_batch]
        with torch.cuda.stream(streams[n % S]):
            # constructed on its own stream: the batch's input upload must not
            # queue behind the decode work of the batches on the main stream
            bb = BeamBatch(model, [jobs[i] for i in idx], beam, alpha, nvs_threshold, use_graph,
                           slot=2 * (n % S) + ((n // S) & 1))
            bb.start()
        pending.append((idx, bb))
        if len(pending) > S:
            take(*pending.pop(0))
    for pi, pb in pending:
        take(pi, pb)
    for st in streams[1:]:
        main.wait_stream(st)
    return results


DECODE_STREAMS = int(os.environ.get("SKB_STREAMS", "5"))  # concurrent decode batches per device (serving mode; 5 measured best on B200, profiles/r2_75-77)
_STREAMS: dict = {}  # device index -> decode streams


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


# ============================================================ teacher forced
def teacher_forced(model: Model, src_ids, src_factor_ids, src_lengths, trg_in_ids,
                   trg_in_factor_ids):
    """The full teacher-forced pass (model.py:444-493) for all B x T target
    positions at once: one batched encoder, then per decoder layer GEMMs over
    B*T rows with the causal self-attention kernel (or the SSRU gate GEMM +
    recurrence scan), cross-attention of the B*T queries against each
    sentence's encoder K/V, the feed-forward block, and one output
    projection.  Returns (surface [B, T, V] fp32, factors [B, T, Vk], enc)."""
    c = model.config
    d, H, dh, D = c.d_model, c.heads, c.head_dim, c.decoder_layers
    dev, cdt = model.device, model.cdt
    trg = np.asarray(trg_in_ids)
    if trg.ndim != 2:
        raise ShapeError(f"trg_in_ids must be [B, T], got shape {trg.shape}")
    B, T = trg.shape
    fac_in = [np.asarray(f) for f in trg_in_factor_ids]
    if len(fac_in) != len(c.target_factor_specs):
        raise ShapeError(f"model wants {len(c.target_factor_specs)} target factor streams, "
                         f"got {len(fac_in)}")
    if T > model.max_steps:
        raise ShapeError(f"target length {T} exceeds the {model.max_steps} decoder positions")
    if (trg < 0).any() or (trg >= c.trg_vocab_size).any():
        raise ShapeError("ids out of range for embedding table")
    st = ProtocolState.create(model, src_ids, src_factor_ids, src_lengths)
    n = B * T
    nf = len(fac_in)
    with torch.cuda.device(dev):
        x = torch.empty(n, d, device=dev)
        ids = torch.from_numpy(trg.reshape(-1).astype(np.int32)).to(dev)
        fids = torch.from_numpy(np.stack(fac_in).reshape(max(nf, 1), -1).astype(np.int32)
                                if nf else np.zeros((1, n), np.int32)).to(dev)
        # target embedding + positions 0..T-1 (+ summed factors), model.py:399-410
        kern.embed_source(ids, model.E_trg, model.pe_trg, [d] * nf, [0] * nf,
                          fids if nf else None, model.trg_ftab_ptrs, x, B, T, d)
        h = torch.empty(n, d, device=dev, dtype=cdt)
        ctx = torch.empty(n, d, device=dev, dtype=cdt)
        q = torch.empty(n, d, device=dev, dtype=cdt)
        f = torch.empty(n, c.ff_dim, device=dev, dtype=cdt)
        tlen = torch.full((B,), T, dtype=I32, device=dev)
        row_sent = torch.arange(n, dtype=I32, device=dev) // T
        int8 = None
        if model.quantized:
            from .quant import Int8Scratch
            int8 = Int8Scratch(n, d, c.ff_dim, dev)
        if c.decoder_kind == SSRU:
            g = torch.empty(n, 2 * d, device=dev)
        else:
            qkv = torch.empty(n, 3 * d, device=dev, dtype=cdt)
        for li, Ly in enumerate(model.dec):
            kern.layernorm(x, *Ly.ln_self, h)
            if c.decoder_kind == SSRU:
                kern.gemm(h, Ly.w_ssru, g, N.EPI_STORE)
                kern.ssru_scan(g, Ly.b_ssru, x, B, T, d)
            else:
                kern.gemm(h, Ly.wqkv, qkv, N.EPI_STORE)
                kern.causal_self_attention(qkv, tlen, ctx, B, T, H, dh)
                kern.gemm(ctx, Ly.wo, x, N.EPI_RESID)
            kern.layernorm(x, *Ly.ln_cross, h)
            kern.gemm(h, Ly.wq_c, q, N.EPI_STORE)
            kern.cross_attention_step(q, st.ckv, li * 2 * d, li * 2 * d + d, st.L, row_sent,
                                      st.len_d, ctx, n, H, dh, T)
            kern.gemm(ctx, Ly.wo_c, x, N.EPI_RESID)
            if getattr(Ly, "q1", None) is not None:
                from .quant import ffn_int8
                ffn_int8(Ly, x, int8, n)
                continue
            kern.layernorm(x, *Ly.ln_ffn, h)
            kern.gemm(h, Ly.w1, f, N.EPI_RELU, Ly.b1)
            kern.gemm(f, Ly.w2, x, N.EPI_RESID, Ly.b2)
        kern.layernorm(x, *model.ln_final, h)
        V = c.trg_vocab_size
        surface = torch.empty(n, V, device=dev)
        kern.gemm(h, model.E_trg_c, surface, N.EPI_STORE)
        facs = []
        if nf:
            fac = torch.empty(n, model.w_fac.shape[0], device=dev)
            kern.gemm(h, model.w_fac, fac, N.EPI_STORE, model.b_fac)
            off = model.fac_off.cpu().numpy()
            facs = [fac[:, off[k]:off[k + 1]].reshape(B, T, -1) for k in range(nf)]
    return surface.view(B, T, V), facs, st
