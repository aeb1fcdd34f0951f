"""Device-resident encoder-decoder model (mirrors skiff model.py:343-585).

Weights live on the GPU in the layout the kernels want:
  * every linear weight stays (out, in) row-major = K-major, the operand
    layout of the tcgen05 "TN" GEMM; Q|K|V of a self-attention block are
    concatenated into one [3d, d] operand, all decoder layers' cross K|V
    into one [D*2d, d] operand (one GEMM per sentence batch), the SSRU's
    [W_f; W] interleaved row-wise so one GEMM feeds the fused cell epilogue;
  * GEMM operands are bf16 (precision="bf16", tensor cores) or fp32
    (precision="fp32", SIMT FFMA parity mode); norms, biases, embedding
    lookups and the residual stream stay fp32.

`Model.decode_init / decode_step / DecodeState.select_rows / nvs_select`
keep the reference's model protocol (the interface search.py and
cli._cmd_bench call, and that test_search.py's StubModel mocks), running on
the same kernels as the batched engine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kern
from . import _native as N
from .config import SSRU, ModelConfig, check_params, init_params
from .errors import ConfigError, ShapeError
from .shortlist import sorted_union

PAD_ID, UNK_ID, BOS_ID, EOS_ID, SHIFT_ID = 0, 1, 2, 3, 4


def positional_encoding(length: int, dim: int, offset: int = 0) -> np.ndarray:
    """Interleaved sinusoids in float64, cast to float32 (model.py:161-171)."""
    pos = np.arange(offset, offset + length, dtype=np.float64)[:, None]
    half = (dim + 1) // 2
    freq = np.exp(-math.log(10000.0) * (2.0 * np.arange(half) / dim))[None, :]
    ang = pos * freq
    pe = np.zeros((length, 2 * half), dtype=np.float64)
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang)
    return pe[:, :dim].astype(np.float32)


def validate_active_ids(config: ModelConfig, active_ids) -> np.ndarray:
    """model.py:333-340."""
    ids = sorted_union(active_ids)
    if ids.size == 0:
        raise ConfigError("restricted output vocabulary is empty")
    if ids[0] < 0 or ids[-1] >= config.trg_vocab_size:
        raise ConfigError("restricted vocabulary ids out of range")
    return ids


class _Layer:
    pass


class Model:
    """Encoder/decoder weights on one GPU plus the reference model protocol."""

    def __init__(self, config: ModelConfig, params: dict | None = None, seed: int = 13,
                 precision: str = "bf16", device: str = "cuda", gemm_split: str = "throughput"):
        """gemm_split (bf16 only) fixes how the tensor-core GEMMs split K, i.e.
        the fp32 summation order of every projection — a property of the model,
        the same at every batch size, so a sentence's result never depends on
        its batch either way.  "throughput": the library's rule (K = 4096 split
        in 4, else whole-K tiles; best at serving batches of hundreds of rows).
        "latency": every decoder/encoder projection split into partials of
        <= 256 K (kern.latency_k_split), so each CTA's weight slice is fetched
        while the previous kernel still runs (best for batch-1 decoding)."""
        config.validate()
        if precision not in ("bf16", "fp32"):
            raise ConfigError(f"precision must be bf16 or fp32, got {precision!r}")
        if gemm_split not in ("throughput", "latency"):
            raise ConfigError(f"gemm_split must be throughput or latency, got {gemm_split!r}")
        if params is None:
            params = init_params(config, seed)
        params = {n: (v.data if hasattr(v, "data") and not isinstance(v, np.ndarray) else v)
                  for n, v in params.items()}
        check_params(config, params)
        self.config = config
        self.precision = precision
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ConfigError("the B200 backend needs a CUDA device (no CPU fallback)")
        if self.device.index is not None:
            N.call("skb_set_device", self.device.index)
        self.cdt = torch.bfloat16 if precision == "bf16" else torch.float32
        self.quantized: dict = {}
        self.gemm_split = gemm_split
        self._upload(params)
        self.params = params
        if gemm_split == "latency" and precision == "bf16":
            for L in self.enc + self.dec:
                for name in ("wqkv", "wo", "wq_c", "wo_c", "w1", "w2", "w_ssru"):
                    w = getattr(L, name, None)
                    if w is not None:
                        w._skb_k_split = kern.latency_k_split(w.shape[1])

    # ------------------------------------------------------------ weights
    def _f32(self, a):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device=self.device)

    def _c(self, a):
        return self._f32(a).to(self.cdt).contiguous()

    def _upload(self, p):
        c = self.config
        d = c.d_model
        f32, cw = self._f32, self._c
        self.E_src = f32(p["embed.src.surface"])
        self.E_trg = f32(p["embed.trg.surface"])
        self.E_trg_c = self.E_trg if self.cdt == torch.float32 else cw(p["embed.trg.surface"])
        self.src_factor_tables = [f32(p[f"embed.src.factor{i}"])
                                  for i in range(len(c.source_factor_specs))]
        self.trg_factor_tables = [f32(p[f"embed.trg.factor{i}"])
                                  for i in range(len(c.target_factor_specs))]
        self.src_ftab_ptrs = torch.tensor([t.data_ptr() for t in self.src_factor_tables] or [0],
                                          dtype=torch.int64, device=self.device)
        self.trg_ftab_ptrs = torch.tensor([t.data_ptr() for t in self.trg_factor_tables] or [0],
                                          dtype=torch.int64, device=self.device)
        # source positions: max_seq_len rounded up to 8 (the engine pads a
        # batch's source width to a multiple of 8; encode_device checks it)
        self.pe_rows = (c.max_seq_len + 7) // 8 * 8
        self.pe_src = f32(positional_encoding(self.pe_rows, c.surface_embed_dim))
        self.max_steps = 2 * c.max_seq_len + 10  # model.py:543-544
        self.pe_trg = f32(positional_encoding(self.max_steps, d))

        def norm(prefix):
            return f32(p[prefix + ".gain"]), f32(p[prefix + ".bias"])

        self.enc = []
        for i in range(c.encoder_layers):
            b = f"encoder.layer{i}"
            L = _Layer()
            L.ln1 = norm(b + ".self_attn_norm")
            L.wqkv = cw(np.concatenate([p[b + ".self_attn.wq"], p[b + ".self_attn.wk"],
                                        p[b + ".self_attn.wv"]], 0))
            L.wo = cw(p[b + ".self_attn.wo"])
            L.ln2 = norm(b + ".ffn_norm")
            L.ln_ffn = L.ln2
            L.w1, L.b1 = cw(p[b + ".ffn.w1"]), f32(p[b + ".ffn.b1"])
            L.w2, L.b2 = cw(p[b + ".ffn.w2"]), f32(p[b + ".ffn.b2"])
            self.enc.append(L)
        self.dec = []
        ckv = []
        for i in range(c.decoder_layers):
            b = f"decoder.layer{i}"
            L = _Layer()
            if c.decoder_kind == SSRU:
                L.ln_self = norm(b + ".ssru_norm")
                wf, w = p[b + ".ssru.wf"], p[b + ".ssru.w"]
                inter = np.empty((2 * d, d), dtype=np.float32)
                inter[0::2], inter[1::2] = wf, w       # rows (f_j, Wx_j)
                L.w_ssru = cw(inter)
                bi = np.zeros(2 * d, dtype=np.float32)
                bi[0::2] = p[b + ".ssru.bf"]
                L.b_ssru = f32(bi)
            else:
                L.ln_self = norm(b + ".self_attn_norm")
                L.wqkv = cw(np.concatenate([p[b + ".self_attn.wq"], p[b + ".self_attn.wk"],
                                            p[b + ".self_attn.wv"]], 0))
                L.wo = cw(p[b + ".self_attn.wo"])
            L.ln_cross = norm(b + ".cross_attn_norm")
            L.wq_c = cw(p[b + ".cross_attn.wq"])
            L.wo_c = cw(p[b + ".cross_attn.wo"])
            ckv += [p[b + ".cross_attn.wk"], p[b + ".cross_attn.wv"]]
            L.ln_ffn = norm(b + ".ffn_norm")
            L.w1, L.b1 = cw(p[b + ".ffn.w1"]), f32(p[b + ".ffn.b1"])
            L.w2, L.b2 = cw(p[b + ".ffn.w2"]), f32(p[b + ".ffn.b2"])
            self.dec.append(L)
        self.w_ckv = cw(np.concatenate(ckv, 0)) if ckv else None
        self.ln_final = norm("decoder.final_norm")
        nf = len(c.target_factor_specs)
        if nf:
            self.w_fac = cw(np.concatenate([p[f"output.factor{k}.w"] for k in range(nf)], 0))
            self.b_fac = f32(np.concatenate([p[f"output.factor{k}.b"] for k in range(nf)], 0))
            off = np.cumsum([0] + [s.vocab_size for s in c.target_factor_specs])
            self.fac_off = torch.tensor(off, dtype=torch.int32, device=self.device)
        else:
            self.w_fac = self.b_fac = None
            self.fac_off = torch.zeros(1, dtype=torch.int32, device=self.device)
        if c.nvs_enabled:
            self.w_nvs, self.b_nvs = cw(p["nvs.w"]), f32(p["nvs.b"])

    # ------------------------------------------------------------ encoder
    def encoder_buffers(self, n: int) -> dict:
        """Preallocated encoder work buffers for n = B*L positions."""
        c, dev, cdt = self.config, self.device, self.cdt
        d = c.d_model
        bufs = dict(x=torch.empty(n, d, device=dev), h=torch.empty(n, d, device=dev, dtype=cdt),
                    qkv=torch.empty(n, 3 * d, device=dev, dtype=cdt),
                    ctx=torch.empty(n, d, device=dev, dtype=cdt),
                    f=torch.empty(n, c.ff_dim, device=dev, dtype=cdt),
                    xc=torch.empty(n, d, device=dev, dtype=cdt))
        if self.quantized:
            from .quant import Int8Scratch
            bufs["int8"] = Int8Scratch(n, d, c.ff_dim, dev)
        return bufs

    def encode_device(self, ids: torch.Tensor, fids: torch.Tensor | None, lengths: torch.Tensor,
                      B: int, L: int, bufs: dict | None = None) -> torch.Tensor:
        """Batched pre-norm encoder (model.py:414-430), no final LN.
        ids [B*L] int32 (padded), fids [n_factors, B*L] int32, lengths [B]
        int32.  Returns enc fp32 [B*L, d]."""
        c = self.config
        d, H, dh = c.d_model, c.heads, c.head_dim
        if L > self.pe_rows:
            # embed_source reads one positional-encoding row per position
            raise ShapeError(f"source width {L} exceeds the model's {c.max_seq_len} positions")
        n = B * L
        dev, cdt = self.device, self.cdt
        bufs = bufs or self.encoder_buffers(n)
        x = bufs["x"]
        specs = c.source_factor_specs
        kern.embed_source(ids, self.E_src, self.pe_src, [s.dim for s in specs],
                          [0 if s.combine == "sum" else 1 for s in specs], fids,
                          self.src_ftab_ptrs, x, B, L, d)
        if not self.enc:
            return x
        h, qkv, ctx, f = bufs["h"], bufs["qkv"], bufs["ctx"], bufs["f"]
        for Ly in self.enc:
            kern.layernorm(x, *Ly.ln1, h)
            kern.gemm(h, Ly.wqkv, qkv)
            kern.encoder_attention(qkv, lengths, ctx, B, L, H, dh)
            kern.gemm(ctx, Ly.wo, x, N.EPI_RESID)
            if getattr(Ly, "q1", None) is not None:  # int8 feed-forward (quant.py)
                from .quant import Int8Scratch, ffn_int8
                if bufs.get("int8") is None or bufs["int8"].h.shape[0] < n:
                    bufs["int8"] = Int8Scratch(n, d, c.ff_dim, dev)
                ffn_int8(Ly, x, bufs["int8"], n)
                continue
            kern.layernorm(x, *Ly.ln2, h)
            kern.gemm(h, Ly.w1, f, N.EPI_RELU, Ly.b1)
            kern.gemm(f, Ly.w2, x, N.EPI_RESID, Ly.b2)
        return x

    def cross_kv_device(self, enc: torch.Tensor, out: torch.Tensor | None = None,
                        tmp: torch.Tensor | None = None) -> torch.Tensor:
        """All decoder layers' cross K|V in one GEMM (model.py:527-531)."""
        n, d = enc.shape
        if self.cdt == torch.float32:
            a = enc
        else:
            a = tmp if tmp is not None else torch.empty(n, d, device=self.device, dtype=self.cdt)
            kern.convert(enc, a)
        if out is None:
            out = torch.empty(n, self.w_ckv.shape[0], device=self.device, dtype=self.cdt)
        kern.gemm(a, self.w_ckv, out)
        return out

    def nvs_logits_device(self, enc, lengths, B, L) -> torch.Tensor:
        """nvs_logits (model.py:496-501): masked max-pool over the unpadded
        encoder positions, then one linear layer; fp32 [B, V]."""
        d, V = self.config.d_model, self.config.trg_vocab_size
        pooled = torch.empty(B, d, device=self.device)
        kern.masked_maxpool(enc, lengths, pooled, B, L, d)
        if self.cdt != torch.float32:
            pc = torch.empty(B, d, device=self.device, dtype=self.cdt)
            kern.convert(pooled, pc)
        else:
            pc = pooled
        logits = torch.empty(B, V, device=self.device)
        kern.gemm(pc, self.w_nvs, logits, N.EPI_STORE, self.b_nvs)
        return logits

    def nvs_mask_device(self, enc, lengths, B, L, threshold) -> torch.Tensor:
        """NVS head (model.py:496-517): masked max-pool, linear, sigmoid >
        threshold, as a [B, ceil(V/32)] bitmask on the device."""
        V = self.config.trg_vocab_size
        logits = self.nvs_logits_device(enc, lengths, B, L)
        mask = torch.empty(B, (V + 31) // 32, device=self.device, dtype=torch.int32)
        kern.nvs_mask(logits, float(np.float32(threshold)), mask)
        return mask

    def nvs_select(self, enc, lengths, threshold: float, always_include) -> list[np.ndarray]:
        """model.py:502-517 on the device; enc is a DeviceEncoding or state."""
        if not self.config.nvs_enabled:
            raise ConfigError("model was built without vocabulary selection")
        if not (0.0 <= threshold <= 1.0):
            raise ConfigError(f"nvs threshold {threshold} outside [0, 1]")
        B, L = enc.B, enc.L
        mask = self.nvs_mask_device(enc.x, enc.lengths, B, L, threshold).cpu().numpy()
        forced = np.asarray(sorted(set(int(i) for i in always_include)), dtype=np.int64)
        return [np.union1d(mask_to_ids(m, self.config.trg_vocab_size), forced).astype(np.int64)
                for m in mask]

    # ----------------------------------------------------------- protocol
    def decode_init(self, src_ids, src_factor_ids, lengths, active_ids=None):
        """model.py:521-534 on the device."""
        from .engine import ProtocolState
        return ProtocolState.create(self, src_ids, src_factor_ids, lengths, active_ids)

    def decode_step(self, state, prev_ids, prev_factor_ids):
        """model.py:536-585 on the device; surface logits come back as a
        host-readable tensor wrapper (`.data` is numpy, `.device_tensor` the
        GPU buffer)."""
        return state.step_forward(prev_ids, prev_factor_ids)

    def forward_sequence(self, src_ids, src_factor_ids, src_lengths, trg_in_ids,
                         trg_in_factor_ids) -> "SequenceOutput":
        """model.py:444-492, teacher forced: target inputs carry BOS at
        position 0 (and the shift marker in factor streams).  One batched
        pass over all B x T positions (engine.teacher_forced: causal
        self-attention kernel, SSRU recurrence scan, B*T-row GEMMs).
        surface: raw logits [B, T, V]."""
        from .engine import _HostView, teacher_forced
        surface, facs, st = teacher_forced(self, src_ids, src_factor_ids, src_lengths,
                                           trg_in_ids, trg_in_factor_ids)
        nvs = None
        if self.config.nvs_enabled:
            nvs = _HostView(self.nvs_logits_device(st.enc.x, st.enc.lengths, st.enc.B, st.enc.L))
        return SequenceOutput(_HostView(surface), [_HostView(f) for f in facs], nvs)

    def forward_sequence_stepwise(self, src_ids, src_factor_ids, src_lengths, trg_in_ids,
                                  trg_in_factor_ids) -> "SequenceOutput":
        """The same outputs position by position through the incremental
        decode step (cached K/V, SSRU state) — the reference's own invariant
        between the two paths (test_model.py:270-282)."""
        from .engine import _HostView
        trg = np.asarray(trg_in_ids)
        if trg.ndim != 2:
            raise ShapeError(f"trg_in_ids must be [B, T], got shape {trg.shape}")
        B, T = trg.shape
        c = self.config
        fac_in = [np.asarray(f) for f in trg_in_factor_ids]
        if len(fac_in) != len(c.target_factor_specs):
            raise ShapeError(f"model wants {len(c.target_factor_specs)} target factor streams, "
                             f"got {len(fac_in)}")
        st = self.decode_init(src_ids, src_factor_ids, src_lengths)
        surf, facs = [], [[] for _ in fac_in]
        for t in range(T):
            o = self.decode_step(st, trg[:, t], [f[:, t] for f in fac_in])
            surf.append(o.surface.device_tensor)
            for k, f in enumerate(o.factors):
                facs[k].append(f.device_tensor)
        nvs = None
        if c.nvs_enabled:
            nvs = _HostView(self.nvs_logits_device(st.enc.x, st.enc.lengths, st.enc.B, st.enc.L))
        return SequenceOutput(_HostView(torch.stack(surf, 1)),
                              [_HostView(torch.stack(f, 1)) for f in facs], nvs)


def mask_to_ids(mask_row: np.ndarray, V: int) -> np.ndarray:
    bits = np.unpackbits(mask_row.astype("<u4").view(np.uint8), bitorder="little")
    return np.flatnonzero(bits[:V]).astype(np.int64)


@dataclass
class SequenceOutput:
    """model.py:283-288: teacher-forced outputs (host-readable wrappers)."""
    surface: object
    factors: list
    nvs: object | None


@dataclass
class DeviceEncoding:
    x: torch.Tensor        # [B*L, d] fp32
    lengths: torch.Tensor  # [B] int32
    B: int
    L: int
