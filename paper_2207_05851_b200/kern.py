"""Thin torch-tensor wrappers over the C ABI (include/skiff_b200.h).

Every function launches hand-written sm_100a kernels on the current torch
stream and counts them in `launches` (the bench reports it as gpu_launches).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _native as N

launches = 0
concurrency = 1  # decode streams sharing the device (GEMM tile sizing; see set_concurrency)


def set_concurrency(n: int) -> None:
    """Tell the GEMMs how many independent decode streams share the device
    (tiles are sized for a 1/n share of the SMs).  Workspaces captured under
    another setting are not reused (the setting is part of their key)."""
    global concurrency
    if not 1 <= int(n) <= 16:
        raise ValueError(f"concurrency {n} out of [1, 16]")
    concurrency = int(n)


def _count(n: int = 1) -> None:
    global launches
    launches += n


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def dcode(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return N.F32
    if t.dtype == torch.bfloat16:
        return N.BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


LATENCY_KB = int(os.environ.get("SKB_LATENCY_KB", "2"))  # k-blocks (64 K) per partial


def latency_k_split(K: int, kb: int = 0) -> int:
    """K-partials of a latency-model projection: the smallest split in
    {1, 2, 4, 8} whose partial spans <= kb 64-wide k-blocks (default 2: a
    128-row weight slice of <= 32 KB per CTA, fetched while the previous
    kernel runs, and 8 serial MMAs).  A function of K only (K = 1024 -> 8,
    K = 4096 -> 8 on the big model: 16-CTA clusters measured slower,
    8.8 vs 6.4 us on the batch-1 critical path)."""
    kb = kb or LATENCY_KB
    nk = (K + 63) // 64
    s = 1
    while s < 8 and (nk + s - 1) // s > kb:
        s *= 2
    return s


def gemm(A, W, out, kind=N.EPI_STORE, bias=None, *, M=None, c_state=None, src_row=None,
         step=None, state_stride=0, lse_part=None, mask=None, rows_per_group=1, simt=False,
         ln=None, ln_out=None, ln_counter=None, eps=1e-5, ln_in=None):
    """out (or residual x) <- epilogue(A[M,K] . W[N,K]^T).  For RESID, ln =
    (gain, bias) with ln_out (bf16) and ln_counter also writes
    ln_out = LayerNorm(x) of the updated rows (fused on the swap-AB kernel,
    else a LayerNorm launch follows).  ln_in = (x, gain, bias): the GEMM input
    is A = LayerNorm(x) (kernels.py:298-324), computed in the GEMM's prologue
    at small M (A is then not written) or by a LayerNorm launch into A."""
    M = A.shape[0] if M is None else M
    Nn, K = W.shape
    epi = N.Epilogue(kind, N.ptr(bias), out.data_ptr(), out.stride(0), dcode(out), None,
                     N.ptr(c_state), N.ptr(src_row), Nn // 2 if kind == N.EPI_SSRU else 0,
                     N.ptr(step), state_stride, N.ptr(lse_part),
                     lse_part.shape[1] // 2 if lse_part is not None else 0, N.ptr(mask),
                     mask.shape[1] if mask is not None else 0, rows_per_group)
    epi.streams = concurrency
    epi.k_split = getattr(W, "_skb_k_split", 0)  # the model's K-split policy (Model.gemm_split)
    if ln is not None:
        epi.ln_gain, epi.ln_bias = ln[0].data_ptr(), ln[1].data_ptr()
        epi.ln_eps = eps
        epi.ln_out, epi.ln_ldo = ln_out.data_ptr(), ln_out.stride(0)
        epi.ln_counter = ln_counter.data_ptr()
    if ln_in is not None:
        x, g, b = ln_in
        epi.ln_in, epi.ln_in_ld = x.data_ptr(), x.stride(0)
        epi.ln_in_gain, epi.ln_in_bias, epi.ln_in_eps = g.data_ptr(), b.data_ptr(), eps
    N.call("skb_gemm_simt" if simt else "skb_gemm", dcode(A), M, Nn, K, A.data_ptr(),
           A.stride(0), W.data_ptr(), W.stride(0), C.byref(epi), stream())
    _count(N.lib().skb_last_launches())


def quantize_rows(x, q, scales, rows=None):
    """q (int8), scales (fp32) <- per-row symmetric quantization of fp32 x
    (quant.py:40-53 / 99-104)."""
    rows = x.shape[0] if rows is None else rows
    N.call("skb_quantize_rows", rows, x.shape[1], x.data_ptr(), x.stride(0), q.data_ptr(),
           q.stride(0), scales.data_ptr(), stream())
    _count()


def gemm_i8(qa, a_scale, qw, w_scale, out, kind=N.EPI_STORE, bias=None, *, M=None):
    """out (or residual x) <- epilogue((f32(qa . qw^T) * a_scale) * w_scale)
    with exact int32 accumulation (quant.py:121-132)."""
    M = qa.shape[0] if M is None else M
    Nn, K = qw.shape
    epi = N.Epilogue(kind, N.ptr(bias), out.data_ptr(), out.stride(0), dcode(out))
    epi.streams = concurrency
    N.call("skb_gemm_i8", M, Nn, K, qa.data_ptr(), qa.stride(0), a_scale.data_ptr(),
           qw.data_ptr(), qw.stride(0), w_scale.data_ptr(), C.byref(epi), stream())
    _count()


def layernorm(x, gain, bias, out, rows=None, eps=1e-5):
    rows = x.shape[0] if rows is None else rows
    N.call("skb_layernorm", rows, x.shape[1], x.data_ptr(), x.stride(0), gain.data_ptr(),
           bias.data_ptr(), C.c_float(eps), out.data_ptr(), out.stride(0), dcode(out), stream())
    _count()


def embed_target(tok, E, pe, step, ftok, ftables, x, rows=None):
    rows = tok.shape[0] if rows is None else rows
    nf = 0 if ftables is None else ftables.shape[0]
    N.call("skb_embed_target", rows, E.shape[1], tok.data_ptr(), E.data_ptr(), pe.data_ptr(),
           step.data_ptr(), nf, N.ptr(ftok) if nf else None, N.ptr(ftables) if nf else None,
           x.data_ptr(), stream())
    _count()


def embed_source(ids, E, pe, fdims, fcombine, fids, ftables, x, B, L, d):
    nf = len(fdims)
    dims = (C.c_int * max(nf, 1))(*fdims)
    comb = (C.c_int * max(nf, 1))(*fcombine)
    N.call("skb_embed_source", B, L, d, E.shape[1], ids.data_ptr(), E.data_ptr(), pe.data_ptr(),
           nf, dims, comb, N.ptr(fids) if nf else None, N.ptr(ftables) if nf else None,
           x.data_ptr(), stream())
    _count()


def encoder_attention(qkv, lengths, ctx, B, L, H, dh):
    N.call("skb_encoder_attention", B, L, H, dh, qkv.data_ptr(), qkv.stride(0), dcode(qkv),
           lengths.data_ptr(), ctx.data_ptr(), ctx.stride(0), dcode(ctx), stream())
    _count()


def causal_self_attention(qkv, lengths, ctx, B, T, H, dh):
    """Teacher-forced decoder self-attention over [B*T, 3d] (model.py:456-462)."""
    N.call("skb_causal_self_attention", B, T, H, dh, qkv.data_ptr(), qkv.stride(0), dcode(qkv),
           lengths.data_ptr(), ctx.data_ptr(), ctx.stride(0), dcode(ctx), stream())
    _count()


def ssru_scan(g, bias, x, B, T, d):
    """SSRU recurrence along T (model.py:482-493): x += relu(c_t)."""
    N.call("skb_ssru_scan", B, T, d, g.data_ptr(), g.stride(0), N.ptr(bias), x.data_ptr(),
           x.stride(0), stream())
    _count()


def self_attention_step(qkv, kc, vc, anc, step, ctx, R, H, dh, S_max, group=1, plan=None):
    """plan (from attn_plan) replaces the per-layer ancestor walk."""
    if plan is not None:
        N.call("skb_self_attention_step_planned", R, H, dh, qkv.data_ptr(), qkv.stride(0),
               dcode(qkv), kc.data_ptr(), vc.data_ptr(), dcode(kc), S_max, plan.data_ptr(),
               step.data_ptr(), group, ctx.data_ptr(), ctx.stride(0), dcode(ctx), stream())
    else:
        N.call("skb_self_attention_step", R, H, dh, qkv.data_ptr(), qkv.stride(0), dcode(qkv),
               kc.data_ptr(), vc.data_ptr(), dcode(kc), S_max, anc.data_ptr(), step.data_ptr(),
               group, ctx.data_ptr(), ctx.stride(0), dcode(ctx), stream())
    _count()


def attn_plan_bytes(R, group, S_max):
    return int(N.lib().skb_attn_plan_bytes(R, group, S_max))


def attn_plan(anc, step, plan, R, S_max, group):
    """Per-step self-attention plan (distinct cache entries + row masks per
    sentence), shared by every decoder layer."""
    N.call("skb_attn_plan", R, group, S_max, anc.data_ptr(), step.data_ptr(), plan.data_ptr(),
           stream())
    _count()


def cross_attention_step(q, kv, koff, voff, L, row_sent, lengths, ctx, R, H, dh, group=1):
    N.call("skb_cross_attention_step", R, H, dh, q.data_ptr(), q.stride(0), dcode(q),
           kv.data_ptr(), kv.stride(0), dcode(kv), koff, voff, L, row_sent.data_ptr(),
           lengths.data_ptr(), group, ctx.data_ptr(), ctx.stride(0), dcode(ctx), stream())
    _count()


def gather_rows(table, idx, out):
    n = idx.shape[0]
    if table.dtype == torch.int32:
        code = N.F32  # 4-byte rows; the kernel moves bytes
    else:
        code = dcode(table)
    N.call("skb_gather_rows", n, table.shape[1], table.data_ptr(), table.stride(0),
           idx.data_ptr(), out.data_ptr(), out.stride(0), code, stream())
    _count()


def convert(src, dst):
    N.call("skb_convert", src.numel(), src.data_ptr(), dcode(src), dst.data_ptr(), dcode(dst),
           stream())
    _count()


def masked_maxpool(enc, lengths, out, B, L, d):
    N.call("skb_masked_maxpool", B, L, d, enc.data_ptr(), lengths.data_ptr(), out.data_ptr(),
           stream())
    _count()


def nvs_mask(logits, threshold, mask):
    B, V = logits.shape
    N.call("skb_nvs_mask", B, V, logits.data_ptr(), logits.stride(0), C.c_float(threshold),
           mask.data_ptr(), stream())
    _count()


def beam_step(logits, state: N.BeamState, lp_in=False):
    N.call("skb_beam_step", logits.data_ptr(), logits.stride(0), int(lp_in), C.byref(state),
           stream())
    _count()


def beam_reorder(anc, parent, step, R, S_max):
    N.call("skb_beam_reorder", R, S_max, anc.data_ptr(), parent.data_ptr(), step.data_ptr(),
           stream())
    _count(2)


def beam_finalize(state: N.BeamState, tokens_out, factors_out):
    N.call("skb_beam_finalize", C.byref(state), tokens_out.data_ptr(), factors_out.data_ptr(),
           stream())
    _count()
