"""Dynamic INT8 feed-forward layers on the device (skiff quant.py).

The reference quantizes every feed-forward weight per output row offline
(scale = max|row| / 127, round half away from zero) and every activation
row on the fly with the same rule, multiplies in exact int32 and rescales
in float32: out = (float32(acc) * a_scale) * w_scale (+ bias)
(quant.py:40-53, 99-132).  Here the row quantization is one kernel
(skb_quantize_rows) and the product a tcgen05 kind::i8 GEMM whose epilogue
applies the rescale, bias, ReLU or residual add (skb_gemm_i8); the integers
are exact, so the layer's output equals the reference's bit for bit given
the same float32 input rows.  Everything else stays in the model's
precision.

`quantize_model(model)` swaps every encoder and decoder feed-forward layer
to this path (quant.py:140-145) and returns the swapped parameter names.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kern
from . import _native as N
from .errors import ConfigError, ShapeError

FFN_WEIGHT_SUFFIXES = (".ffn.w1", ".ffn.w2")
_MAX_INNER = (2 ** 31) // (127 * 127)  # int32 accumulation stays exact


class QuantizedLinear:
    """Device int8 weight [out, in] with per-row fp32 scales."""

    def __init__(self, q: torch.Tensor, scales: torch.Tensor):
        if q.dim() != 2 or q.dtype != torch.int8 or scales.shape != (q.shape[0],):
            raise ShapeError("QuantizedLinear needs int8 (out, in) values and per-row scales")
        self.q = q.contiguous()
        self.scales = scales.contiguous()

    @classmethod
    def from_weights(cls, w, device) -> "QuantizedLinear":
        w = np.asarray(w, dtype=np.float32)
        if w.ndim != 2:
            raise ShapeError(f"quantize_rows needs a matrix, got shape {w.shape}")
        if w.shape[1] > _MAX_INNER:
            raise ConfigError(f"inner extent {w.shape[1]} would overflow int32 accumulation")
        if w.shape[1] % 16:
            raise ConfigError(f"int8 GEMM needs the inner extent to be a multiple of 16, got {w.shape[1]}")
        if not np.isfinite(w).all():
            raise ShapeError("quantize_rows: non-finite weights")
        wd = torch.as_tensor(np.ascontiguousarray(w), device=device)
        q = torch.empty(w.shape, dtype=torch.int8, device=device)
        s = torch.empty(w.shape[0], dtype=torch.float32, device=device)
        quantize_rows(wd, q, s)
        return cls(q, s)

    @property
    def shape(self):
        return tuple(self.q.shape)


def quantize_rows(x: torch.Tensor, q: torch.Tensor, scales: torch.Tensor, rows=None) -> None:
    """Per-row symmetric int8 quantization of fp32 rows (quant.py:40-53)."""
    kern.quantize_rows(x, q, scales, rows)


class Int8Scratch:
    """Stable device buffers of the int8 feed-forward path for up to `rows`
    rows (captured into the decode-step graphs)."""

    def __init__(self, rows: int, d: int, ff: int, device):
        self.h = torch.zeros(rows, d, device=device)                      # LN(x), fp32
        self.qa = torch.zeros(rows, d, dtype=torch.int8, device=device)
        self.sa = torch.ones(rows, device=device)
        self.f = torch.zeros(rows, ff, device=device)                     # relu(FFN1), fp32
        self.qf = torch.zeros(rows, ff, dtype=torch.int8, device=device)
        self.sf = torch.ones(rows, device=device)


def ffn_int8(Ly, x: torch.Tensor, scratch: Int8Scratch, rows: int, eps: float = 1e-5) -> None:
    """x += FFN(LN(x)) on the int8 path (model.py:432-438 with the
    quantized hook): LN in fp32, quantize, int8 FFN1 (+b1, ReLU) in fp32,
    quantize, int8 FFN2 (+b2) added to the residual stream."""
    s = scratch
    kern.layernorm(x, *Ly.ln_ffn, s.h, rows=rows, eps=eps)
    kern.quantize_rows(s.h, s.qa, s.sa, rows)
    kern.gemm_i8(s.qa, s.sa, Ly.q1.q, Ly.q1.scales, s.f, N.EPI_RELU, Ly.b1, M=rows)
    kern.quantize_rows(s.f, s.qf, s.sf, rows)
    kern.gemm_i8(s.qf, s.sf, Ly.q2.q, Ly.q2.scales, x, N.EPI_RESID, Ly.b2, M=rows)


def quantized_param_names(model) -> list[str]:
    return [n for n in model.params if n.endswith(FFN_WEIGHT_SUFFIXES)]


def quantize_model(model) -> list[str]:
    """Swap every feed-forward linear to the int8 path (quant.py:140-145).
    Returns the swapped parameter names in parameter order."""
    names = quantized_param_names(model)
    layers = {f"encoder.layer{i}": Ly for i, Ly in enumerate(model.enc)}
    layers.update({f"decoder.layer{i}": Ly for i, Ly in enumerate(model.dec)})
    for name in names:
        base, _, which = name.rpartition(".ffn.")
        ql = QuantizedLinear.from_weights(model.params[name], model.device)
        setattr(layers[base], "q1" if which == "w1" else "q2", ql)
        model.quantized[name] = ql
    # workspaces built before the swap have no int8 scratch
    from .engine import _WS_CACHE
    _WS_CACHE.pop(model, None)
    return names
