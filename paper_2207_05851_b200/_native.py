"""ctypes binding of lib/libskiff_b200.so (the C ABI in include/skiff_b200.h).

There is no CPU fallback: if the library is missing or the device is not a
B200 (sm_100a), the first call raises.  Status codes map onto the
reference's error hierarchy (errors.py:10-39).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import ConfigError, NumericError, ShapeError

import os

# SKB_LIB: alternative build of the same library (A/B experiments)
LIB_PATH = Path(os.environ.get("SKB_LIB") or
                Path(__file__).resolve().parent / "lib" / "libskiff_b200.so")

SKB_OK, SKB_ERR_SHAPE, SKB_ERR_CONFIG, SKB_ERR_LAUNCH, SKB_ERR_NUMERIC, SKB_ERR_UNSUPPORTED = range(6)
F32, BF16 = 0, 1
EPI_STORE, EPI_RELU, EPI_RESID, EPI_SSRU, EPI_LOGITS = 0, 1, 2, 3, 4

vp = C.c_void_p
i32 = C.c_int


class Epilogue(C.Structure):
    _fields_ = [("kind", i32), ("bias", vp), ("out", vp), ("ldo", i32), ("out_dtype", i32),
                ("c_prev", vp), ("c_next", vp), ("src_row", vp), ("ld_state", i32),
                ("step", vp), ("state_stride", C.c_longlong), ("lse_part", vp),
                ("lse_ld", i32), ("mask", vp), ("mask_words", i32), ("rows_per_group", i32),
                ("splitk_ws", vp), ("splitk_ws_elems", C.c_longlong), ("splitk_counters", vp),
                ("splitk_counters_n", i32), ("ln_gain", vp), ("ln_bias", vp),
                ("ln_eps", C.c_float), ("ln_out", vp), ("ln_ldo", i32), ("ln_counter", vp),
                ("ln_in", vp), ("ln_in_ld", i32), ("ln_in_gain", vp), ("ln_in_bias", vp),
                ("ln_in_eps", C.c_float), ("streams", i32), ("k_split", i32)]


class BeamState(C.Structure):
    _fields_ = [("B", i32), ("K", i32), ("U", i32), ("S_max", i32), ("n_factors", i32),
                ("len_pen", vp), ("step", vp), ("col_token", vp), ("mask", vp),
                ("eos_col", i32), ("max_len", vp), ("prefix_len", vp), ("prefix_col", vp),
                ("P", i32), ("prefix_fac", vp), ("n_alive", vp), ("done", vp), ("score", vp),
                ("tok_next", vp), ("ftok_next", vp), ("parent", vp),
                ("tok_hist", vp), ("par_hist", vp), ("fac_hist", vp), ("fac_logits", vp),
                ("fac_ld", i32), ("fac_off", vp), ("lse_part", vp), ("lse_ld", i32), ("prune", i32),
                ("stage_partials", i32),
                ("cand_score", vp), ("cand_lp", vp),
                ("cand_col", vp), ("cand_cnt", vp), ("row_argmax", vp), ("fac_choice", vp),
                ("counter", vp), ("best_norm", vp), ("best_logprob", vp), ("best_steps", vp),
                ("best_forced", vp), ("best_parent", vp), ("best_fac", vp), ("n_done", vp)]


# (name, argtypes) — must match include/skiff_b200.h
SIGNATURES = {
    "skb_version": [],
    "skb_last_error": [],
    "skb_tc_available": [],
    "skb_last_launches": [],
    "skb_gemm": [i32, i32, i32, i32, vp, i32, vp, i32, C.POINTER(Epilogue), vp],
    "skb_gemm_simt": [i32, i32, i32, i32, vp, i32, vp, i32, C.POINTER(Epilogue), vp],
    "skb_gemm_force": [i32, i32, i32],
    "skb_gemm_force_sw": [i32, i32, i32],
    "skb_attn_force_heads": [i32],
    "skb_gemm_force_pc": [i32, i32, i32],
    "skb_quantize_rows": [i32, i32, vp, i32, vp, i32, vp, vp],
    "skb_causal_self_attention": [i32, i32, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp],
    "skb_ssru_scan": [i32, i32, i32, vp, i32, vp, vp, i32, vp],
    "skb_gemm_i8": [i32, i32, i32, vp, i32, vp, vp, i32, vp, C.POINTER(Epilogue), vp],
    "skb_layernorm": [i32, i32, vp, i32, vp, vp, C.c_float, vp, i32, i32, vp],
    "skb_embed_target": [i32, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp],
    "skb_embed_source": [i32, i32, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp],
    "skb_encoder_attention": [i32, i32, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp],
    "skb_attn_plan_bytes": [i32, i32, i32],
    "skb_attn_plan": [i32, i32, i32, vp, vp, vp, vp],
    "skb_self_attention_step_planned": [i32, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp, vp, i32,
                                        vp, i32, i32, vp],
    "skb_self_attention_step": [i32, i32, i32, vp, i32, i32, vp, vp, i32, i32, vp, vp, i32, vp,
                                i32, i32, vp],
    "skb_cross_attention_step": [i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, i32, i32, vp,
                                 vp, i32, vp, i32, i32, vp],
    "skb_gather_rows": [i32, i32, vp, i32, vp, vp, i32, i32, vp],
    "skb_beam_step": [vp, i32, i32, C.POINTER(BeamState), vp],
    "skb_beam_reorder": [i32, i32, vp, vp, vp, vp],
    "skb_beam_finalize": [C.POINTER(BeamState), vp, vp, vp],
    "skb_masked_maxpool": [i32, i32, i32, vp, vp, vp, vp],
    "skb_convert": [C.c_longlong, vp, i32, vp, i32, vp],
    "skb_nvs_mask": [i32, i32, vp, i32, C.c_float, vp, vp],
    "skb_set_device": [i32],
    "skb_debug_beam_prof": [vp],
    "skb_debug_gemm_trace": [vp],
    "skb_debug_attn_trace": [vp],
}

_lib = None


def lib():
    """Load the library once; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2207_05851_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                continue  # reported as missing by tests/test_native_lib.py
            fn.argtypes = args
            fn.restype = (C.c_char_p if name in ("skb_version", "skb_last_error")
                          else C.c_size_t if name == "skb_attn_plan_bytes" else C.c_int)
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == SKB_OK:
        return
    msg = lib().skb_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == SKB_ERR_SHAPE:
        raise ShapeError(text)
    if rc == SKB_ERR_CONFIG:
        raise ConfigError(text)
    if rc == SKB_ERR_NUMERIC:
        raise NumericError(text)
    raise RuntimeError(f"CUDA kernel failure ({rc}) {text}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
