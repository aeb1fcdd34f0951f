"""Model configuration surface (mirrors skiff model.py:38-101, 182-265).

ModelConfig / SourceFactorSpec / TargetFactorSpec keep the reference's
field names, defaults and validation so a reference `config` file and
parameter set load unchanged.  `init_params` draws the same random-init
weights as the reference for a given seed (one default_rng stream in
parameter order), which is how synthetic benchmark models are built.
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

SELF_ATTENTION = "self_attention"
SSRU = "ssru"
NAME_RE = re.compile(r"^[a-z0-9_]+(\.[a-z0-9_]+)*$")


@dataclass(frozen=True)
class SourceFactorSpec:
    vocab_size: int
    dim: int
    combine: str = "sum"  # "sum" or "concat"


@dataclass(frozen=True)
class TargetFactorSpec:
    vocab_size: int


@dataclass
class ModelConfig:
    src_vocab_size: int
    trg_vocab_size: int
    d_model: int = 512
    heads: int = 8
    ff_dim: int = 2048
    encoder_layers: int = 6
    decoder_layers: int = 6
    decoder_kind: str = SELF_ATTENTION
    source_factor_specs: list[SourceFactorSpec] = field(default_factory=list)
    target_factor_specs: list[TargetFactorSpec] = field(default_factory=list)
    nvs_enabled: bool = False
    max_seq_len: int = 128

    @property
    def surface_embed_dim(self) -> int:
        return self.d_model - sum(s.dim for s in self.source_factor_specs if s.combine == "concat")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.heads

    def validate(self) -> None:
        """model.py:71-101."""
        if self.d_model <= 0 or self.ff_dim <= 0:
            raise ConfigError("d_model and ff_dim must be positive")
        if self.heads <= 0 or self.d_model % self.heads != 0:
            raise ConfigError(f"d_model {self.d_model} must be divisible by heads {self.heads}")
        if self.encoder_layers < 0 or self.decoder_layers < 0:
            raise ConfigError("layer counts must be non-negative")
        if self.decoder_kind not in (SELF_ATTENTION, SSRU):
            raise ConfigError(f"unknown decoder kind {self.decoder_kind!r}")
        if self.src_vocab_size < 4 or self.trg_vocab_size < 4:
            raise ConfigError("vocabularies must at least hold the special ids")
        if self.max_seq_len < 1:
            raise ConfigError("max_seq_len must be at least 1")
        for i, spec in enumerate(self.source_factor_specs):
            if spec.combine not in ("sum", "concat"):
                raise ConfigError(f"source factor {i}: unknown combine {spec.combine!r}")
            if spec.combine == "sum" and spec.dim != self.d_model:
                raise ConfigError(f"source factor {i}: sum-combined dim {spec.dim} must equal "
                                  f"d_model {self.d_model}")
            if spec.vocab_size < 4:
                raise ConfigError(f"source factor {i}: vocabulary too small")
        if self.surface_embed_dim < 1:
            raise ConfigError("concat factor dims leave no room for the surface embedding")
        for i, spec in enumerate(self.target_factor_specs):
            if spec.vocab_size <= 4:
                raise ConfigError(f"target factor {i}: vocabulary must hold the shift id")


def param_shapes(config: ModelConfig) -> dict[str, tuple[str, tuple[int, ...]]]:
    """Ordered name -> (init kind, shape), the reference's draw order
    (model.py:182-241)."""
    config.validate()
    d, ff = config.d_model, config.ff_dim
    out: dict[str, tuple[str, tuple[int, ...]]] = {}

    def norm(p):
        out[p + ".gain"] = ("one", (d,))
        out[p + ".bias"] = ("zero", (d,))

    def attn(p):
        for w in ("wq", "wk", "wv", "wo"):
            out[f"{p}.{w}"] = ("mat", (d, d))

    def ffn(p):
        out[p + ".w1"] = ("mat", (ff, d))
        out[p + ".b1"] = ("zero", (ff,))
        out[p + ".w2"] = ("mat", (d, ff))
        out[p + ".b2"] = ("zero", (d,))

    out["embed.src.surface"] = ("emb", (config.src_vocab_size, config.surface_embed_dim))
    for i, s in enumerate(config.source_factor_specs):
        out[f"embed.src.factor{i}"] = ("emb", (s.vocab_size, s.dim))
    out["embed.trg.surface"] = ("emb", (config.trg_vocab_size, d))
    for i, s in enumerate(config.target_factor_specs):
        out[f"embed.trg.factor{i}"] = ("emb", (s.vocab_size, d))
    for i in range(config.encoder_layers):
        p = f"encoder.layer{i}"
        attn(p + ".self_attn"); norm(p + ".self_attn_norm")
        ffn(p + ".ffn"); norm(p + ".ffn_norm")
    for i in range(config.decoder_layers):
        p = f"decoder.layer{i}"
        if config.decoder_kind == SSRU:
            out[p + ".ssru.wf"] = ("mat", (d, d))
            out[p + ".ssru.bf"] = ("zero", (d,))
            out[p + ".ssru.w"] = ("mat", (d, d))
            norm(p + ".ssru_norm")
        else:
            attn(p + ".self_attn"); norm(p + ".self_attn_norm")
        attn(p + ".cross_attn"); norm(p + ".cross_attn_norm")
        ffn(p + ".ffn"); norm(p + ".ffn_norm")
    norm("decoder.final_norm")
    for i, s in enumerate(config.target_factor_specs):
        out[f"output.factor{i}.w"] = ("mat", (s.vocab_size, d))
        out[f"output.factor{i}.b"] = ("zero", (s.vocab_size,))
    if config.nvs_enabled:
        out["nvs.w"] = ("mat", (config.trg_vocab_size, d))
        out["nvs.b"] = ("zero", (config.trg_vocab_size,))
    return out


def init_params(config: ModelConfig, seed: int = 13) -> dict[str, np.ndarray]:
    """Random-init weights identical to model.py:244-265 for the same seed."""
    rng = np.random.default_rng(seed)
    params: dict[str, np.ndarray] = {}
    for name, (kind, shape) in param_shapes(config).items():
        if kind == "mat":
            limit = math.sqrt(6.0 / (shape[0] + shape[1]))
            arr = rng.uniform(-limit, limit, size=shape)
        elif kind == "emb":
            arr = rng.normal(0.0, 0.3 / math.sqrt(shape[1]), size=shape)
        elif kind == "one":
            arr = np.ones(shape)
        else:
            arr = np.zeros(shape)
        params[name] = np.asarray(arr, dtype=np.float32)
    return params


def check_params(config: ModelConfig, params: dict[str, np.ndarray]) -> None:
    """model.py:352-366: names and shapes must match the config exactly."""
    expected = param_shapes(config)
    have, want = set(params), set(expected)
    if have != want:
        raise ConfigError(f"parameters do not match config (missing {sorted(want - have)[:4]}, "
                          f"extra {sorted(have - want)[:4]})")
    for name, (_, shape) in expected.items():
        if tuple(params[name].shape) != shape:
            raise ConfigError(f"parameter {name}: shape {tuple(params[name].shape)}, "
                              f"config wants {shape}")


# ------------------------------------------------------------ cost model
def decoder_step_cost(config: ModelConfig, step: int, src_len: int, out_cols: int | None = None) -> int:
    """MACs of one decode step per row (model.py:590-606); out_cols replaces
    the vocabulary width under a restriction."""
    d, ff = config.d_model, config.ff_dim
    inner = 2 * d * d if config.decoder_kind == SSRU else 4 * d * d + 2 * (step + 1) * d
    cross = 2 * d * d + 2 * src_len * d
    v = config.trg_vocab_size if out_cols is None else out_cols
    return (config.decoder_layers * (inner + cross + 2 * d * ff) + d * v
            + sum(d * s.vocab_size for s in config.target_factor_specs))


def encoder_cost(config: ModelConfig, src_len: int) -> int:
    """model.py:609-613."""
    d, ff = config.d_model, config.ff_dim
    return config.encoder_layers * (4 * src_len * d * d + 2 * src_len * src_len * d
                                    + 2 * src_len * d * ff)


def translation_cost(config: ModelConfig, src_len: int, out_len: int) -> int:
    """model.py:616-621."""
    cross_kv = config.decoder_layers * 2 * src_len * config.d_model * config.d_model
    return encoder_cost(config, src_len) + cross_kv + sum(
        decoder_step_cost(config, t, src_len) for t in range(out_len))
