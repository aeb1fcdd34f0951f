"""Model directory I/O (mirrors skiff checkpoint.py:1-353, vocab.py:33-78).

A model directory holds `config` (key = value, 12 keys), `params.bin` (SKP1:
magic, then per parameter u32 name length, UTF-8 name, u32 rank, u32
extents, float32 LE values) and vocab.{src,trg}[.factorN].json.  The loader
accepts exactly what the reference writes, with the same validation.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .config import NAME_RE, ModelConfig, SourceFactorSpec, TargetFactorSpec
from .errors import ConfigError, DataError

MAGIC = b"SKP1"
PARAMS_FILE = "params.bin"
CONFIG_FILE = "config"
CONFIG_KEYS = ["src_vocab_size", "trg_vocab_size", "d_model", "heads", "ff_dim",
               "encoder_layers", "decoder_layers", "decoder_kind", "source_factor_specs",
               "target_factor_specs", "nvs_enabled", "max_seq_len"]
SPECIALS = ["<pad>", "<unk>", "<s>", "</s>"]
FACTOR_SPECIALS = SPECIALS + ["<shift>"]
PAD_ID, UNK_ID, BOS_ID, EOS_ID, SHIFT_ID = 0, 1, 2, 3, 4


class Vocabulary:
    """Dense token<->id map with the pinned specials first (vocab.py:33-78)."""

    def __init__(self, tokens: list[str]):
        self._tokens = list(tokens)
        self._ids = {t: i for i, t in enumerate(self._tokens)}
        if len(self._ids) != len(self._tokens):
            raise DataError("vocabulary contains duplicate tokens")

    def __len__(self) -> int:
        return len(self._tokens)

    def __contains__(self, token: str) -> bool:
        return token in self._ids

    def to_id(self, token: str) -> int:
        return self._ids.get(token, UNK_ID)

    def to_token(self, idx: int) -> str:
        return self._tokens[idx]

    def encode(self, tokens) -> list[int]:
        return [self._ids.get(t, UNK_ID) for t in tokens]

    def decode(self, ids) -> list[str]:
        return [self._tokens[i] for i in ids]

    @property
    def tokens(self) -> list[str]:
        return list(self._tokens)

    def save(self, path) -> None:
        with open(path, "w", encoding="utf-8") as f:
            json.dump(self._tokens, f, ensure_ascii=False, indent=0)
            f.write("\n")

    @classmethod
    def load(cls, path) -> "Vocabulary":
        with open(path, encoding="utf-8") as f:
            tokens = json.load(f)
        if not isinstance(tokens, list) or not all(isinstance(t, str) for t in tokens):
            raise DataError(f"{path}: vocabulary file must hold a list of strings")
        if tokens[:4] != SPECIALS:
            raise DataError(f"{path}: first four entries must be {SPECIALS}")
        return cls(tokens)


def _atomic_write(path: Path, payload: bytes) -> None:
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name + ".")
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(payload)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def write_checkpoint(path, arrays: dict[str, np.ndarray]) -> None:
    chunks = [MAGIC]
    for name, arr in arrays.items():
        if not NAME_RE.match(name):
            raise ConfigError(f"bad parameter name {name!r}")
        a = np.ascontiguousarray(arr, dtype="<f4")
        raw = name.encode("utf-8")
        chunks.append(struct.pack("<I", len(raw)) + raw + struct.pack("<I", a.ndim)
                      + b"".join(struct.pack("<I", n) for n in a.shape))
        chunks.append(a.tobytes())
    _atomic_write(Path(path), b"".join(chunks))


def read_checkpoint(path) -> dict[str, np.ndarray]:
    """checkpoint.py:99-163 (float32 container)."""
    path = Path(path)
    buf = path.read_bytes()
    if buf[:4] != MAGIC:
        raise DataError(f"{path}: not a checkpoint file (bad magic)")
    off, out = 4, {}
    mv = memoryview(buf)

    def take(n):
        nonlocal off
        if off + n > len(buf):
            raise DataError(f"{path}: truncated checkpoint")
        s = mv[off:off + n]
        off += n
        return s

    while off < len(buf):
        (nlen,) = struct.unpack("<I", take(4))
        name = bytes(take(nlen)).decode("utf-8")
        if not NAME_RE.match(name):
            raise DataError(f"{path}: bad parameter name {name!r}")
        (rank,) = struct.unpack("<I", take(4))
        if rank > 8:
            raise DataError(f"{path}: parameter {name} has implausible rank {rank}")
        shape = struct.unpack(f"<{rank}I", take(4 * rank)) if rank else ()
        if name in out:
            raise DataError(f"{path}: duplicate parameter {name}")
        count = int(np.prod(shape, dtype=np.int64)) if shape else 1
        arr = np.frombuffer(take(4 * count), dtype="<f4").reshape(shape).astype(np.float32)
        if not np.isfinite(arr).all():
            raise DataError(f"{path}: parameter {name} holds non-finite values")
        out[name] = arr
    return out


def format_config(c: ModelConfig) -> str:
    vals = {
        "src_vocab_size": c.src_vocab_size, "trg_vocab_size": c.trg_vocab_size,
        "d_model": c.d_model, "heads": c.heads, "ff_dim": c.ff_dim,
        "encoder_layers": c.encoder_layers, "decoder_layers": c.decoder_layers,
        "decoder_kind": c.decoder_kind,
        "source_factor_specs": ",".join(f"{s.vocab_size}:{s.dim}:{s.combine}"
                                        for s in c.source_factor_specs),
        "target_factor_specs": ",".join(str(s.vocab_size) for s in c.target_factor_specs),
        "nvs_enabled": "true" if c.nvs_enabled else "false", "max_seq_len": c.max_seq_len,
    }
    return "".join(f"{k} = {vals[k]}\n" for k in CONFIG_KEYS)


def parse_config(text: str, origin: str = "config") -> ModelConfig:
    """checkpoint.py:223-275."""
    vals: dict[str, str] = {}
    for n, line in enumerate(text.splitlines(), 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise DataError(f"{origin}:{n}: expected 'key = value'")
        k, _, v = line.partition("=")
        k, v = k.strip(), v.strip()
        if k not in CONFIG_KEYS:
            raise DataError(f"{origin}:{n}: unknown key {k!r}")
        if k in vals:
            raise DataError(f"{origin}:{n}: duplicate key {k!r}")
        vals[k] = v
    missing = [k for k in CONFIG_KEYS if k not in vals]
    if missing:
        raise DataError(f"{origin}: missing keys {missing}")

    def ival(k):
        try:
            return int(vals[k])
        except ValueError:
            raise DataError(f"{origin}: key {k} is not an integer") from None

    src = []
    if vals["source_factor_specs"]:
        for item in vals["source_factor_specs"].split(","):
            f = item.split(":")
            if len(f) != 3 or f[2] not in ("sum", "concat"):
                raise DataError(f"{origin}: bad source factor spec {item!r}")
            src.append(SourceFactorSpec(int(f[0]), int(f[1]), f[2]))
    trg = [TargetFactorSpec(int(v)) for v in vals["target_factor_specs"].split(",")] \
        if vals["target_factor_specs"] else []
    if vals["nvs_enabled"] not in ("true", "false"):
        raise DataError(f"{origin}: nvs_enabled must be true or false")
    cfg = ModelConfig(ival("src_vocab_size"), ival("trg_vocab_size"), ival("d_model"),
                      ival("heads"), ival("ff_dim"), ival("encoder_layers"),
                      ival("decoder_layers"), vals["decoder_kind"], src, trg,
                      vals["nvs_enabled"] == "true", ival("max_seq_len"))
    cfg.validate()
    return cfg


@dataclass
class ModelDir:
    """checkpoint.py:305-313; duck-types as `vocabs` for translate()."""
    model: object
    src_vocab: Vocabulary
    trg_vocab: Vocabulary
    src_factor_vocabs: list
    trg_factor_vocabs: list
    path: Path


def save_model_dir(path, config: ModelConfig, params: dict[str, np.ndarray],
                   src_vocab: Vocabulary, trg_vocab: Vocabulary, src_factor_vocabs=(),
                   trg_factor_vocabs=()) -> None:
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    _atomic_write(path / CONFIG_FILE, format_config(config).encode("utf-8"))
    write_checkpoint(path / PARAMS_FILE, params)
    src_vocab.save(path / "vocab.src.json")
    trg_vocab.save(path / "vocab.trg.json")
    for i, v in enumerate(src_factor_vocabs):
        v.save(path / f"vocab.src.factor{i}.json")
    for i, v in enumerate(trg_factor_vocabs):
        v.save(path / f"vocab.trg.factor{i}.json")


def load_model_dir(path, params_file: str | None = None, precision: str = "bf16",
                   device: str = "cuda") -> ModelDir:
    """checkpoint.py:333-353: config + SKP1 weights + vocabularies, with the
    weights uploaded to the GPU in the requested precision ("bf16" tensor
    core GEMMs, or "fp32" parity mode)."""
    from .model import Model
    path = Path(path)
    if not path.is_dir():
        raise DataError(f"{path}: not a model directory")
    config = parse_config((path / CONFIG_FILE).read_text(encoding="utf-8"), str(path / CONFIG_FILE))
    arrays = read_checkpoint(path / (params_file or PARAMS_FILE))
    model = Model(config, params=arrays, precision=precision, device=device)
    src = Vocabulary.load(path / "vocab.src.json")
    trg = Vocabulary.load(path / "vocab.trg.json")
    sf = [Vocabulary.load(path / f"vocab.src.factor{i}.json")
          for i in range(len(config.source_factor_specs))]
    tf = [Vocabulary.load(path / f"vocab.trg.factor{i}.json")
          for i in range(len(config.target_factor_specs))]
    if len(src) != config.src_vocab_size or len(trg) != config.trg_vocab_size:
        raise DataError(f"{path}: vocabulary sizes disagree with the config")
    return ModelDir(model, src, trg, sf, tf, path)
