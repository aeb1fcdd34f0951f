"""Build the golden-fixture models/vocabularies for the oracle (tests only)."""

from functools import lru_cache

from oracle import skiff_oracle as O
from oracle.fixture_configs import CONFIGS, make_words


@lru_cache(maxsize=None)
def oracle_model(name: str) -> O.OracleModel:
    spec = CONFIGS[name]
    cfg = O.OConfig(**spec["config"])
    return O.OracleModel(cfg, O.init_params(cfg, spec["seed"]))


def oracle_vocabs(name: str) -> dict:
    cfg = CONFIGS[name]["config"]
    specials = ["<pad>", "<unk>", "<s>", "</s>"]
    return dict(
        src=O.OVocab(specials + make_words(cfg["src_vocab_size"] - 4)),
        trg=O.OVocab(specials + make_words(cfg["trg_vocab_size"] - 4)),
        src_f=[O.OVocab(specials + [f"s{i}_{j}" for j in range(v - 4)])
               for i, (v, _, _) in enumerate(cfg.get("source_factor_specs", []))],
        trg_f=[O.OVocab(specials + ["<shift>"] + [f"F{i}_{j}" for j in range(v - 5)])
               for i, v in enumerate(cfg.get("target_factor_specs", []))],
    )


def product_config(name: str, **override):
    from paper_2207_05851_b200.config import ModelConfig, SourceFactorSpec, TargetFactorSpec
    cfg = dict(CONFIGS[name]["config"])
    cfg.update(override)
    cfg["source_factor_specs"] = [SourceFactorSpec(*s) for s in cfg.get("source_factor_specs", [])]
    cfg["target_factor_specs"] = [TargetFactorSpec(v) for v in cfg.get("target_factor_specs", [])]
    return ModelConfig(**cfg)


_PM = {}


def product_model(name: str, precision: str = "fp32", **override):
    """The product's device Model with the fixture's random-init weights."""
    from paper_2207_05851_b200.model import Model
    key = (name, precision, tuple(sorted(override.items())))
    if key not in _PM:
        _PM[key] = Model(product_config(name, **override), params=oracle_model(name).p,
                         precision=precision)
    return _PM[key]


def product_vocabs(name: str):
    from types import SimpleNamespace

    from paper_2207_05851_b200.checkpoint import Vocabulary
    ov = oracle_vocabs(name)
    return SimpleNamespace(src_vocab=Vocabulary(ov["src"].tokens),
                           trg_vocab=Vocabulary(ov["trg"].tokens),
                           src_factor_vocabs=[Vocabulary(v.tokens) for v in ov["src_f"]],
                           trg_factor_vocabs=[Vocabulary(v.tokens) for v in ov["trg_f"]])
