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
