"""Host-side logic of the drop-in surface (CPU only): input parsing,
chunking, config/checkpoint/vocab/shortlist I/O, init, cost model —
checked against the reference's recorded behaviour (tests/golden)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN
from fixture_models import oracle_model, product_config
from oracle.fixture_configs import CONFIGS


def test_parse_input_lines_match_reference():
    from paper_2207_05851_b200.errors import InputError
    from paper_2207_05851_b200.search import parse_input_line
    g = json.loads((GOLDEN / "search.json").read_text())
    lines = ['a b   c', '{"text": "a b", "source_prefix": "<t>", "target_prefix": "x y", '
             '"target_prefix_factors": ["O O B"], "source_factors": ["P Q"]}',
             '{"text": "a", "extra": 1}', '{bad json', '{"text": 3}']
    for ln, want in zip(lines, g["parsed"]):
        if want["ok"]:
            s = parse_input_line(ln)
            assert s.tokens == want["tokens"] and s.source_factors == want["source_factors"]
            assert s.source_prefix == want["source_prefix"]
            assert s.target_prefix == want["target_prefix"]
            assert s.target_prefix_factors == want["target_prefix_factors"]
        else:
            with pytest.raises(InputError):
                parse_input_line(ln)


def test_chunking_matches_reference():
    from paper_2207_05851_b200.search import SentenceInput, chunk_input
    g = json.loads((GOLDEN / "search.json").read_text())
    got = [[c.tokens for c in chunk_input(SentenceInput(tokens=list("abcdefghij"),
                                                        source_prefix=["<p>"]), 4)]]
    assert got == g["chunks"]


@pytest.mark.parametrize("name", list(CONFIGS))
def test_product_init_equals_reference_init(name):
    from paper_2207_05851_b200.config import init_params
    ref = json.loads((GOLDEN / "params.json").read_text())[name]
    p = init_params(product_config(name), CONFIGS[name]["seed"])
    assert set(p) == set(ref)
    for n, (s, a, first, last) in ref.items():
        assert p[n].astype(np.float64).sum() == s and float(p[n].ravel()[0]) == first


def test_model_dir_round_trip(tmp_path):
    from paper_2207_05851_b200.checkpoint import (Vocabulary, format_config, parse_config,
                                                  read_checkpoint, write_checkpoint)
    cfg = product_config("srcfac")
    assert parse_config(format_config(cfg)) == cfg
    params = oracle_model("srcfac").p
    write_checkpoint(tmp_path / "p.bin", params)
    back = read_checkpoint(tmp_path / "p.bin")
    assert set(back) == set(params)
    assert all(np.array_equal(back[n], params[n]) for n in params)
    v = Vocabulary(["<pad>", "<unk>", "<s>", "</s>", "a", "b"])
    v.save(tmp_path / "v.json")
    assert Vocabulary.load(tmp_path / "v.json").tokens == v.tokens
    assert v.encode(["a", "zz"]) == [4, 1]


def test_bad_checkpoints_are_data_errors(tmp_path):
    from paper_2207_05851_b200.checkpoint import read_checkpoint, write_checkpoint
    from paper_2207_05851_b200.errors import DataError
    (tmp_path / "bad").write_bytes(b"XXXX")
    with pytest.raises(DataError):
        read_checkpoint(tmp_path / "bad")
    write_checkpoint(tmp_path / "nan", {"a.b": np.array([np.nan], dtype=np.float32)})
    with pytest.raises(DataError):
        read_checkpoint(tmp_path / "nan")
    write_checkpoint(tmp_path / "ok", {"a.b": np.ones(4, dtype=np.float32)})
    raw = (tmp_path / "ok").read_bytes()
    (tmp_path / "trunc").write_bytes(raw[:-3])
    with pytest.raises(DataError):
        read_checkpoint(tmp_path / "trunc")


def test_shortlist_file(tmp_path):
    from paper_2207_05851_b200.checkpoint import Vocabulary
    from paper_2207_05851_b200.shortlist import Shortlist
    (tmp_path / "sl").write_text("a\tx:0.5 y:0.25\nb\ty:1\nq\tx:1\n")
    sv = Vocabulary(["<pad>", "<unk>", "<s>", "</s>", "a", "b"])
    tv = Vocabulary(["<pad>", "<unk>", "<s>", "</s>", "x", "y"])
    sl = Shortlist.from_file(tmp_path / "sl", sv, tv)
    assert sl.lookup([4]).tolist() == [4, 5] and sl.lookup([5, 5]).tolist() == [5]
    assert sl.lookup([0]).size == 0


def test_cost_model_matches_survey_numbers():
    """big 6-6 beam 5 at L=30 = 89.49 GFLOP/sentence."""
    from paper_2207_05851_b200.config import ModelConfig
    from oracle.skiff_oracle import sentence_flops
    big = ModelConfig(32000, 32000, 1024, 16, 4096, 6, 6)
    rows = [1] + [5] * 69
    assert abs(sentence_flops(big, 30, rows) / 1e9 - 89.49) < 0.05


def test_config_validation():
    from paper_2207_05851_b200.config import ModelConfig, SourceFactorSpec
    from paper_2207_05851_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        ModelConfig(11, 13, d_model=10, heads=4).validate()
    with pytest.raises(ConfigError):
        ModelConfig(11, 13, d_model=16, heads=4,
                    source_factor_specs=[SourceFactorSpec(6, 8, "sum")]).validate()


def test_bench_shortlist_generator_matches_fixture_generator():
    """bench.py builds the top-200 shortlist of the SSRU config on its own
    (the product leg may not import oracle/); it must be the fixtures' one."""
    import numpy as np
    import bench
    from oracle.fixture_configs import synthetic_shortlist_rows
    a = bench.synthetic_shortlist_rows(300, 20)
    b = synthetic_shortlist_rows(300, 20)
    assert a.keys() == b.keys() and all(np.array_equal(a[k], b[k]) for k in a)


def test_bench_distinct_kv_entries_counts_shared_prefix():
    """distinct_kv_entries walks the beam back-pointers: two rows of one
    sentence that share their whole history read t + 2 distinct entries at
    step t (the shared prefix once, plus their own newest entry each)."""
    import types
    import torch
    import bench
    K, B, S = 2, 1, 4
    par = torch.zeros(S * K, dtype=torch.int32)  # every new row's parent is row 0
    bb = types.SimpleNamespace(K=K, B=B, ws=types.SimpleNamespace(par_hist=par))
    got = bench.distinct_kv_entries(bb, S)
    # step 0: one row; step t >= 1: 2 rows at position t, row 0 at positions < t
    assert got == [1, 3, 4, 5]


REFDIRS = ["srcfac", "ssru", "factored"]


@pytest.mark.parametrize("name", REFDIRS)
def test_reads_model_dirs_written_by_the_reference(name):
    """tests/golden/refdir_<cfg> was written by skiff's own save_model_dir
    (checkpoint.py:316-330; oracle/make_golden.py modeldirs): the product's
    readers take its config, SKP1 parameters and vocabularies unchanged."""
    import numpy as np
    from conftest import GOLDEN
    from fixture_models import oracle_model, oracle_vocabs, product_config
    from paper_2207_05851_b200.checkpoint import Vocabulary, parse_config, read_checkpoint
    d = GOLDEN / f"refdir_{name}"
    cfg = parse_config((d / "config").read_text(), str(d / "config"))
    assert cfg == product_config(name)
    params = read_checkpoint(d / "params.bin")
    want = oracle_model(name).p
    assert params.keys() == want.keys()
    for k in want:
        assert params[k].dtype == np.float32 and np.array_equal(params[k], want[k]), k
    ov = oracle_vocabs(name)
    assert Vocabulary.load(d / "vocab.src.json").tokens == ov["src"].tokens
    assert Vocabulary.load(d / "vocab.trg.json").tokens == ov["trg"].tokens
    for i, v in enumerate(ov["src_f"]):
        assert Vocabulary.load(d / f"vocab.src.factor{i}.json").tokens == v.tokens
    for i, v in enumerate(ov["trg_f"]):
        assert Vocabulary.load(d / f"vocab.trg.factor{i}.json").tokens == v.tokens


def test_sorted_union_equals_numpy_unique():
    """The shortlist / restriction union (bitmap) is np.unique of the
    concatenation: sorted, unique, int64, for any mix of inputs."""
    import numpy as np
    from paper_2207_05851_b200.shortlist import sorted_union
    rng = np.random.default_rng(3)
    for _ in range(50):
        parts = [rng.integers(0, int(rng.integers(1, 40000)), size=int(rng.integers(0, 300)))
                 for _ in range(int(rng.integers(1, 6)))]
        want = np.unique(np.concatenate(parts)).astype(np.int64)
        got = sorted_union(*parts)
        assert got.dtype == np.int64 and np.array_equal(got, want)
    assert sorted_union(np.array([-3, 2, 2])).tolist() == [-3, 2]  # fallback path
    assert sorted_union(np.zeros(0, dtype=np.int64)).size == 0
    assert sorted_union([7, 1], np.array([1, 4])).tolist() == [1, 4, 7]
