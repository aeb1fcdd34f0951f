"""The C-ABI library loads without a GPU and exports every entry point
declared in include/skiff_b200.h (no compute calls here)."""

import ctypes
import re

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "skiff_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(skb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_hot_path():
    names = _declared()
    for must in ("skb_gemm", "skb_layernorm", "skb_self_attention_step",
                 "skb_cross_attention_step", "skb_encoder_attention", "skb_beam_step",
                 "skb_beam_reorder", "skb_beam_finalize"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2207_05851_b200 import build
    lib_path = build.LIB
    if not lib_path.exists():
        build.build()
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    from paper_2207_05851_b200 import _native as N
    assert set(N.SIGNATURES) == set(_declared())


def test_version_and_error_strings_without_gpu():
    from paper_2207_05851_b200 import _native as N
    assert b"sm_100a" in N.lib().skb_version()
    assert isinstance(N.lib().skb_last_error(), bytes)
