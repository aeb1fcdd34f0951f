"""Lexical shortlist file format and id-space lookup (mirrors skiff
shortlist.py:134-207).  The offline IBM-Model-1 training of the reference is
out of scope; this module reads its output.

File format: one line per source token, `source<TAB>target:prob ...`.
"""

from __future__ import annotations

import logging
from pathlib import Path

import numpy as np

from .errors import DataError

logger = logging.getLogger(__name__)


def read_shortlist_file(path) -> dict[str, list[tuple[str, float]]]:
    """shortlist.py:153-175."""
    out: dict[str, list[tuple[str, float]]] = {}
    with open(path, encoding="utf-8") as f:
        for n, line in enumerate(f, 1):
            line = line.rstrip("\n")
            if not line:
                continue
            if "\t" not in line:
                raise DataError(f"{path}:{n}: expected 'source<TAB>entries'")
            tok, _, rest = line.partition("\t")
            if tok in out:
                raise DataError(f"{path}:{n}: duplicate source token {tok!r}")
            entries = []
            for item in rest.split(" ") if rest else []:
                trg, sep, prob = item.rpartition(":")
                if not sep or not trg:
                    raise DataError(f"{path}:{n}: bad entry {item!r}")
                try:
                    entries.append((trg, float(prob)))
                except ValueError:
                    raise DataError(f"{path}:{n}: bad probability in {item!r}") from None
            out[tok] = entries
    return out


def write_shortlist_file(path, rows: dict[str, list[tuple[str, float]]]) -> None:
    with open(path, "w", encoding="utf-8") as f:
        for tok, entries in rows.items():
            f.write(tok + "\t" + " ".join(f"{t}:{p:.6g}" for t, p in entries) + "\n")


class Shortlist:
    """Id-space shortlist for one vocabulary pair (shortlist.py:178-207)."""

    def __init__(self, rows: dict[int, np.ndarray]):
        self.rows = rows

    @classmethod
    def from_file(cls, path, src_vocab, trg_vocab) -> "Shortlist":
        raw = read_shortlist_file(path)
        rows: dict[int, np.ndarray] = {}
        dropped = 0
        for tok, entries in raw.items():
            if tok not in src_vocab:
                dropped += 1
                continue
            ids = [trg_vocab.to_id(t) for t, _ in entries if t in trg_vocab]
            rows[src_vocab.to_id(tok)] = np.asarray(sorted(set(ids)), dtype=np.int64)
        if dropped:
            logger.info("shortlist: dropped %d source tokens unknown to the model", dropped)
        return cls(rows)

    def lookup(self, src_ids) -> np.ndarray:
        """Union of the rows for the given source ids."""
        parts = [self.rows[i] for i in set(int(i) for i in src_ids) if i in self.rows]
        if not parts:
            return np.empty(0, dtype=np.int64)
        return np.unique(np.concatenate(parts))
