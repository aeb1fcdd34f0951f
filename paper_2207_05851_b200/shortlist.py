"""Lexical shortlists: the on-disk table the reference's offline trainer
writes, and the per-sentence id-space union the search restricts to
(behaviour of skiff shortlist.py:153-207; its IBM-Model-1 trainer is out of
scope for this backend).

On disk, each non-empty line maps one source token to its candidate target
tokens:  ``<source token> TAB <target>:<prob> <target>:<prob> ...``.
A target token may itself contain ':' (the probability follows the last
one).  Malformed lines raise DataError naming the file and line.
"""

from __future__ import annotations

import logging
from pathlib import Path

import numpy as np

from .errors import DataError

log = logging.getLogger(__name__)

Entries = list[tuple[str, float]]


def _entry(where: str, field: str) -> tuple[str, float]:
    token, colon, prob = field.rpartition(":")
    if not (colon and token):
        raise DataError(f"{where}: malformed shortlist entry {field!r}")
    try:
        return token, float(prob)
    except ValueError:
        raise DataError(f"{where}: entry {field!r} has a non-numeric probability") from None


def read_shortlist_file(path) -> dict[str, Entries]:
    """Parse a shortlist file into {source token: [(target token, prob)]}
    in file order; a source token may appear on one line only."""
    table: dict[str, Entries] = {}
    text = Path(path).read_text(encoding="utf-8")
    for number, line in enumerate(text.split("\n"), 1):
        if not line:
            continue
        where = f"{path}:{number}"
        source, tab, rest = line.partition("\t")
        if not tab:
            raise DataError(f"{where}: a shortlist line is 'source<TAB>entries'")
        if source in table:
            raise DataError(f"{where}: source token {source!r} appears twice")
        table[source] = [_entry(where, f) for f in rest.split(" ")] if rest else []
    return table


def write_shortlist_file(path, rows: dict[str, Entries]) -> None:
    """Inverse of read_shortlist_file (test fixtures)."""
    body = "".join(f"{src}\t{' '.join(f'{t}:{p:.6g}' for t, p in ents)}\n"
                   for src, ents in rows.items())
    Path(path).write_text(body, encoding="utf-8")


class Shortlist:
    """Candidate target ids per source id, for one (source, target)
    vocabulary pair: rows[src_id] is a sorted unique int64 array."""

    def __init__(self, rows: dict[int, np.ndarray]):
        self.rows = rows

    @classmethod
    def from_file(cls, path, src_vocab, trg_vocab) -> "Shortlist":
        """Map a shortlist file into the model's id space.  Source lines whose
        token the model does not know are skipped (the file may have been
        built on another corpus), as are unknown target tokens."""
        rows: dict[int, np.ndarray] = {}
        skipped = 0
        for source, entries in read_shortlist_file(path).items():
            if source not in src_vocab:
                skipped += 1
                continue
            known = {trg_vocab.to_id(t) for t, _ in entries if t in trg_vocab}
            rows[src_vocab.to_id(source)] = np.array(sorted(known), dtype=np.int64)
        if skipped:
            log.info("shortlist: %d source tokens are not in the model vocabulary", skipped)
        return cls(rows)

    def lookup(self, src_ids) -> np.ndarray:
        """Sorted union of the candidate rows of the given source ids (empty
        when none of them has a row)."""
        hits = [self.rows[s] for s in {int(i) for i in src_ids} if s in self.rows]
        return sorted_union(*hits) if hits else np.zeros(0, dtype=np.int64)


def sorted_union(*arrays) -> np.ndarray:
    """np.unique(np.concatenate(arrays)) as int64 for vocabulary ids: a
    presence bitmap over [0, max id] instead of a sort/hash (the batch-1
    latency path calls this on every sentence's ~6k shortlist ids; numpy's
    unique took ~0.4 ms per call there).  Falls back to np.unique for
    negative or huge ids."""
    parts = [np.asarray(a, dtype=np.int64).ravel() for a in arrays]
    cat = np.concatenate(parts) if len(parts) != 1 else parts[0]
    if cat.size == 0:
        return np.zeros(0, dtype=np.int64)
    lo, hi = int(cat.min()), int(cat.max())
    if lo < 0 or hi > (1 << 26):
        return np.unique(cat)
    seen = np.zeros(hi + 1, dtype=bool)
    seen[cat] = True
    return np.flatnonzero(seen).astype(np.int64)
