"""Command-line front end of the B200 backend.

    python -m paper_2207_05851_b200 translate -m MODEL_DIR [--beam 5] < in > out
    python -m paper_2207_05851_b200 bench -m MODEL_DIR [--sentences 16 ...]

Contract shared with the reference CLI (skiff cli.py:124-252 for the two
commands, :364-384 for the exit codes), so scripts driving one drive the
other: the same flags; stdin lines in plain text or the JSON record format
(search.parse_input_line); stdout one translation per input line, plain or
`{"translation", "score", ["factors"], "forced_eos", ["error"]}` JSON; a
malformed line yields an error record in its place and never aborts the
others; exit status 0 ok / 1 usage or configuration / 2 input or data /
3 numeric.  Training, data preparation and shortlist building belong to the
reference package and exit 1 here (SURVEY §2 scope).
"""

from __future__ import annotations

import argparse
import dataclasses
import itertools
import json
import logging
import sys
import time
from typing import Iterable, Iterator

import numpy as np

from .checkpoint import load_model_dir
from .config import decoder_step_cost
from .errors import CapabilityError, DataError, InputError, NumericError, SkiffError
from .search import (NvsRestriction, SearchSettings, ShortlistRestriction, parse_input_line,
                     translate)
from .quant import quantize_model
from .shortlist import Shortlist

log = logging.getLogger(__name__)
DEFAULT_SEED = 13
BOS_ID, SHIFT_ID = 2, 4

# exception class -> process exit status (most specific first)
EXIT_CODES: tuple[tuple[type, int], ...] = (
    (InputError, 2), (DataError, 2), (OSError, 2), (NumericError, 3), (SkiffError, 1))


class ArgumentParser(argparse.ArgumentParser):
    """Usage errors exit with status 1 (argparse's own default is 2)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(1)


# ------------------------------------------------------------------ helpers
def _load(args):
    mdir = load_model_dir(args.model, precision=args.precision)
    if args.quantize == "int8":  # cli.py:130-131 / 216-217
        quantize_model(mdir.model)
    return mdir


def _show(config) -> int:
    print("\n".join(f"{f.name} = {getattr(config, f.name)}" for f in dataclasses.fields(config)))
    return 0


def _settings(args, mdir) -> SearchSettings:
    if args.shortlist is not None:
        sl = Shortlist.from_file(args.shortlist, mdir.src_vocab, mdir.trg_vocab)
        restriction = ShortlistRestriction(sl)
    elif args.nvs_threshold is not None:
        restriction = NvsRestriction(args.nvs_threshold)
    else:
        restriction = None
    return SearchSettings(beam=args.beam, length_alpha=args.length_alpha, restriction=restriction,
                          use_greedy=True if args.greedy else None)


def _parsed_lines(stream: Iterable[str], args) -> Iterator:
    """One item per input line: a SentenceInput, or the InputError that the
    line raised (kept in place so the output stays line-aligned)."""
    for raw in stream:
        try:
            item = parse_input_line(raw.rstrip("\n"))
        except InputError as err:
            yield err
            continue
        item.strip_prefix = args.strip_prefix
        item.prefix_all_chunks = args.prefix_all_chunks
        yield item


def _as_output(args, text, score, factors, forced, error) -> str:
    if not args.json:
        return text
    rec = {"translation": text, "score": score}
    if factors:
        rec["factors"] = factors
    rec["forced_eos"] = forced
    if error is not None:
        rec["error"] = error
    return json.dumps(rec, ensure_ascii=False)


def _translate_group(args, mdir, settings, group: list) -> Iterator[str]:
    inputs = [g for g in group if not isinstance(g, InputError)]
    done = iter(translate(mdir.model, mdir, inputs, settings))
    for g in group:
        if isinstance(g, InputError):
            log.warning("input error: %s", g)
            yield _as_output(args, "", 0.0, [], False, str(g))
            continue
        rec = next(done)
        if rec.error is not None:
            log.warning("input error: %s", rec.error)
        yield _as_output(args, rec.text, rec.score, rec.factors, rec.forced_eos, rec.error)


# ------------------------------------------------------------------ commands
def cmd_translate(args) -> int:
    """Translate stdin to stdout in groups of --batch-size lines (each group
    is one translate() call, i.e. one batched device run)."""
    mdir = _load(args)
    if args.show_config:
        return _show(mdir.model.config)
    settings = _settings(args, mdir)
    lines = _parsed_lines(sys.stdin, args)
    while True:
        group = list(itertools.islice(lines, max(1, args.batch_size)))
        if not group:
            break
        sys.stdout.write("".join(o + "\n" for o in _translate_group(args, mdir, settings, group)))
    sys.stdout.flush()
    return 0


class _ProtocolBench:
    """Batch-1 decode speed through the model protocol the reference bench
    drives: decode_init on a random source, then a fixed number of
    decode_step calls feeding back the argmax token (no early stop)."""

    def __init__(self, model, length, steps, seed):
        self.model, self.length, self.steps = model, length, steps
        self.rng = np.random.default_rng(seed)

    def source(self):
        c = self.model.config
        ids = self.rng.integers(4, c.src_vocab_size, size=self.length, dtype=np.int32)
        facs = [self.rng.integers(4, spec.vocab_size, size=self.length, dtype=np.int32)[None]
                for spec in c.source_factor_specs]
        return ids[None], facs

    def sentence(self):
        ids, facs = self.source()
        state = self.model.decode_init(ids, facs, np.array([self.length]))
        token = np.array([BOS_ID], dtype=np.int64)
        factor_tokens = [np.array([SHIFT_ID], dtype=np.int64)
                         for _ in self.model.config.target_factor_specs]
        for _ in range(self.steps):
            out = self.model.decode_step(state, token, factor_tokens)
            token = out.surface.data.argmax(axis=-1).reshape(1)
            factor_tokens = [f.data.argmax(axis=-1).reshape(1) for f in out.factors]


def cmd_bench(args) -> int:
    import torch
    mdir = _load(args)
    model = mdir.model
    if args.show_config:
        return _show(model.config)
    bench = _ProtocolBench(model, args.length, args.steps, args.seed)
    for _ in range(args.warmup):
        bench.sentence()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.sentences):
        bench.sentence()
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    mean_cost = np.mean([decoder_step_cost(model.config, t, args.length) for t in range(args.steps)])
    report = {"sentences_per_sec": args.sentences / secs,
              "tokens_per_sec": args.sentences * args.steps / secs,
              "decoder_step_cost": mean_cost}
    for key, val in report.items():
        print(f"{key} = {val:.{1 if key == 'decoder_step_cost' else 3}f}")
    return 0


def cmd_reference_only(args) -> int:
    raise CapabilityError(f"'{args.command}' is not part of the B200 translation backend; "
                          "use the reference package for training and data preparation")


# ------------------------------------------------------------------ parser
def _common(p, *, quantize=True):
    p.add_argument("-m", "--model", required=True, help="model directory")
    if quantize:
        p.add_argument("--quantize", choices=["int8"],
                       help="int8 feed-forward layers (dynamic per-row quantization)")
    p.add_argument("--precision", choices=["bf16", "fp32"], default="bf16",
                   help="GEMM operand precision (fp32 = parity mode)")
    p.add_argument("--show-config", action="store_true")


def build_parser() -> argparse.ArgumentParser:
    top = ArgumentParser(prog="skiff-b200", description="B200-native translation (skiff drop-in).")
    cmds = top.add_subparsers(dest="command", required=True, parser_class=ArgumentParser)

    tr = cmds.add_parser("translate", help="translate stdin lines to stdout")
    _common(tr)
    search = tr.add_mutually_exclusive_group()
    search.add_argument("--beam", type=int, default=1, help="beam size")
    search.add_argument("--greedy", action="store_true", help="force the dedicated greedy decoder")
    vocab = tr.add_mutually_exclusive_group()
    vocab.add_argument("--shortlist", help="lexical shortlist file")
    vocab.add_argument("--nvs-threshold", type=float, help="vocabulary selection threshold")
    tr.add_argument("--json", action="store_true", help="emit one JSON object per line")
    tr.add_argument("--strip-prefix", action="store_true")
    tr.add_argument("--prefix-all-chunks", action="store_true")
    tr.add_argument("--length-alpha", type=float, default=1.0)
    tr.add_argument("--batch-size", type=int, default=32)
    tr.set_defaults(func=cmd_translate)

    be = cmds.add_parser("bench", help="measure batch-1 decoding speed for a model")
    _common(be)
    for flag, default, text in (("--sentences", 16, "timed sentences"),
                                ("--length", 12, "source length"),
                                ("--steps", 24, "decode steps per sentence"),
                                ("--warmup", 2, "untimed sentences"),
                                ("--seed", DEFAULT_SEED, "source sampling seed")):
        be.add_argument(flag, type=int, default=default, help=text)
    be.set_defaults(func=cmd_bench)

    for name in ("prepare-data", "train", "build-shortlist"):
        cmds.add_parser(name, help="(reference only: out of scope here)").set_defaults(
            func=cmd_reference_only)
    return top


def exit_code(err: BaseException) -> int:
    return next(code for cls, code in EXIT_CODES if isinstance(err, cls))


def main(argv: list[str] | None = None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as stop:
        return int(stop.code or 0)
    logging.basicConfig(stream=sys.stderr, level=logging.INFO, format="[%(levelname)s] %(message)s")
    try:
        return args.func(args)
    except (SkiffError, OSError) as err:
        print(f"skiff: error: {err}", file=sys.stderr)
        return exit_code(err)


if __name__ == "__main__":
    sys.exit(main())
