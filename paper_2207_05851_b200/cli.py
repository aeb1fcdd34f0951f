"""Command-line front end on the B200 backend (mirrors skiff cli.py:124-252,
257-384 for the translation entry points).

    python -m paper_2207_05851_b200 translate -m MODEL_DIR [--beam 5] < in > out
    python -m paper_2207_05851_b200 bench -m MODEL_DIR [--sentences 16 ...]

Same flags, stdin/stdout wire format (plain or JSON lines), per-line error
isolation and exit codes as the reference: 0 ok, 1 usage/config, 2 bad
input or data, 3 numeric.  Training, data preparation and shortlist
building are out of scope for this hot-path backend and exit 1.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import logging
import sys
import time

import numpy as np

from .checkpoint import load_model_dir
from .config import decoder_step_cost
from .errors import CapabilityError, DataError, InputError, NumericError, SkiffError
from .search import (NvsRestriction, SearchSettings, ShortlistRestriction, parse_input_line,
                     translate)
from .shortlist import Shortlist

logger = logging.getLogger(__name__)
DEFAULT_SEED = 13


class _Parser(argparse.ArgumentParser):
    """argparse exits 2 on usage errors; the contract is 1 (cli.py:39-46)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(1)


def _print_config(config) -> None:
    for f in dataclasses.fields(config):
        print(f"{f.name} = {getattr(config, f.name)}")


def _cmd_translate(args) -> int:
    """cli.py:124-160."""
    if args.quantize:
        raise CapabilityError("int8 feed-forward is not part of the B200 backend (bf16/fp32)")
    md = load_model_dir(args.model, precision=args.precision)
    model = md.model
    if args.show_config:
        _print_config(model.config)
        return 0
    restriction = None
    if args.shortlist is not None:
        restriction = ShortlistRestriction(Shortlist.from_file(args.shortlist, md.src_vocab,
                                                               md.trg_vocab))
    elif args.nvs_threshold is not None:
        restriction = NvsRestriction(args.nvs_threshold)
    settings = SearchSettings(beam=args.beam, length_alpha=args.length_alpha,
                              restriction=restriction, use_greedy=True if args.greedy else None)
    out = sys.stdout
    pending: list = []
    for line in sys.stdin:
        try:
            inp = parse_input_line(line.rstrip("\n"))
            inp.strip_prefix = args.strip_prefix
            inp.prefix_all_chunks = args.prefix_all_chunks
            pending.append(inp)
        except InputError as e:
            pending.append(e)  # a malformed line must not sink its batch
        if len(pending) >= args.batch_size:
            _emit(out, args, model, md, settings, pending)
            pending.clear()
    if pending:
        _emit(out, args, model, md, settings, pending)
    out.flush()
    return 0


def _emit(out, args, model, md, settings, pending) -> None:
    """cli.py:163-186: parse failures are carried as exceptions in order."""
    good = [p for p in pending if not isinstance(p, InputError)]
    records = iter(translate(model, md, good, settings))
    for p in pending:
        if isinstance(p, InputError):
            logger.warning("input error: %s", p)
            text, score, factors, forced, error = "", 0.0, [], False, str(p)
        else:
            r = next(records)
            if r.error is not None:
                logger.warning("input error: %s", r.error)
            text, score, factors, forced, error = r.text, r.score, r.factors, r.forced_eos, r.error
        if args.json:
            obj: dict = {"translation": text, "score": score}
            if factors:
                obj["factors"] = factors
            obj["forced_eos"] = forced
            if error is not None:
                obj["error"] = error
            out.write(json.dumps(obj, ensure_ascii=False) + "\n")
        else:
            out.write(text + "\n")


def _cmd_bench(args) -> int:
    """cli.py:210-252: batch-1 greedy decode speed through the model protocol
    (decode_init + a fixed number of decode_step calls with argmax feedback),
    on the device."""
    if args.quantize:
        raise CapabilityError("int8 feed-forward is not part of the B200 backend (bf16/fp32)")
    import torch
    md = load_model_dir(args.model, precision=args.precision)
    model = md.model
    if args.show_config:
        _print_config(model.config)
        return 0
    config = model.config
    rng = np.random.default_rng(args.seed)

    def synth():
        src = rng.integers(4, config.src_vocab_size, size=args.length, dtype=np.int32)[None, :]
        factors = [rng.integers(4, s.vocab_size, size=args.length, dtype=np.int32)[None, :]
                   for s in config.source_factor_specs]
        return src, factors

    def run_one() -> None:
        src, factors = synth()
        state = model.decode_init(src, factors, np.array([args.length]))
        prev = np.array([2], dtype=np.int64)
        prev_fac = [np.array([4], dtype=np.int64) for _ in config.target_factor_specs]
        for _ in range(args.steps):
            step = model.decode_step(state, prev, prev_fac)
            prev = step.surface.data.argmax(axis=-1).reshape(1)
            prev_fac = [f.data.argmax(axis=-1).reshape(1) for f in step.factors]

    for _ in range(args.warmup):
        run_one()
    torch.cuda.synchronize()
    start = time.perf_counter()
    for _ in range(args.sentences):
        run_one()
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - start
    cost = sum(decoder_step_cost(config, t, args.length) for t in range(args.steps)) / args.steps
    print(f"sentences_per_sec = {args.sentences / elapsed:.3f}")
    print(f"tokens_per_sec = {args.sentences * args.steps / elapsed:.3f}")
    print(f"decoder_step_cost = {cost:.1f}")
    return 0


def _out_of_scope(args) -> int:
    raise CapabilityError(f"'{args.command}' is not part of the B200 translation backend; "
                          "use the reference package for training and data preparation")


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="skiff-b200", description="B200-native translation (skiff drop-in).")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)
    p = sub.add_parser("translate", help="translate stdin lines to stdout")
    p.add_argument("-m", "--model", required=True, help="model directory")
    mode = p.add_mutually_exclusive_group()
    mode.add_argument("--beam", type=int, default=1, help="beam size")
    mode.add_argument("--greedy", action="store_true", help="force the dedicated greedy decoder")
    restrict = p.add_mutually_exclusive_group()
    restrict.add_argument("--shortlist", help="lexical shortlist file")
    restrict.add_argument("--nvs-threshold", type=float,
                          help="vocabulary selection probability threshold")
    p.add_argument("--quantize", choices=["int8"], help="(not supported on this backend)")
    p.add_argument("--json", action="store_true", help="emit one JSON object per line")
    p.add_argument("--strip-prefix", action="store_true")
    p.add_argument("--prefix-all-chunks", action="store_true")
    p.add_argument("--length-alpha", type=float, default=1.0)
    p.add_argument("--batch-size", type=int, default=32)
    p.add_argument("--precision", choices=["bf16", "fp32"], default="bf16",
                   help="GEMM operand precision (fp32 = parity mode)")
    p.add_argument("--show-config", action="store_true")
    p.set_defaults(func=_cmd_translate)
    p = sub.add_parser("bench", help="measure batch-1 decoding speed for a model")
    p.add_argument("-m", "--model", required=True, help="model directory")
    p.add_argument("--sentences", type=int, default=16)
    p.add_argument("--length", type=int, default=12, help="source length")
    p.add_argument("--steps", type=int, default=24, help="decode steps per sentence")
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--quantize", choices=["int8"], help="(not supported on this backend)")
    p.add_argument("--seed", type=int, default=DEFAULT_SEED)
    p.add_argument("--precision", choices=["bf16", "fp32"], default="bf16")
    p.add_argument("--show-config", action="store_true")
    p.set_defaults(func=_cmd_bench)
    for name in ("prepare-data", "train", "build-shortlist"):
        p = sub.add_parser(name, help="(reference only: out of scope here)")
        p.set_defaults(func=_out_of_scope)
    return parser


def main(argv: list[str] | None = None) -> int:
    """cli.py:364-384 exit-code contract."""
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    logging.basicConfig(stream=sys.stderr, level=logging.INFO,
                        format="[%(levelname)s] %(message)s")
    try:
        return args.func(args)
    except (InputError, DataError) as e:
        print(f"skiff: error: {e}", file=sys.stderr)
        return 2
    except NumericError as e:
        print(f"skiff: error: {e}", file=sys.stderr)
        return 3
    except OSError as e:
        print(f"skiff: error: {e}", file=sys.stderr)
        return 2
    except SkiffError as e:
        print(f"skiff: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
