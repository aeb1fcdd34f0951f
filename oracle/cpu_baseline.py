"""CPU baseline timing of the reference algorithm — TEST/BENCH INFRASTRUCTURE.

Runs the oracle port (skiff_oracle.beam, the reference's decode path with
float64-accumulated numpy matmuls, kernels.py:167-176) in P single-threaded
worker processes (OPENBLAS_NUM_THREADS=1, as the reference pins BLAS,
__init__.py:9-11).  A bounded sample: each worker encodes one sentence and
runs the first n_steps beam steps; the per-sentence time is extrapolated to
the full 2L+10 steps (every random-init decode runs to the cap).
Only bench.py's cpu_baseline leg and --impl reference import this module.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

_MODEL = None


_RESTRICTION = None


def _init(cfg_kwargs, seed, shortlist_topk=None):
    global _MODEL, _RESTRICTION
    from oracle import skiff_oracle as O
    cfg = O.OConfig(**cfg_kwargs)
    _MODEL = O.OracleModel(cfg, O.init_params(cfg, seed))
    if shortlist_topk:
        from oracle.fixture_configs import synthetic_shortlist_rows
        _RESTRICTION = ("shortlist", synthetic_shortlist_rows(cfg.trg_vocab_size, shortlist_topk))


def _work(args):
    from oracle import skiff_oracle as O
    src, beam, alpha, n_steps = args
    timings = []
    t0 = time.perf_counter()
    O.beam(_MODEL, O.OChunk(list(src)), beam, restriction=_RESTRICTION, alpha=alpha,
           max_steps=n_steps, timings=timings)
    return timings, time.perf_counter() - t0


def default_procs() -> int:
    """P = min(nproc, floor(RAM / 4 GB)) single-threaded workers."""
    ncpu = os.cpu_count() or 1
    try:
        with open("/proc/meminfo") as f:
            kb = next(int(ln.split()[1]) for ln in f if ln.startswith("MemTotal"))
        by_ram = max(1, kb // (4 * 1024 * 1024))
    except (OSError, StopIteration, ValueError):
        by_ram = ncpu
    return max(1, min(ncpu, by_ram))


class CpuBaseline:
    """Pool of P single-threaded oracle workers holding the same weights."""

    def __init__(self, cfg_kwargs: dict, seed: int = 13, procs: int | None = None,
                 shortlist_topk: int | None = None):
        for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        self.procs = procs or default_procs()
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.procs, initializer=_init,
                             initargs=(cfg_kwargs, seed, shortlist_topk))
        # make sure every worker has built its model before timing
        self.pool.map(_noop, range(self.procs * 2))

    def sample(self, sources: list[list[int]], beam: int, alpha: float, n_steps: int):
        """Run len(sources) (<= procs) bounded decodes in parallel.  Returns
        (extrapolated sentences/s over the pool, wall seconds, detail)."""
        t0 = time.perf_counter()
        res = self.pool.map(_work, [(s, beam, alpha, n_steps) for s in sources])
        wall = time.perf_counter() - t0
        per_sent = []
        for (tim, _), src in zip(res, sources):
            S = 2 * len(src) + 10
            init, steps = tim[0], tim[1:]
            rest = steps[1:] if len(steps) > 1 else steps
            per_sent.append(init + sum(steps) + (S - len(steps)) * (sum(rest) / len(rest)))
        mean_sent = sum(per_sent) / len(per_sent)
        return self.procs / mean_sent, wall, {"sec_per_sentence": mean_sent,
                                              "measured_steps": n_steps}

    def close(self):
        self.pool.terminate()


def _noop(_):
    time.sleep(0.05)
    return _MODEL is not None
