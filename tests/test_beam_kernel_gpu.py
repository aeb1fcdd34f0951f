"""The device beam kernel (skb_beam_step) against exact search oracles.

North star: top-k indices and beam back-pointers bit-exact GIVEN IDENTICAL
SCORES.  The oracle's recorded fp32 log-probs are fed to the kernel as-is
(lp_in mode) through a replaying stub model; every pick, every parent, the
final hypothesis and its float64 log-prob must match exactly.  Plus the
reference's own scripted-model oracles (test_search.py:291-395):
exhaustive enumeration, forced EOS at the cap, natural EOS.
"""

from types import SimpleNamespace

import numpy as np
import pytest

from fixture_models import oracle_model
from oracle import skiff_oracle as O

pytestmark = pytest.mark.gpu


class _State:
    def __init__(self):
        self.active_ids = None
        self.enc = None
        self.step = 0
        self.rows = [0]

    def select_rows(self, idx):
        self.rows = list(idx)


class ReplayModel:
    """Replays an oracle beam trace: decode_step returns the recorded fp32
    log-prob matrix and checks the device fed exactly the recorded tokens."""

    def __init__(self, trace, V, nf=0):
        self.trace = trace
        self.config = SimpleNamespace(target_factor_specs=[], source_factor_specs=[],
                                      max_seq_len=999, trg_vocab_size=V)

    def decode_init(self, src_ids, src_factor_ids, lengths):
        return _State()

    def decode_step(self, state, prev_ids, prev_factor_ids):
        rec = self.trace[state.step]
        assert list(np.asarray(prev_ids)) == list(rec["fed"]), (state.step, prev_ids, rec["fed"])
        state.step += 1
        return SimpleNamespace(surface=SimpleNamespace(data=rec["lp"]), factors=[],
                               active_ids=None)


def _device_beam(model, src, beam, alpha=1.0, prefix=()):
    from paper_2207_05851_b200.engine import ChunkJob
    from paper_2207_05851_b200.search import ProtocolSearch
    job = ChunkJob(list(src), [], list(prefix), [])
    return ProtocolSearch.from_job(model, job, beam, None, alpha)


@pytest.mark.parametrize("name,beam,L,alpha", [("toy", 4, 4, 1.0), ("toy", 5, 7, 0.6),
                                               ("ssru", 3, 5, 1.0), ("tiny", 5, 4, 1.0),
                                               ("tiny", 1, 6, 1.0), ("toy", 12, 3, 1.0)])
def test_replayed_oracle_trace_bit_exact(name, beam, L, alpha):
    om = oracle_model(name)
    rng = np.random.default_rng(beam * 100 + L)
    src = [int(x) for x in rng.integers(4, om.cfg.src_vocab_size, size=L)]
    trace = []
    hyp = O.beam(om, O.OChunk(src), beam, alpha=alpha, trace=trace)
    ps = _device_beam(ReplayModel(trace, om.cfg.trg_vocab_size), src, beam, alpha)
    ps.lp_in = True
    dh = ps.run()
    assert dh.tokens == hyp.tokens
    assert dh.logprob == hyp.logprob
    assert dh.steps == hyp.steps and dh.forced_eos == hyp.forced_eos


class TieModel:
    """Markov toy with heavily tied, quantised log-probs: exercises the
    (score desc, token asc, parent asc) ordering and EOS routing."""

    def __init__(self, V, seed, q=0.5, T=6):
        rng = np.random.default_rng(seed)
        tab = np.round(rng.normal(size=(T, V, V)) / q) * q
        self.lp = O.log_softmax(tab.astype(np.float32))
        self.lp = np.round(self.lp / q).astype(np.float32) * np.float32(q)  # exact ties
        self.config = SimpleNamespace(target_factor_specs=[], source_factor_specs=[],
                                      max_seq_len=999, trg_vocab_size=V)
        self.cfg = O.OConfig(src_vocab_size=V, trg_vocab_size=V)

    class St:
        def __init__(self):
            self.last = [2]
            self.step = 0
            self.active_ids = None
            self.enc = None

        def select_rows(self, idx):
            self.last = [self.last[i] for i in idx]

    def decode_init(self, *a, **k):
        return TieModel.St()

    def decode_step(self, state, prev_ids, prev_factor_ids):
        state.last = [int(i) for i in prev_ids]
        t = min(state.step, self.lp.shape[0] - 1)
        state.step += 1
        lp = np.stack([self.lp[t, last] for last in state.last])
        return SimpleNamespace(surface=SimpleNamespace(data=lp), factors=[], active_ids=None)


class _OracleAdapter:
    """Expose a protocol model to the oracle's beam() (surface, factors)."""

    def __init__(self, m):
        self.m = m
        self.cfg = m.cfg

    def decode_init(self, ids, fids, lengths, active_ids=None):
        s = self.m.decode_init()
        return s

    def decode_step(self, st, prev, prev_f):
        out = self.m.decode_step(st, prev, prev_f)
        return out.surface.data, []


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("beam", [2, 4, 5])
def test_ties_match_oracle(seed, beam):
    m = TieModel(V=9, seed=seed)
    src = [5, 6]
    want = O.beam(_OracleAdapter(m), O.OChunk(src), beam, normalize=lambda x: x)
    ps = _device_beam(m, src, beam)
    ps.lp_in = True
    got = ps.run()
    assert got.tokens == want.tokens and got.logprob == want.logprob
    assert got.steps == want.steps and got.forced_eos == want.forced_eos


def test_prefix_forcing_and_forced_keys():
    m = TieModel(V=9, seed=11)
    src = [5, 6, 7]
    want = O.beam(_OracleAdapter(m), O.OChunk(src, prefix_ids=[7, 8, 4]), 4,
                  normalize=lambda x: x)
    ps = _device_beam(m, src, 4, prefix=[7, 8, 4])
    ps.lp_in = True
    got = ps.run()
    assert got.tokens[:3] == [7, 8, 4]
    assert got.tokens == want.tokens and got.logprob == want.logprob


# ---------------------------- reference scripted-model oracles (test_search.py)
class StubModel:
    """test_search.py:305-320: logits depend only on (step, previous token)."""

    def __init__(self, tables):
        self.tables = np.asarray(tables, dtype=np.float32)
        V = self.tables.shape[1]
        self.config = SimpleNamespace(target_factor_specs=[], source_factor_specs=[],
                                      max_seq_len=99, trg_vocab_size=V)

    def decode_init(self, src_ids, src_factor_ids, lengths):
        s = TieModel.St()
        return s

    def decode_step(self, state, prev_ids, prev_factor_ids):
        state.last = [int(i) for i in prev_ids]
        t = min(state.step, self.tables.shape[0] - 1)
        state.step += 1
        logits = np.stack([self.tables[t, last] for last in state.last])
        return SimpleNamespace(surface=SimpleNamespace(data=logits), factors=[], active_ids=None)


def _exhaustive(tables, horizon, alpha):
    V = tables.shape[1]
    best = None
    stack = [([], 2, 0.0)]
    while stack:
        toks, last, lp_sum = stack.pop()
        t = min(len(toks), tables.shape[0] - 1)
        lp = O.log_softmax(tables[t, last][None, :])[0]
        done = (toks, lp_sum + float(lp[3]), len(toks) + 1)
        if best is None or done[1] / done[2] ** alpha > best[0]:
            best = (done[1] / done[2] ** alpha, done)
        if len(toks) < horizon:
            for tok in range(V):
                if tok != 3:
                    stack.append((toks + [tok], tok, lp_sum + float(lp[tok])))
    return best[1]


def test_beam_four_matches_exhaustive_enumeration():
    rng = np.random.default_rng(21)
    tables = rng.normal(size=(4, 6, 6)).astype(np.float32)
    tables[3] = O.NEG_INF
    tables[3, :, 3] = 0.0
    got = _device_beam(StubModel(tables), [4], 4).run()
    toks, lp, steps = _exhaustive(tables, 3, 1.0)
    assert got.tokens == toks and abs(got.logprob - lp) < 1e-6 and got.steps == steps


def test_cap_forces_eos_and_flags_it():
    tables = np.zeros((1, 6, 6), dtype=np.float32)
    tables[:, :, 3] = O.NEG_INF
    tables[:, :, 5] = 1.0
    for beam in (1, 2):
        got = _device_beam(StubModel(tables), [4], beam).run()
        assert got.forced_eos and got.steps == 12 and got.tokens == [5] * 11


def test_natural_eos_at_the_last_step_is_not_flagged():
    tables = np.zeros((1, 6, 6), dtype=np.float32)
    tables[:, :, 3] = 5.0
    got = _device_beam(StubModel(tables), [4], 1).run()
    assert got.tokens == [] and not got.forced_eos
