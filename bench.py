#!/usr/bin/env python
"""Benchmark: transformer-big 6-6 beam-5 translation throughput on B200.

Metric (BASELINE.json): sentences/sec (transformer-big beam 5) at 1/2/4/8
B200.  Workload per GPU and step: one batch of 128 synthetic WMT-shaped
sentences (L = 30 source tokens, uniform ids) decoded with beam
5 and length penalty alpha = 1.0 (search.py:74-75) in bf16 on random-init
weights (seed 13, model.py:244-265).  Every random-init decode runs to the
2L+10 = 70-step cap, so the work per sentence is fixed.

  value       device throughput: inputs staged in HBM, timed region =
              encoder + cross K/V + 70 captured decode steps + finalize
  e2e         the public API: translate(model, vocabs, SentenceInput list)
              from host strings to TranslationRecords (H2D/D2H inside)
  roofline    all tcgen05 GEMMs of one decode step (the dominant kernel
              class), timed live with CUDA events on their stream
  cpu_baseline the reference algorithm (oracle port, float64 numpy) on this
              box's host cores, bounded sample, rank 0 at N=1 only

Multi-GPU: `python -m torch.distributed.run --nproc-per-node N bench.py
--gpus N`; sentences are sharded (weak scaling, replicas), the only
collective is the final gather of hypotheses to rank 0.
`--impl reference` times the reference's CPU algorithm (oracle port) on the
same workload instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sentences/sec (transformer-big beam 5)"
UNIT = "sentences/s"
BIG = dict(src_vocab_size=32000, trg_vocab_size=32000, d_model=1024, heads=16, ff_dim=4096,
           encoder_layers=6, decoder_layers=6, decoder_kind="self_attention", max_seq_len=128)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=9)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="big", choices=sorted(MODELS))
    ap.add_argument("--batch", type=int, default=0, help="sentences per batch (0 = the config's)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other configs' lines (base, SSRU + shortlist, batch 256, "
                         "batch-1 latency by architecture)")
    ap.add_argument("--beam", type=int, default=5)
    ap.add_argument("--src-len", type=int, default=30)
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--cpu-steps", type=int, default=6, help="decode steps in the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no JSON rules)")
    ap.add_argument("--gemm-split", default="throughput", choices=["throughput", "latency"],
                    help="GEMM K-split policy of the measured model (Model(gemm_split=...))")
    ap.add_argument("--streams", type=int, default=int(os.environ.get("SKB_STREAMS", "5")),
                    help="independent batches decoded concurrently on separate CUDA streams")
    return ap.parse_args()


def synth_sentences(n, L, V, seed):
    """default_rng(seed).integers(0, V-4) -> tokens w{i} (ids 4..V-1)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    return [[f"w{int(i)}" for i in rng.integers(0, V - 4, size=L)] for _ in range(n)]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(device_index)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        loaded = [x for x in sm if smax and x > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- our path
BASE = dict(BIG, d_model=512, heads=8, ff_dim=2048)
BIG_SSRU = dict(BIG, encoder_layers=20, decoder_layers=2, decoder_kind="ssru")
BIG_20_2 = dict(BIG, encoder_layers=20, decoder_layers=2)
MODELS = {
    "big": (BIG, "transformer-big 6-6 (d1024 H16 ff4096 V32000)", None),
    "base": (BASE, "transformer-base 6-6 (d512 H8 ff2048 V32000)", None),
    "big_ssru": (BIG_SSRU, "transformer-big 20-2 hybrid, SSRU decoder (d1024 H16 ff4096 V32000), "
                           "lexical shortlist top-200", 200),
    "big_20_2": (BIG_20_2, "transformer-big 20-2, self-attention decoder (d1024 H16 ff4096 V32000)",
                 None),
    "big_ssru_nosl": (BIG_SSRU, "transformer-big 20-2 hybrid, SSRU decoder (d1024 H16 ff4096 V32000)",
                      None),
}
DEFAULT_BATCH = {"big": 128, "base": 64, "big_ssru": 128, "big_20_2": 128, "big_ssru_nosl": 128}


def synthetic_shortlist_rows(V: int, k: int = 200, seed: int = 7) -> dict:
    """SURVEY §8d synthetic lexical shortlist: every source id 4..V-1 gets k
    distinct target ids drawn from 4..V-1 with default_rng(seed) (the first k
    distinct values of an oversampled draw), sorted as Shortlist rows are.
    Same generator as the golden fixtures' (tests check they agree)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    draw = rng.integers(4, V, size=(V - 4, k + k // 2 + 16))
    rows = {}
    for i in range(V - 4):
        u, first = np.unique(draw[i], return_index=True)
        pick = u[np.argsort(first)][:k]
        if pick.size < k:  # pragma: no cover
            extra = np.setdiff1d(np.arange(4, V), pick)[: k - pick.size]
            pick = np.concatenate([pick, extra])
        rows[i + 4] = np.sort(pick).astype(np.int64)
    return rows


def build_model(name="big", precision="bf16", gemm_split="throughput"):
    from paper_2207_05851_b200.checkpoint import SPECIALS, Vocabulary
    from paper_2207_05851_b200.config import ModelConfig, init_params
    from paper_2207_05851_b200.model import Model
    from paper_2207_05851_b200.search import ShortlistRestriction
    from paper_2207_05851_b200.shortlist import Shortlist
    spec, _, topk = MODELS[name]
    cfg = ModelConfig(**spec)
    model = Model(cfg, params=init_params(cfg, 13), precision=precision, gemm_split=gemm_split)
    words = SPECIALS + [f"w{i}" for i in range(cfg.trg_vocab_size - 4)]
    v = Vocabulary(words)
    vocabs = SimpleNamespace(src_vocab=v, trg_vocab=v, src_factor_vocabs=[], trg_factor_vocabs=[])
    restriction = None
    if topk:
        restriction = ShortlistRestriction(Shortlist(synthetic_shortlist_rows(cfg.trg_vocab_size, topk)))
    return model, vocabs, restriction


def make_batch(model, vocabs, sentences, beam, alpha, slot=0, restriction=None):
    from paper_2207_05851_b200.engine import BeamBatch
    from paper_2207_05851_b200.search import SentenceInput, _chunk_job
    jobs = [_chunk_job(model, SentenceInput(tokens=s), vocabs, restriction)[0] for s in sentences]
    return BeamBatch(model, jobs, beam, alpha, slot=slot)


def batch1_latency(model, vocabs, L, V, n=21, restriction=None, which=(("greedy", 1), ("beam5", 5))):
    """The metric's second part: batch-1 latency through translate() (host
    strings in, records out, one sentence per call), greedy and beam 5, p50
    over n sentences of length L (wall clock around the public call, which
    synchronises on its result)."""
    import torch
    from paper_2207_05851_b200 import kern
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    kern.set_concurrency(1)
    out = {}
    for name, beam in which:
        sents = synth_sentences(n + 2, L, V, seed=4242)
        st = SearchSettings(beam=beam, restriction=restriction)
        for s in sents[:2]:  # warm-up: workspace + captured graphs for this shape
            translate(model, vocabs, [SentenceInput(tokens=s)], st)
        torch.cuda.synchronize()
        ts = []
        for s in sents[2:]:
            t0 = time.perf_counter()
            recs = translate(model, vocabs, [SentenceInput(tokens=s)], st)
            ts.append((time.perf_counter() - t0) * 1e3)
            assert recs[0].error is None
        ts.sort()
        out[name] = {"p50_ms": round(statistics.median(ts), 3), "p90_ms": round(ts[int(0.9 * (n - 1))], 3),
                     "steps": 2 * L + 10}
    out["api"] = "paper_2207_05851_b200.search.translate, 1 sentence per call, L=%d" % L
    return out


def _gemm_traffic():
    """DRAM bytes (read + write) of one decode step's GEMM launches from the
    committed ncu --set full capture (profiles/r2_gemm_step_traffic.json,
    made by tools/ncu_step.sh; cold-L2 serialised replay), or None."""
    p = next((q for q in (ROOT / "profiles" / f"{r}_gemm_step_traffic.json" for r in ("r2", "r1"))
              if q.exists()), None)
    if p is None:
        return None
    d = json.loads(p.read_text())
    return {"bytes_per_step": d["dram_bytes_per_step"], "source": d["source"]}


def gemm_roofline(model, R, L, peak, U=None):
    """Time every GEMM of one decode step (all decoder layers + output
    projection over U columns) with CUDA events on the launching stream;
    achieved = algorithmic FLOPs (2*M*N*K summed) / measured time."""
    import torch
    from paper_2207_05851_b200 import _native as N
    from paper_2207_05851_b200 import kern
    c = model.config
    d = c.d_model
    U = U or c.trg_vocab_size
    dev, cdt = model.device, model.cdt
    h = torch.randn(R, d, device=dev).to(cdt)
    f = torch.randn(R, c.ff_dim, device=dev).to(cdt)
    x = torch.zeros(R, d, device=dev)
    qkv = torch.empty(R, 3 * d, device=dev, dtype=cdt)
    q = torch.empty(R, d, device=dev, dtype=cdt)
    ff = torch.empty(R, c.ff_dim, device=dev, dtype=cdt)
    cell = torch.zeros(R, d, device=dev)
    rows = torch.arange(R, dtype=torch.int32, device=dev)
    E = model.E_trg_c[:U]
    logits = torch.empty(R, U, device=dev)
    part = torch.empty(R, 2 * ((U + 31) // 32), device=dev)
    calls, flops = [], 0
    for Ly in model.dec:
        if hasattr(Ly, "w_ssru"):
            calls += [(h, Ly.w_ssru, x, N.EPI_SSRU, Ly.b_ssru)]
        else:
            calls += [(h, Ly.wqkv, qkv, N.EPI_STORE, None), (h, Ly.wo, x, N.EPI_RESID, None)]
        calls += [(h, Ly.wq_c, q, N.EPI_STORE, None), (h, Ly.wo_c, x, N.EPI_RESID, None),
                  (h, Ly.w1, ff, N.EPI_RELU, Ly.b1), (f, Ly.w2, x, N.EPI_RESID, Ly.b2)]
    out_call = (h, E, logits, N.EPI_LOGITS, None)
    calls.append(out_call)
    for A, W, o, kind, b in calls:
        flops += 2 * R * W.shape[0] * W.shape[1]

    def run(cs):
        for A, W, o, kind, b in cs:
            kern.gemm(A, W, o, kind, b, lse_part=part if kind == N.EPI_LOGITS else None,
                      c_state=cell if kind == N.EPI_SSRU else None,
                      src_row=rows if kind == N.EPI_SSRU else None)

    for _ in range(3):
        run(calls)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run(calls)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    e0.record()
    for _ in range(reps):
        run([out_call])
    e1.record()
    torch.cuda.synchronize()
    ms_out = e0.elapsed_time(e1) / reps
    out_flops = 2 * R * U * d
    achieved = flops / (ms / 1e3) / 1e12
    return_kernel = ("tcgen05 GEMMs: k_gemm_sw (swap-AB, 128 weight rows x Na activation rows per "
                     "CTA; FFN2 split over a 2-CTA cluster), all GEMMs of one decode step, R=%d" % R)
    return {"kernel": return_kernel,
            "bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": _gemm_traffic(),
            "flops_per_step": flops, "ms_per_decode_step_gemms": round(ms, 4),
            "out_proj": {"ms": round(ms_out, 4), "cols": U,
                         "tflops": round(out_flops / (ms_out / 1e3) / 1e12, 1)}}


def topk_roofline(bb, hbm_peak, reps=20):
    """k_beam_step (top-k + log-softmax finish + beam bookkeeping) at step 35
    of the benchmark batch, launched back to back on its stream; achieved =
    the algorithmic bytes R*A*4 (the fp32 logits it ranks) per
    launch / average launch time.  The kernel itself reads only the output
    GEMM's per-32-column (max, sum exp) partials and the candidate groups,
    so its DRAM traffic is far below the algorithmic figure."""
    import torch
    from paper_2207_05851_b200 import kern
    sb = bb.sb
    sb.step.fill_(35)
    R, U = bb.B * bb.K, sb.logits.shape[1]
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        bb.done.zero_()
        bb.n_alive.fill_(bb.K)
        e0.record(st)
        for _ in range(reps):
            kern.beam_step(sb.logits, bb.state)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    nbytes = R * U * 4
    achieved = nbytes / (best / 1e3) / 1e9
    return {"kernel": "k_beam_step (K=%d, R=%d, A=%d)" % (bb.K, R, U), "bound": "hbm",
            "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4), "us_per_launch": round(best * 1e3, 2),
            "algorithmic_bytes_per_launch": nbytes, "traffic": _beam_traffic()}


def attention_roofline(bb, model, hbm_peak, t=35, reps=10):
    """The decode step's attention kernels at step t of the benchmark batch,
    all decoder layers back to back on their stream (CUDA events):
    self-attention over the KV cache (k_self_attn_tc over the step plan;
    algorithmic bytes = the distinct cached (slot, position) entries the
    sentences' beam rows read, K and V of every head, bf16) and
    cross-attention (k_cross_tc; bytes = every sentence's encoder K and V
    rows up to its length, once per layer).  achieved = bytes per layer / time per layer."""
    import numpy as np
    import torch
    from paper_2207_05851_b200 import kern
    c = model.config
    if c.decoder_kind == "ssru":
        return None
    sb, K, B = bb.sb, bb.K, bb.B
    R, H, dh, d = B * K, c.heads, c.head_dim, c.d_model
    D = len(model.dec)
    sb.step.fill_(t)
    if sb.plan is not None:
        kern.attn_plan(sb.anc, sb.step, sb.plan, R, sb.S_max, sb.group)
    anc = sb.anc[t & 1, :, :t].cpu().numpy()
    entries = sum(len({(int(anc[r, p]), p) for r in range(b * K, b * K + K) for p in range(t)}) + K
                  for b in range(B))
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0.record(st)
            for _ in range(reps):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / (reps * D))
        return best * 1e3  # us per layer

    def self_all():
        for li in range(D):
            kern.self_attention_step(sb.qkv, sb.kc[li], sb.vc[li], sb.anc, sb.step, sb.ctx, R, H, dh,
                                     sb.S_max, sb.group, plan=sb.plan)

    def cross_all():
        for li in range(D):
            kern.cross_attention_step(sb.q, sb.ckv, li * 2 * d, li * 2 * d + d, sb.L, sb.row_sent,
                                      sb.lengths, sb.ctx, R, H, dh, sb.group)

    us_self, us_cross = timed(self_all), timed(cross_all)
    b_self = entries * H * dh * 2 * 2
    b_cross = int(sb.lengths.sum().item()) * 2 * d * 2  # encoder K,V rows within each length
    out = {}
    for name, us, nb, kern_name in (("self", us_self, b_self, "k_self_attn_tc (step plan)"),
                                    ("cross", us_cross, b_cross, "k_cross_tc")):
        ach = nb / (us / 1e6) / 1e9
        out[name] = {"kernel": kern_name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(ach / hbm_peak, 4), "us_per_layer": round(us, 2),
                     "algorithmic_bytes_per_layer": int(nb)}
    out["self"]["distinct_entries"] = int(entries)
    out["step"] = t
    out["how"] = ("all decoder layers back to back at step %d of the benchmark batch, CUDA events; "
                  "the kernels stage cached entries before griddepcontrol.wait, which these "
                  "back-to-back launches overlap as in the decode graph" % t)
    return out


def _beam_traffic():
    """DRAM bytes per k_beam_step launch from the committed ncu capture
    (profiles/r2_beam_step_traffic.json), or None."""
    p = next((q for q in (ROOT / "profiles" / f"{r}_beam_step_traffic.json" for r in ("r2", "r1"))
              if q.exists()), None)
    if p is None:
        return None
    d = json.loads(p.read_text())
    return {"bytes_per_launch": d["dram_bytes_per_launch"], "source": d["source"]}


def distinct_kv_entries(bb, S):
    """Distinct (cache slot, position) entries the self-attention of each
    decode step reads, from the run's beam back-pointers (par_hist[t][row] =
    the parent's index within its sentence): the beam rows of a sentence
    share their common prefix, and the kernels stage each shared entry once
    (k_attn_plan).  Returns a list over steps t = 0..S-1."""
    import numpy as np
    K, R = bb.K, bb.B * bb.K
    par = bb.ws.par_hist.view(-1, R)[:S].cpu().numpy().astype(np.int64)
    base = (np.arange(R) // K) * K
    out = []
    for t in range(S):
        rows = np.arange(R) if t > 0 else np.arange(0, R, K)  # step 0: one row per sentence
        n = rows.size
        cur = rows
        for p in range(t - 1, -1, -1):
            cur = base[cur] + par[p][cur]
            n += np.unique(cur).size
        out.append(n)
    return out


def ideal_floor(model, B, K, L, S, peak_tf_sustained, hbm, U=None, distinct=None):
    """SURVEY.md 8d per-GPU floor: every GEMM FLOP at the sustained bf16 peak
    plus the HBM terms (top-k logits, self-attention KV, cross K/V) at the
    measured copy bandwidth, for one batch of B sentences over S steps.
    The KV term charges the distinct cache entries the step reads
    (`distinct`, measured from the run's back-pointers) — not every row's
    whole history, which double-counts the beam's shared prefix; the per-row
    figure is kept as `ms_per_batch_per_row_kv`."""
    from paper_2207_05851_b200.config import SSRU, decoder_step_cost, encoder_cost
    c = model.config
    d, D = c.d_model, c.decoder_layers
    U = U or c.trg_vocab_size
    sa = c.decoder_kind != SSRU
    macs = encoder_cost(c, L) + D * 2 * L * d * d + sum(
        (1 if t == 0 else K) * (decoder_step_cost(c, t, L) - d * (c.trg_vocab_size - U))
        for t in range(S))
    flops = 2.0 * macs * B
    R = B * K
    gemm_ms = flops / (peak_tf_sustained * 1e12) * 1e3

    def hbm_ms(kv_rows):
        tot = 0
        for t in range(S):
            tot += R * U * 4 + D * 2 * B * L * d * 2
            if sa:
                tot += D * 2 * kv_rows(t) * d * 2
            else:
                tot += 2 * D * R * d * 4  # SSRU cell state read + write
        return tot, tot / (hbm * 1e9) * 1e3

    per_row_b, per_row_ms = hbm_ms(lambda t: R * (t + 1))
    if distinct is not None:
        hb, hms = hbm_ms(lambda t: distinct[t])
    else:
        hb, hms = per_row_b, per_row_ms
    ms = gemm_ms + hms
    return {"ms_per_batch": round(ms, 3), "sentences_per_s": round(B / (ms / 1e3), 1),
            "gflop_per_sentence": round(flops / B / 1e9, 2), "hbm_gb_per_batch": round(hb / 1e9, 2),
            "kv": "distinct entries (measured back-pointers)" if distinct is not None and sa
            else ("SSRU state" if not sa else "per-row history"),
            "ms_per_batch_per_row_kv": round(gemm_ms + per_row_ms, 3)}


def step_breakdown(bb):
    """Eager replay of one mid-sequence decode step with CUDA events between
    kernel groups (attention, GEMMs, LN, beam) — explains `value`."""
    import torch
    from paper_2207_05851_b200 import engine, kern
    from paper_2207_05851_b200 import _native as N
    sb = bb.sb
    sb.step.fill_(35)
    bb.done.zero_()
    bb.n_alive.fill_(bb.K)
    groups = {}
    ev = []

    orig = {n: getattr(kern, n) for n in ("gemm", "layernorm", "self_attention_step",
                                          "cross_attention_step", "embed_target", "beam_step",
                                          "beam_reorder")}

    def wrap(name, fn):
        def inner(*a, **k):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            fn(*a, **k)
            e.record()
            ev.append((name, s, e))
        return inner

    for n, fn in orig.items():
        setattr(kern, n, wrap(n, fn))
    try:
        for _ in range(2):
            ev.clear()
            engine.step_forward(bb.model, sb)
            kern.beam_step(sb.logits, bb.state)
        torch.cuda.synchronize()
    finally:
        for n, fn in orig.items():
            setattr(kern, n, fn)
    for name, s, e in ev:
        groups[name] = groups.get(name, 0.0) + s.elapsed_time(e)
    total = sum(groups.values())
    return {k: round(v, 4) for k, v in sorted(groups.items(), key=lambda kv: -kv[1])} | {
        "total_ms": round(total, 4)}


def _env():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measure(model, vocabs, restriction, B, K, L, alpha, steps, warmup, n_streams, seed0=13,
            gather=None, clocks_device=None):
    """Device throughput of B-sentence batches: `steps` batches decoded on
    n_streams CUDA streams (batch i on stream i % S; on each stream batch i+S
    is launched before batch i is read back, so a stream alternates two
    workspace slots), inputs staged in HBM first; the same batches also run
    on one stream.  Returns per-stream-count timings and the last batches."""
    import torch
    import torch.distributed as dist
    from paper_2207_05851_b200 import kern
    world, rank, local = _env()
    V = model.config.trg_vocab_size

    def sents(step):
        return synth_sentences(B, L, V, seed=seed0 + 7919 * rank + 104729 * step)

    def timed(S):
        kern.set_concurrency(S)  # GEMM tiles sized for a 1/S share of the SMs
        streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(S - 1)]

        def slot_of(i):
            return 2 * (i % S) + ((i // S) & 1)

        # warm-up (compiles TMA descriptors, captures every slot's graphs)
        for w in range(max(warmup, 2 * S)):
            bb = make_batch(model, vocabs, sents(1000 + w), K, alpha, slot=slot_of(w),
                            restriction=restriction)
            with torch.cuda.stream(streams[w % S]):
                bb.run()
            if gather:
                gather(bb)
        torch.cuda.synchronize()
        batches = [make_batch(model, vocabs, sents(s), K, alpha, slot=slot_of(s),
                              restriction=restriction) for s in range(steps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = ClockSampler(clocks_device) if clocks_device is not None else None
        l0 = kern.launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in streams[1:]:
            st.wait_stream(streams[0])
        results, inflight = [], []
        for i, bb in enumerate(batches):
            with torch.cuda.stream(streams[i % S]):
                bb.start()
            inflight.append(bb)
            if len(inflight) > S:
                done = inflight.pop(0)
                results.append(done.finish())
                if gather:
                    gather(done)
        for done in inflight:
            results.append(done.finish())
            if gather:
                gather(done)
        for st in streams[1:]:
            streams[0].wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk = clocks.stop() if clocks else None
        launches = kern.launches - l0
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), results, launches, clk, batches

    ms1, results, launches, clk, batches = timed(1)
    out = {"ms_single": ms1, "value_single": world * B * steps / (ms1 / 1e3), "ms": ms1,
           "results": results, "launches": launches, "clocks": clk, "batches": batches}
    if n_streams > 1:
        ms, results, launches, clk, batches = timed(n_streams)
        out.update(ms=ms, results=results, launches=launches, clocks=clk, batches=batches)
    out["value"] = world * B * steps / (out["ms"] / 1e3)
    return out


def e2e_translate(model, vocabs, restriction, B, K, L, alpha, steps, n_streams, seed0=500):
    """The public API end to end: translate() over all the step batches'
    sentences at once (host strings in, TranslationRecords out; H2D of the
    inputs and D2H of the results inside the timed region)."""
    import torch
    import torch.distributed as dist
    from paper_2207_05851_b200 import engine as _eng
    from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
    world, rank, _ = _env()
    V = model.config.trg_vocab_size

    def sents(step):
        return synth_sentences(B, L, V, seed=13 + 7919 * rank + 104729 * step)

    settings = SearchSettings(beam=K, length_alpha=alpha, restriction=restriction)
    host_inputs = [[SentenceInput(tokens=s) for s in sents(seed0 + s)] for s in range(steps)]
    _eng.DECODE_STREAMS = n_streams
    # warm-up: one untimed translate() of the timed call's size (other
    # sentences), so the timed passes see the steady state (every decode
    # stream's workspace, pinned staging and allocator blocks in place; the
    # first full-size call otherwise measured ~half speed, r2_150)
    nw = int(os.environ.get("SKB_E2E_WARM_BATCHES", str(steps)))
    warm = [SentenceInput(tokens=s) for w in range(nw) for s in sents(900 + w)] or \
        [SentenceInput(tokens=s) for s in sents(900)[:8]]
    translate(model, vocabs, warm, settings, max_rows=B * K)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    flat = sum(host_inputs, [])
    per_call = int(os.environ.get("SKB_E2E_CALL_SENTS", "0")) or len(flat)
    groups = [flat[g:g + per_call] for g in range(0, len(flat), per_call)]
    # REPS timed passes over the same host inputs (each one complete: H2D,
    # decode, D2H, records); the median is reported, every pass listed — a
    # single pass of ~0.2 s varies with the device's power-capped clocks
    reps = max(1, int(os.environ.get("SKB_E2E_REPS", "3")))
    s0 = dict(_eng.STATS)
    samples = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for inp in groups:
            recs = translate(model, vocabs, inp, settings, max_rows=B * K)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        samples.append(float(t.item()))
    misses = {k: _eng.STATS[k] - s0[k] for k in s0}
    e2e_ms = statistics.median(samples)
    S = 2 * L + 10
    h2d = B * L * 4 + B * 4 * 4 + B * 8          # ids, lengths/limits/prefix, step tables
    d2h = B * S * 4 + B * (8 + 4 + 4) + B * S * 4  # tokens, best score/steps/forced, factors
    assert len(recs) == len(groups[-1]) and all(r.error is None for r in recs)
    return {"value": round(world * B * steps / (e2e_ms / 1e3), 2), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "paper_2207_05851_b200.search.translate",
            "passes_sentences_per_s": [round(world * B * steps / (m / 1e3), 2) for m in samples],
            "cache_misses_in_timed_call": misses}


def workload_name(name, K, alpha, B, L):
    desc = MODELS[name][1]
    search = "greedy" if K == 1 else f"beam {K} alpha {alpha}"
    return f"{desc} {search}, batch {B} sentences/GPU, src len {L}, {2 * L + 10}-step cap"


def latency_model_batch1(name, L=30, which=(("greedy", 1), ("beam5", 5))):
    """batch1_latency on Model(gemm_split="latency") of config `name`."""
    import gc
    import torch
    from paper_2207_05851_b200 import engine
    m, v, rs = build_model(name, gemm_split="latency")
    out = batch1_latency(m, v, L, m.config.trg_vocab_size, restriction=rs, which=which)
    out["gemm_split"] = "latency"
    del m, v, rs
    engine.clear_workspaces()
    gc.collect()
    torch.cuda.empty_cache()
    return out


def secondary_configs(args, peaks):
    """The other BASELINE.json configs, measured in the same run (rank 0,
    N=1): base 6-6 beam 5 batch 64; big 20-2 SSRU + top-200 shortlist greedy
    and beam 5; the latency sweep's batch-256 beam-5 point; batch-1 greedy
    latency of big 6-6 vs big 20-2 vs big 20-2 SSRU (the reference's
    acceptance ordering, tests/test_acceptance.py:466-490)."""
    import gc
    import torch
    from paper_2207_05851_b200 import engine
    L, alpha = args.src_len, args.alpha
    hbm = peaks.get("hbm_gbs", 6466.1)
    tf_s = peaks.get("bf16_tflops_sustained", 1422.5)
    out = {}

    def one(key, name, B, K, streams, steps, model=None, vocabs=None, restriction=None):
        own = model is None
        if own:
            model, vocabs, restriction = build_model(name)
        r = measure(model, vocabs, restriction, B, K, L, alpha, steps, 2, streams, seed0=31)
        bb = r["batches"][-1]
        U = bb.ws.U if hasattr(bb.ws, "U") else None
        fl = ideal_floor(model, B, K, L, 2 * L + 10, tf_s, hbm, U=U,
                         distinct=distinct_kv_entries(bb, 2 * L + 10))
        fl["frac"] = round(r["value"] / fl["sentences_per_s"], 4)
        out[key] = {"workload": workload_name(name, K, alpha, B, L), "value": round(r["value"], 2),
                    "unit": UNIT, "streams": streams, "value_single_stream": round(r["value_single"], 2),
                    "ms_per_batch_single_stream": round(r["ms_single"] / steps, 3),
                    "floor": fl, "gpu_launches": r["launches"],
                    "mean_steps": round(statistics.mean(x.steps for res in r["results"] for x in res), 2)}
        if U is not None:
            out[key]["union_columns"] = int(U)
        if own:
            del model, r, bb
            engine.clear_workspaces()
            gc.collect()
            torch.cuda.empty_cache()

    nb = max(6, 2 * args.streams)  # batches per secondary config: the stream pipeline fills
    one("base_beam5_b64", "base", 64, 5, args.streams, nb)
    m, v, rs = build_model("big_ssru")
    one("big_ssru_sl200_beam5_b128", "big_ssru", 128, 5, args.streams, nb, m, v, rs)
    one("big_ssru_sl200_greedy_b128", "big_ssru", 128, 1, args.streams, nb, m, v, rs)
    del m, v, rs
    engine.clear_workspaces()
    gc.collect()
    torch.cuda.empty_cache()
    # batch-1 latency by architecture, latency-configured models
    lat = {"big_ssru_sl200": latency_model_batch1("big_ssru", L),
           "big_ssru": latency_model_batch1("big_ssru_nosl", L, which=(("greedy", 1),)),
           "big_20_2": latency_model_batch1("big_20_2", L, which=(("greedy", 1),))}
    out["batch1_latency_by_architecture"] = lat
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2207_05851_b200 import engine, kern

    world, rank, local = _env()
    torch.cuda.set_device(local)
    from paper_2207_05851_b200 import _native as N
    N.call("skb_set_device", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak_tf = peaks.get("bf16_tflops", 1590.0)
    peak_src = "measured (MEASURED_PEAKS.json bf16_tflops, burst)" if peaks else "fallback"
    hbm = peaks.get("hbm_gbs", 6466.1)

    name = args.config
    model, vocabs, restriction = build_model(name, gemm_split=args.gemm_split)
    V = model.config.trg_vocab_size
    B = args.batch or DEFAULT_BATCH[name]
    K, L = args.beam, args.src_len

    def gather(bb):
        if world > 1:
            toks = bb.tokens_out
            out = [torch.empty_like(toks) for _ in range(world)] if rank == 0 else None
            dist.gather(toks, out, dst=0)

    n_streams = max(1, args.streams)
    r = measure(model, vocabs, restriction, B, K, L, args.alpha, args.steps, args.warmup, n_streams,
                gather=gather, clocks_device=local)
    value, ms_step = r["value"], r["ms"] / args.steps
    results, launches, clk, batches = r["results"], r["launches"], r["clocks"], r["batches"]
    forced = sum(x.forced_eos for res in results for x in res)
    steps_per_sent = statistics.mean(x.steps for res in results for x in res)
    bb = batches[-1]
    S = 2 * L + 10
    distinct = distinct_kv_entries(bb, S)
    U = bb.ws.U

    e2e = None if args.no_e2e else e2e_translate(model, vocabs, restriction, B, K, L, args.alpha,
                                                 args.steps, n_streams)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    lat = None
    if not args.no_e2e:
        # batch-1 latency on the latency-configured model (same weights, every
        # projection split into short K-partials: Model(gemm_split="latency"));
        # the serving model's own batch-1 numbers beside it
        lat = latency_model_batch1(args.config)
        lat["throughput_model"] = batch1_latency(model, vocabs, L, V, restriction=restriction)
    roof = gemm_roofline(model, B * K, L, peak_tf, U=U)
    roof["peak_source"] = peak_src
    breakdown = step_breakdown(bb)
    topk = topk_roofline(bb, hbm)
    topk["peak_source"] = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks else "fallback"
    attn_roof = attention_roofline(bb, model, hbm)
    floor = ideal_floor(model, B, K, L, S, peaks.get("bf16_tflops_sustained", 1422.5), hbm, U=U,
                        distinct=distinct)
    floor["frac"] = round(value / world / floor["sentences_per_s"], 4)
    # the same FLOP count over the headline's own wall time: every decode
    # GEMM / attention FLOP of the served batches (all streams overlapping)
    # divided by the measured per-GPU time, against the sustained peak
    agg = floor["gflop_per_sentence"] * 1e9 * value / world / 1e12
    peak_sus = peaks.get("bf16_tflops_sustained", 1422.5)
    roof["pipeline"] = {"achieved": round(agg, 1), "peak": peak_sus, "unit": "TFLOP/s",
                        "frac": round(agg / peak_sus, 4),
                        "note": "reference cost-model FLOPs per sentence x headline sentences/s per GPU "
                                "(all streams) / sustained bf16 peak"}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (uniform random source ids, random-init weights seed 13)",
        "config": {"workload": workload_name(name, K, args.alpha, B, L),
                   "global_batch": B * world, "seq_len": L, "parallelism": f"replicas x{world}",
                   "streams_per_gpu": n_streams, "batch_per_stream": B,
                   "value_single_stream": round(r["value_single"], 2),
                   "ms_per_batch_single_stream": round(r["ms_single"] / args.steps, 3),
                   "union_columns": int(U),
                   "l2": "working set > L2 (weights 0.48 GB + KV cache 1.1 GB per batch)"},
        "e2e": e2e, "batch1_latency": lat, "roofline": roof, "roofline_topk": topk, "roofline_attention": attn_roof,
        "floor": floor, "gpu_launches": launches,
        "clocks": clk,
        "decode": {"mean_steps_per_sentence": round(steps_per_sent, 2),
                   "forced_eos_sentences": forced, "step_breakdown_ms": breakdown,
                   "distinct_kv_entries_per_step_mean": round(statistics.mean(distinct), 1),
                   "per_row_kv_entries_per_step_mean": round(
                       statistics.mean(B * K * (t + 1) for t in range(S)), 1)},
    }
    if world == 1 and not args.no_secondary and name == "big":
        del bb, batches, results, r
        engine.clear_workspaces()
        line["configs"] = secondary_configs(args, peaks)
        line["configs"]["big_beam5_b256_single_stream"] = None
        m256 = measure(model, vocabs, None, 256, K, L, args.alpha, 4, 2, 1, seed0=77)
        line["configs"]["big_beam5_b256_single_stream"] = {
            "workload": workload_name("big", K, args.alpha, 256, L),
            "value": round(m256["value"], 2), "unit": UNIT,
            "ms_per_batch": round(m256["ms"] / 4, 3)}
        lat_arch = line["configs"]["batch1_latency_by_architecture"]
        if lat:
            lat_arch["big_6_6"] = {"greedy": lat["greedy"]}
            g = {k: v["greedy"]["p50_ms"] for k, v in lat_arch.items() if isinstance(v, dict)}
            # tests/test_acceptance.py:466-490: recurrent 20:2 >= deep 20:2 >
            # balanced 6:6 in speed (all unrestricted)
            lat_arch["ordering_ssru_20_2_le_20_2_lt_6_6"] = bool(
                g["big_ssru"] <= g["big_20_2"] < g["big_6_6"])
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args, L, K, name=name)
        if name == "big" and not args.no_secondary:
            line["cpu_baseline"]["batch1_greedy_latency"] = cpu_batch1_latency(args, L)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _host_info():
    model = "unknown"
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem_gb = None
    try:
        for ln in Path("/proc/meminfo").read_text().splitlines():
            if ln.startswith("MemTotal"):
                mem_gb = round(int(ln.split()[1]) / 1024 ** 2, 1)
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gb": mem_gb}


def cpu_baseline_leg(args, L, K, pool=None, name="big"):
    import numpy as np
    from oracle.cpu_baseline import CpuBaseline
    spec, _, topk = MODELS[name]
    own = pool is None
    pool = pool or CpuBaseline(spec, shortlist_topk=topk)
    rng = np.random.default_rng(13)
    srcs = [[int(i) + 4 for i in rng.integers(0, spec["trg_vocab_size"] - 4, size=L)]
            for _ in range(pool.procs)]
    rate, wall, det = pool.sample(srcs, K, args.alpha, args.cpu_steps)
    if own:
        pool.close()
    host = _host_info()
    return {"value": round(rate, 4), "unit": UNIT, "cores": pool.procs, "kind": "port",
            "sample": f"{pool.procs} single-thread processes x 1 sentence (L={L}, "
                      f"{'greedy' if K == 1 else f'beam {K}'}): encode + first {args.cpu_steps} of "
                      f"{2 * L + 10} steps, extrapolated linearly; "
                      f"{det['sec_per_sentence']:.1f} s/sentence/core",
            "procs_rule": "P = min(nproc, floor(RAM / 4 GB)) (SURVEY 8d)",
            "host": host, "wall_s": round(wall, 2)}


def cpu_batch1_latency(args, L, n=21, steps=2):
    """Batch-1 greedy latency of the reference algorithm on one host core
    (single-process greedy runs over >= 21 sentences): encode +
    the first `steps` greedy steps of each sentence timed, the rest of the
    2L+10 steps extrapolated from the measured per-step time; p50 over n."""
    import numpy as np
    from oracle.cpu_baseline import CpuBaseline
    pool = CpuBaseline(BIG, procs=1)
    rng = np.random.default_rng(4242)
    lat = []
    for _ in range(n):
        src = [int(i) + 4 for i in rng.integers(0, BIG["trg_vocab_size"] - 4, size=L)]
        _, _, det = pool.sample([src], 1, args.alpha, steps)
        lat.append(det["sec_per_sentence"] * 1e3)
    pool.close()
    lat.sort()
    return {"p50_ms": round(statistics.median(lat), 1), "p90_ms": round(lat[int(0.9 * (n - 1))], 1),
            "sentences": n, "cores": 1, "kind": "port",
            "sample": f"encode + first {steps} of {2 * L + 10} greedy steps per sentence, "
                      "extrapolated; big 6-6, L=%d" % L}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuBaseline
    name = args.config
    spec, _, topk = MODELS[name]
    pool = CpuBaseline(spec, shortlist_topk=topk)
    L, K = args.src_len, args.beam
    for _ in range(args.warmup):
        cpu_baseline_leg(args, L, K, pool, name=name)
    vals, walls = [], []
    for _ in range(args.steps):
        r = cpu_baseline_leg(args, L, K, pool, name=name)
        vals.append(r["value"])
        walls.append(r["wall_s"])
    pool.close()
    value = statistics.mean(vals)
    B = args.batch or DEFAULT_BATCH[name]
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.mean(walls), 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
            "data": "synthetic", "config": {"workload": workload_name(name, K, args.alpha, B, L)},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": pool.procs,
                             "kind": "port", "host": _host_info(),
                             "sample": f"per step: {pool.procs} processes x 1 sentence, encode + "
                                       f"{args.cpu_steps} of {2 * L + 10} steps, extrapolated"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
