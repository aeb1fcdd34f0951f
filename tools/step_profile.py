"""Label an ncu launch list of tools/profile_run.py by decoder-step op.

Eager step order (engine.step_forward + beam): embed, 6 x [LN, QKV, self-attn,
Wo, LN, Qc, cross-attn, Woc, LN, FFN1, FFN2], LN, out-proj, beam, reorder,
advance.  Prints mean device time per op over the captured steps.
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
seq = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr + 1:]
       if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
layer = ["ln_self", "qkv", "self_attn", "wo", "ln_cross", "q_cross", "cross_attn", "wo_cross",
         "ln_ffn", "ffn1", "ffn2"]
ops = ["embed"] + [f"L{i}.{o}" for i in range(6) for o in layer] + ["ln_final", "out_proj",
                                                                      "beam_step", "reorder",
                                                                      "advance"]
# find step starts: k_embed_target
starts = [i for i, (n, _) in enumerate(seq) if "k_embed_target" in n]
tot = defaultdict(list)
for s in starts:
    chunk = seq[s:s + len(ops)]
    if len(chunk) < len(ops):
        break
    for op, (n, t) in zip(ops, chunk):
        tot[op.split(".")[-1]].append(t)
steps = len(tot["embed"])
print(f"steps profiled: {steps}")
allt = 0.0
agg = {}
for op, ts in tot.items():
    per_step = sum(ts) / steps
    agg[op] = per_step
    allt += per_step
for op, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    n = len(tot[op]) // steps
    print(f"{op:12s} {n:3d}/step {v / 1e3:9.1f} us/step  {v / n / 1e3:8.2f} us each  {100 * v / allt:5.1f}%")
print(f"{'TOTAL':12s} {allt / 1e3:9.1f} us/step (serialised, cold-ish caches)")
