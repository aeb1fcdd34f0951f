"""Run-to-run variance of the e2e translate() measurement: the bench's
device-resident warm-up, then the e2e call several times in one process,
with the workspace / graph-capture cache misses of each call and (with
SKB_HOST_TRACE=1) the largest host-side gaps between engine marks."""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_05851_b200 import engine  # noqa: E402

model, vocabs, rs = bench.build_model("big")
r = bench.measure(model, vocabs, rs, 128, 5, 30, 1.0, 9, 3, 5)
print("value", round(r["value"], 1), "stats after measure", dict(engine.STATS), flush=True)
for i in range(int(os.environ.get("REPS", "4"))):
    s0 = dict(engine.STATS)
    engine.HOST_MARKS.clear()
    t0 = time.perf_counter()
    nb = int(os.environ.get("NB", "9"))  # batches of 128 sentences in the call
    e = bench.e2e_translate(model, vocabs, rs, 128, 5, 30, 1.0, nb, 5, seed0=500 + 10 * i)
    dt = time.perf_counter() - t0
    gaps = sorted(((b[1] - a[1]) * 1e3, a[0], b[0]) for a, b in zip(engine.HOST_MARKS, engine.HOST_MARKS[1:]))[-3:]
    print(i, "e2e", e["value"], "wall %.3f s" % dt, {k: engine.STATS[k] - s0[k] for k in s0},
          [(round(g, 1), x, y) for g, x, y in gaps], flush=True)
    if os.environ.get("DUMP") and engine.HOST_MARKS:
        m0 = engine.HOST_MARKS[0][1]
        print("   marks (ms):", " | ".join(f"{(t - m0) * 1e3:.1f} {lab}" for lab, t in engine.HOST_MARKS))
