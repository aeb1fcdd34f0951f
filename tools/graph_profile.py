"""Kernel durations INSIDE the captured decode graphs (CUPTI via
torch.profiler), i.e. with PDL overlap and warm caches as in bench.py —
unlike the ncu launch list, which serialises and flushes caches.

    python tools/graph_profile.py > gpurun_out/graph_profile.txt
"""
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

import os
B = int(os.environ.get("BATCH", "128"))
K = int(os.environ.get("BEAM", "5"))
model, vocabs, rs = bench.build_model(os.environ.get("CONFIG", "big"),
                                     gemm_split=os.environ.get("GEMM_SPLIT", "throughput"))
sents = bench.synth_sentences(B, 30, 32000, seed=13)
bb = bench.make_batch(model, vocabs, sents, K, 1.0, restriction=rs)
for _ in range(2):
    bb.run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bb.run()
    torch.cuda.synchronize()
evs = []
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    evs.append((ev.time_range.start, ev.time_range.end, ev.name.split("(")[0][:60]))
evs.sort()
# Kernels of one stream run in order; with PDL a kernel starts early and waits
# in griddepcontrol.wait, so its own duration overlaps its predecessor.  The
# critical-path cost of kernel i is end_i - end_{i-1} (what the step would
# lose without it); the inclusive duration is shown beside it.
tot = defaultdict(float)
incl = defaultdict(float)
cnt = defaultdict(int)
prev_end = evs[0][0]
for s0, e0, name in evs:
    tot[name] += max(0.0, e0 - prev_end)
    incl[name] += e0 - s0
    cnt[name] += 1
    prev_end = max(prev_end, e0)
wall = evs[-1][1] - evs[0][0]
print(f"wall (first kernel start -> last end): {wall / 1e3:.3f} ms over {len(evs)} kernels")
print(f"{'kernel':60s} {'n':>6s} {'crit ms':>8s} {'crit us':>8s} {'incl us':>8s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:60s} {cnt[k]:6d} {v / 1e3:8.3f} {v / cnt[k]:8.2f} {incl[k] / cnt[k]:8.2f} "
          f"{100 * v / wall:5.1f}%")
if os.environ.get("GAPS"):
    # idle gaps on the device timeline (next kernel start - max end so far) > 2 us
    prev_end = evs[0][1]
    gaps = []
    for s0, e0, name in evs[1:]:
        if s0 - prev_end > 2.0:
            gaps.append((round(s0 - prev_end, 1), name))
        prev_end = max(prev_end, e0)
    print(f"idle gaps > 2 us: {len(gaps)}, total {sum(g for g, _ in gaps) / 1e3:.3f} ms")
    for g, n in gaps[:40]:
        print(f"   {g:8.1f} us before {n}")
