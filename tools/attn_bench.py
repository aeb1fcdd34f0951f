"""Decoder self-attention kernel alone on the benchmark shape (R = 640 rows =
128 sentences x beam 5, H 16, d_h 64, S_max 70), six layer caches (cold
working set as in the decode graph), a realistic beam-tree ancestor table.

    python tools/attn_bench.py          # env SKB_ATTN_PF selects the variant
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import kern  # noqa: E402

import os
B, K = int(os.environ.get("B", "128")), int(os.environ.get("K", "5"))
H, dh, S = 16, 64, 70
R, D = B * K, H * dh
dev = "cuda"
rng = np.random.default_rng(0)
# beam tree: at each step every row picks a parent in its sentence, skewed
anc_np = np.zeros((R, S), dtype=np.int32)
hist = np.tile(np.arange(R, dtype=np.int32)[:, None], (1, S))
for p in range(1, S):
    par = np.minimum(rng.geometric(0.55, size=R) - 1, K - 1)
    rows = (np.arange(R) // K) * K + par
    hist[:, :p] = hist[rows, :p]
anc_np[:] = hist
anc = torch.zeros(2, R, S, dtype=torch.int32, device=dev)
anc[0] = torch.from_numpy(anc_np).to(dev)
anc[1] = anc[0]
qkv = torch.randn(R, 3 * D, device=dev).bfloat16()
caches = [(torch.randn(R, S, D, device=dev).bfloat16(), torch.randn(R, S, D, device=dev).bfloat16())
          for _ in range(6)]
ctx = torch.empty(R, D, device=dev, dtype=torch.bfloat16)
uniq = np.mean([len(set(zip(anc_np[b * K:(b + 1) * K, :36].ravel(), np.tile(np.arange(36), K))))
                / (K * 36) for b in range(B)])
import os
for t in [int(x) for x in os.environ.get('TS', '10,35,60').split(',')]:
    step = torch.tensor([t], dtype=torch.int32, device=dev)

    plan = None
    if os.environ.get("PLAN", "1") == "1":  # the engine's path: one step plan for all layers
        plan = torch.empty(kern.attn_plan_bytes(R, K, S), dtype=torch.uint8, device=dev)
        kern.attn_plan(anc, step, plan, R, S, K)

    def run():
        for kc, vc in caches:
            kern.self_attention_step(qkv, kc, vc, anc, step, ctx, R, H, dh, S, group=K, plan=plan)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 6)
    rows_bytes = R * H * (t + 1) * dh * 2 * 2
    print(f"t={t:2d}: {best * 1e3:6.2f} us/layer  all-row K/V bytes {rows_bytes / 1e6:.1f} MB "
          f"({rows_bytes / best / 1e9:.0f} GB/s); unique fraction at t=35 ~{uniq:.2f}")
