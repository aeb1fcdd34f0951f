"""Per-CTA phase timeline of one tensor-core self-attention launch (build
with SKB_NVCC_EXTRA=-DSKB_ATTN_TRACE).  Run like tools/attn_bench.py."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("TS", "35")
from paper_2207_05851_b200 import _native as N  # noqa: E402
import runpy  # noqa: E402

runpy.run_path("tools/attn_bench.py")  # warms and leaves the last launch traced
buf = (C.c_ulonglong * (4096 * 8))()
N.call("skb_debug_attn_trace", buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
labels = ["entry", "pdl", "sweep1", "entries+issue", "kvwrite", "staged", "attended"]
t = t[:, [0, 1, 7, 2, 6, 4, 5]]
print(f"ctas {len(t)}")
for j, lab in enumerate(labels):
    col = (t[:, j] - t0) / 1e3
    print(f"  {lab:9s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
d = (t[:, 1:7] - t[:, 0:6]) / 1e3
print("  per-CTA phase durations (median us):", dict(zip(labels[1:], np.round(np.median(d, 0), 2))))
