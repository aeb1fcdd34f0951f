"""Per-phase timing of the beam kernel (build with
SKB_NVCC_EXTRA=-DSKB_PROFILE_PHASES)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2207_05851_b200 import _native as N, kern, engine  # noqa: E402

model, vocabs, _ = bench.build_model("big")
sents = bench.synth_sentences(128, 30, 32000, seed=13)
bb = bench.make_batch(model, vocabs, sents, 5, 1.0)
bb.use_graph = False
bb.run()
torch.cuda.synchronize()
sb = bb.sb
sb.step.fill_(35)
bb.done.zero_(); bb.n_alive.fill_(5); bb.n_done.zero_()
engine.step_forward(model, sb)
torch.cuda.synchronize()
for rep in range(3):
    bb.done.zero_(); bb.n_alive.fill_(5)
    torch.cuda.synchronize()
    kern.beam_step(sb.logits, bb.state)
    torch.cuda.synchronize()
buf = (C.c_ulonglong * (4096 * 10))()
print("rc", N.lib().skb_debug_beam_prof(buf))
A = np.frombuffer(buf, dtype=np.uint64).reshape(4, 1024, 10)[:, :640].astype(np.int64)
t0 = A[0, :, 0].min()
for sw in range(4):  # warp s of each row (SUB warps per row)
    a = A[sw]
    if not (a > 0).any():
        continue
    print(f"-- warp {sw} of each row")
    rel = (a - t0) / 1000.0
    for k in range(10):
        col = rel[:, k][a[:, k] > 0]
        if len(col):
            print(f"phase {k}: n={len(col):4d} min={col.min():8.2f} med={np.median(col):8.2f} max={col.max():8.2f} us")
