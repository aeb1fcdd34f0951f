import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2207_05851_b200 import _native as N, kern, engine
model, vocabs = bench.build_model("bf16")
sents = bench.synth_sentences(128, 30, 32000, seed=13)
bb = bench.make_batch(model, vocabs, sents, 5, 1.0)
bb.use_graph = False
bb.run()
torch.cuda.synchronize()
# replay one mid step eagerly
sb = bb.sb
sb.step.fill_(35); bb.done.zero_(); bb.n_alive.fill_(5); bb.n_done.zero_()
engine.step_forward(model, sb)
torch.cuda.synchronize()
for rep in range(2):
    bb.done.zero_(); bb.n_alive.fill_(5)
    torch.cuda.synchronize()
    kern.beam_step(sb.logits, bb.state)
    torch.cuda.synchronize()
buf = (C.c_ulonglong * (1024 * 10))()
N.lib().skb_debug_beam_prof(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 10)[:640].astype(np.int64)
t0 = a[:, 0].min()
rel = (a - t0) / 1000.0
for k in range(8):
    col = rel[:, k][a[:, k] > 0]
    if len(col): print(f"phase {k}: n={len(col):4d} min={col.min():8.2f} med={np.median(col):8.2f} max={col.max():8.2f} us")
d = rel[:, 1:5] - rel[:, 0:4]
print("per-row phase durations median us:", np.median(d, 0), "max:", d.max(0))
