"""Time skb_beam_step alone on the benchmark batch at step 35 (CUDA events,
20 launches back to back).  SKB_LIB selects the library build."""
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2207_05851_b200 import kern, engine  # noqa: E402

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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for rep in range(5):
    bb.done.zero_(); bb.n_alive.fill_(5)
    e0.record()
    for _ in range(20):
        kern.beam_step(sb.logits, bb.state)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
print(f"beam_step {best:.2f} us  ({sys.argv[1] if len(sys.argv) > 1 else ''})")
