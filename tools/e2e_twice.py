"""translate() over the e2e workload twice in a row (fresh workspaces, then
reused ones): device-timed, to compare the two paths."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_05851_b200 import engine  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

model, vocabs, _ = bench.build_model("big")
settings = SearchSettings(beam=5, length_alpha=1.0)
engine.DECODE_STREAMS = 3
translate(model, vocabs, [SentenceInput(tokens=s) for s in bench.synth_sentences(8, 30, 32000, 1)], settings)
torch.cuda.synchronize()
for rep in range(6):
    inputs = [SentenceInput(tokens=s) for k in range(9)
              for s in bench.synth_sentences(128, 30, 32000, seed=500 + 10 * rep + k)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    translate(model, vocabs, inputs, settings, max_rows=640)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"call {rep}: {ms:.1f} ms device, {1e3 * (time.perf_counter() - t0):.1f} ms host, "
          f"{len(inputs) / ms * 1e3:.0f} sent/s, workspaces {len(engine._WS_CACHE)}")
