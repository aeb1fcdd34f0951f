"""Host-side profile of translate() over the e2e workload (9 x 128 sentences,
beam 5, 3 decode streams): where the Python time goes around the GPU work."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_05851_b200 import engine  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

model, vocabs, _ = bench.build_model("big")
inputs = [SentenceInput(tokens=s) for k in range(9) for s in bench.synth_sentences(128, 30, 32000, seed=500 + k)]
settings = SearchSettings(beam=5, length_alpha=1.0)
engine.DECODE_STREAMS = 5
translate(model, vocabs, inputs, settings, max_rows=640)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
recs = translate(model, vocabs, inputs, settings, max_rows=640)
torch.cuda.synchronize()
pr.disable()
print(f"translate: {time.perf_counter() - t0:.3f} s for {len(inputs)} sentences")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
