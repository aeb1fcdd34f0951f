"""Host-side profile of batch-1 translate() calls (latency model; optional
shortlist): where the wall time goes around the GPU work.

    python tools/b1_prof.py [big|big_ssru|...] [beam]
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "big_ssru"
beam = int(sys.argv[2]) if len(sys.argv) > 2 else 1
model, vocabs, rs = bench.build_model(name, gemm_split="latency")
sents = bench.synth_sentences(12, 30, model.config.trg_vocab_size, seed=4242)
st = SearchSettings(beam=beam, restriction=rs)
for s in sents[:2]:
    translate(model, vocabs, [SentenceInput(tokens=s)], st)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for s in sents[2:]:
    translate(model, vocabs, [SentenceInput(tokens=s)], st)
pr.disable()
print(f"{name} beam {beam}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per call")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
