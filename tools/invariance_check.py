"""Batch-composition invariance end to end: translate() a mixed-length batch
(default max_rows -> R = 2560 rows per device batch, several streams), then
re-translate a sample of those sentences one at a time (R = beam: the
prologue-LayerNorm GEMMs, one stream) and require identical tokens and
scores (test_search.py:400-405 on the device path, at scale)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

model, vocabs, _ = bench.build_model("big")
rng = np.random.default_rng(5)
sents = [[f"w{i}" for i in rng.integers(0, 31996, size=int(n))] for n in rng.integers(1, 121, size=600)]
settings = SearchSettings(beam=5, length_alpha=1.0)
big = translate(model, vocabs, [SentenceInput(tokens=s) for s in sents], settings)
bad = 0
for i in list(range(0, 600, 37)):
    one = translate(model, vocabs, [SentenceInput(tokens=sents[i])], settings)[0]
    if one.text != big[i].text or one.score != big[i].score:
        bad += 1
        print("MISMATCH", i, len(sents[i]), one.score, big[i].score)
print(f"checked {len(range(0, 600, 37))} sentences, mismatches {bad}")
torch.cuda.synchronize()
