"""Which batch property changes a sentence's score?  Same sentence alone,
with same-length neighbours (decode M changes), with a longer neighbour
(source padding L changes), and with many neighbours (M > 1024)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

model, vocabs, _ = bench.build_model("big")
rng = np.random.default_rng(5)
mk = lambda n: [f"w{i}" for i in rng.integers(0, 31996, size=n)]  # noqa: E731
s = mk(25)
same = [mk(25) for _ in range(4)]
longer = [mk(120)]
many = [mk(25) for _ in range(300)]
st = SearchSettings(beam=5, length_alpha=1.0)


def score(batch, **kw):
    return translate(model, vocabs, [SentenceInput(tokens=x) for x in batch], st, **kw)[0].score


print("alone             ", score([s]))
print("alone again       ", score([s]))
print("+4 same length    ", score([s] + same))
print("+1 longer (L=120) ", score([s] + longer))
print("+300 same length  ", score([s] + many))
print("+300, max_rows 640", score([s] + many, max_rows=640))
