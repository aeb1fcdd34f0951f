"""Host-side timeline of one batch-1 translate() call (perf_counter marks in
BeamBatch / DecodeWorkspace via SKB_HOST_TRACE=1) next to the device time."""
import os
import sys
import time

os.environ["SKB_HOST_TRACE"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_05851_b200 import engine  # noqa: E402
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "big"
m, v, rs = bench.build_model(name, gemm_split="latency")
sents = bench.synth_sentences(6, 30, m.config.trg_vocab_size, seed=4)
st = SearchSettings(beam=1, restriction=rs)
for s in sents[:3]:
    translate(m, v, [SentenceInput(tokens=s)], st)
torch.cuda.synchronize()
engine.HOST_MARKS.clear()
t0 = time.perf_counter()
translate(m, v, [SentenceInput(tokens=sents[4])], st)
t1 = time.perf_counter()
for label, t in engine.HOST_MARKS:
    print(f"{(t - t0) * 1e3:8.3f} ms  {label}")
print(f"{(t1 - t0) * 1e3:8.3f} ms  translate returned")
