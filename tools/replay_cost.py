import sys, time
sys.path.insert(0, '.')
import torch, bench
from paper_2207_05851_b200.search import SearchSettings, SentenceInput, translate
m, v, rs = bench.build_model("big", gemm_split="latency")
sents = bench.synth_sentences(4, 30, 32000, seed=1)
st = SearchSettings(beam=1)
for s in sents[:2]:
    translate(m, v, [SentenceInput(tokens=s)], st)
torch.cuda.synchronize()
from paper_2207_05851_b200 import engine
print("workspaces:", len(engine._WS_CACHE))
for key, w in [kv for per in engine._WS_CACHE.values() for kv in per.items()]:
    for name in ("graph_enc", "graph_1", "graph_n"):
        g = getattr(w, name, None)
        if g is None: continue
        torch.cuda.synchronize()
        t = time.perf_counter(); g.replay(); dt = time.perf_counter() - t
        torch.cuda.synchronize()
        t2 = time.perf_counter(); g.replay(); dt2 = time.perf_counter() - t2
        torch.cuda.synchronize()
        print(name, "host replay us: %.1f %.1f" % (dt * 1e6, dt2 * 1e6), "launches", getattr(w, "launches_" + name.split("_")[1], None))
