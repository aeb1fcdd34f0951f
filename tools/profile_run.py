"""Short eager run of the bench workload for ncu (one batch, no graph).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_run.py
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--beam", type=int, default=5)
ap.add_argument("--src-len", type=int, default=30)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--gemm-split", default="throughput", choices=["throughput", "latency"])
a = ap.parse_args()
model, vocabs, _ = bench.build_model("big", gemm_split=a.gemm_split)
sents = bench.synth_sentences(a.batch, a.src_len, 32000, seed=13)
bb = bench.make_batch(model, vocabs, sents, a.beam, 1.0)
bb.use_graph = a.graph
bb.run()
torch.cuda.synchronize()
print("profiled batch done", bb.steps_run, "steps")
