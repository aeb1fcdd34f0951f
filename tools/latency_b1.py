"""Batch-1 latency of the throughput and latency GEMM-split models (same
weights), greedy and beam 5, through translate().

    python tools/latency_b1.py [big|big_ssru_sl200|...] > gpurun_out/latency_b1.txt
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "big"
splits = sys.argv[2].split(",") if len(sys.argv) > 2 else ["throughput", "latency"]
for split in splits:
    model, vocabs, rs = bench.build_model(name, gemm_split=split)
    lat = bench.batch1_latency(model, vocabs, 30, model.config.trg_vocab_size, n=11, restriction=rs)
    print(json.dumps({"config": name, "gemm_split": split, **lat}), flush=True)
    del model
