"""Time the tcgen05 GEMM on the decode-step shapes (CUDA events), with the
split-K workspace.  Env SKB_GEMM_BN / SKB_GEMM_SPLITS force a config."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 640
SHAPES = {"qkv": (M, 3072, 1024), "wo": (M, 1024, 1024), "ffn1": (M, 4096, 1024),
          "ffn2": (M, 1024, 4096), "out_proj": (M, 32000, 1024)}
ws = torch.empty(8 << 20, device="cuda")
cnt = torch.zeros(8192, dtype=torch.int32, device="cuda")
res = {}
for name, (m, Nn, K) in SHAPES.items():
    A = torch.randn(m, K, device="cuda").bfloat16()
    W = torch.randn(Nn, K, device="cuda").bfloat16()
    out = torch.zeros(m, Nn, device="cuda")
    epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None, 0,
                     None, 0, None, 0, 1, ws.data_ptr(), ws.numel(), cnt.data_ptr(), cnt.numel())
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.call("skb_gemm", N.BF16, m, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi), st)
    try:
        for _ in range(3):
            run()
    except Exception as e:  # noqa: BLE001
        print(name, "skip", e)
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 30
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    err = (out - A.float() @ W.float().T).abs().max().item()
    res[name] = dict(us=round(ms * 1e3, 2), tflops=round(2 * m * Nn * K / ms / 1e9, 1),
                     err=round(err, 4))
print(json.dumps({"BN": os.environ.get("SKB_GEMM_BN", "auto"),
                  "CS": os.environ.get("SKB_GEMM_CS", "auto"),
                  "S": os.environ.get("SKB_GEMM_SPLITS", "auto"), **res}))
