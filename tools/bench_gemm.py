"""Time the tcgen05 GEMM on the decode-step shapes (CUDA events).
Run with SKB_GEMM_BN=64|128|256 to force a tile width."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 640
SHAPES = {"qkv": (M, 3072, 1024), "wo": (M, 1024, 1024), "ffn1": (M, 4096, 1024),
          "ffn2": (M, 1024, 4096), "out_proj": (M, 32000, 1024), "big": (8192, 8192, 8192)}
res = {}
for name, (m, Nn, K) in SHAPES.items():
    A = torch.randn(m, K, device="cuda").bfloat16()
    W = torch.randn(Nn, K, device="cuda").bfloat16()
    out = torch.zeros(m, Nn, device="cuda")
    epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.F32)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.call("skb_gemm", N.BF16, m, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi), st)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (A.float() @ W.float().T)
    err = (out - ref).abs().max().item()
    res[name] = dict(ms=round(ms, 4), tflops=round(2 * m * Nn * K / ms / 1e9, 1), err=err)
    print(name, json.dumps(res[name]), flush=True)
