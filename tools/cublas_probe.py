"""Run cuBLAS (torch.matmul bf16) and our tcgen05 GEMM once per decode-step
shape, for an ncu capture that compares kernel choice, grid and counters."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 640
which = sys.argv[2] if len(sys.argv) > 2 else "both"
SHAPES = {"qkv": (3072, 1024), "wo": (1024, 1024), "ffn1": (4096, 1024), "ffn2": (1024, 4096),
          "out_proj": (32000, 1024)}
for name, (Nn, K) in SHAPES.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(Nn, K, device="cuda").bfloat16()
    out = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    if which in ("both", "cublas"):
        for _ in range(2):
            torch.matmul(A, W.T, out=out)
    if which in ("both", "ours"):
        epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.BF16, None, None, None, 0, None,
                         0, None, 0, None, 0, 1, None, 0, None, 0)
        for _ in range(2):
            N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
print("done")
