"""Launch one swap-AB GEMM shape/config a few times (for ncu captures).
    python tools/gemm_one.py NAME NA CS [M]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

shapes = {"wo": (1024, 1024), "ffn2": (1024, 4096), "qkv": (3072, 1024), "ffn1": (4096, 1024),
          "out_proj": (32000, 1024)}
name, na, cs = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
M = int(sys.argv[4]) if len(sys.argv) > 4 else 640
Nn, K = shapes[name]
A = torch.randn(M, K, device="cuda").bfloat16()
W = torch.randn(Nn, K, device="cuda").bfloat16()
out = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
import os
if os.environ.get("LOGITS"):
    out = torch.zeros(M, Nn, device="cuda")
    part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda")
    epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None, 0,
                     part.data_ptr(), part.shape[1] // 2, None, 0, 1, None, 0, None, 0)
else:
    epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.BF16, None, None, None, 0, None, 0,
                     None, 0, None, 0, 1, None, 0, None, 0)
N.call("skb_gemm_force_sw", 2 if na >= 0 else 1, max(na, 0), cs)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(3):
    if i == 2:
        torch.cuda.synchronize()
        e0.record()
    N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
           torch.cuda.current_stream().cuda_stream)
e1.record()
torch.cuda.synchronize()
print(f"{name} na={na} cs={cs} M={M} logits={bool(os.environ.get('LOGITS'))}: {e0.elapsed_time(e1) * 1e3:.1f} us")
