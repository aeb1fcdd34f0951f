"""Quick correctness probe of the persistent CTA-pair GEMM on a few shapes."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

for (M, Nn, K, na) in [(64, 256, 64, 32), (640, 3072, 1024, 0), (640, 32000, 1024, 0), (5, 1000, 256, 0)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(Nn, K, device="cuda") * 0.05).bfloat16()
    out = torch.zeros(M, Nn, device="cuda")
    e = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.F32, None, None, None, 0)
    N.call("skb_gemm_force_pc", 2, na, 0)
    N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(e),
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.double() @ W.double().T
    print(M, Nn, K, na, "maxerr", (out.double() - ref).abs().max().item(), flush=True)
