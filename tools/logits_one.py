"""Launch the LOGITS-epilogue output projection a few times at the bench
shape (M = 640, N = 32000, K = 1024) for an ncu capture of its source page.
    ncu --set full --import-source on -k regex:k_gemm_sw -s 2 -c 1 -o out python tools/logits_one.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M, Nn, K = int(sys.argv[1]) if len(sys.argv) > 1 else 640, 32000, 1024
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(Nn, K, device="cuda") * 0.05).bfloat16()
out = torch.zeros(M, Nn, device="cuda")
part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda")
epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None,
                 0, part.data_ptr(), part.shape[1] // 2, None, 0, 1)
for _ in range(4):
    N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
           torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
