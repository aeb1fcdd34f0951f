"""Launch the SSRU-epilogue GEMM a few times at the bench shape (M = 640,
N = 2048 interleaved [W_f; W], K = 1024, decode-loop double buffer at step 5)
for an ncu capture of its source page.
    ncu --set full --import-source on -k regex:k_gemm_sw -s 2 -c 1 -o out python tools/ssru_one.py"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M, Nn, K = int(sys.argv[1]) if len(sys.argv) > 1 else 640, 2048, 1024
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(Nn, K, device="cuda") * 0.05).bfloat16()
x = torch.zeros(M, Nn // 2, device="cuda")
cell = torch.randn(2, M, Nn // 2, device="cuda")
rows = torch.randperm(M, device="cuda").int()
stp = torch.tensor([5], dtype=torch.int32, device="cuda")
epi = N.Epilogue(N.EPI_SSRU, None, x.data_ptr(), Nn // 2, N.F32, None, cell.data_ptr(), rows.data_ptr(),
                 Nn // 2, stp.data_ptr(), M * (Nn // 2))
for _ in range(4):
    N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
           torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
