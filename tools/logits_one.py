"""One decode-step output projection (M=640 rows x 32000 columns x 1024, the
LOGITS epilogue) launched a few times — for ncu.  CAND=1: candidate mode."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M, Nn, K = int(os.environ.get("M", "640")), 32000, 1024
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(Nn, K, device="cuda") * 0.05).bfloat16()
out = torch.zeros(M, Nn, device="cuda")
part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda")
epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None, 0,
                 part.data_ptr(), part.shape[1] // 2, None, 0, 5)
if os.environ.get("CAND"):
    cand = torch.zeros(M, ((Nn + 127) // 128) * 12, device="cuda")
    fs = torch.zeros(1, dtype=torch.int32, device="cuda")
    fp = torch.zeros(M // 5 + 1, dtype=torch.int32, device="cuda")
    fm = torch.full((M // 5 + 1,), 70, dtype=torch.int32, device="cuda")
    epi.cand, epi.cand_ld, epi.cand_k = cand.data_ptr(), (Nn + 127) // 128, 5
    epi.force_step, epi.force_prefix_len, epi.force_max_len = fs.data_ptr(), fp.data_ptr(), fm.data_ptr()
for _ in range(int(os.environ.get("REPS", "3"))):
    N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
           torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
