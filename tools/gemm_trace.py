"""Per-CTA timeline of one swap-AB GEMM launch (build with
SKB_NVCC_EXTRA=-DSKB_GEMM_TRACE).  Prints, relative to the earliest CTA
entry: entry, producer pdl-wait done, first stage landed, last MMA issued,
accumulator ready, exit — min/median/max over CTAs (us)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

import os
M = int(os.environ.get("M", "640"))
shapes = {"wo": (1024, 1024), "ffn2": (1024, 4096), "qkv": (3072, 1024), "ffn1": (4096, 1024),
          "out_proj": (32000, 1024), "ssru": (2048, 1024),
          "wide": (20480, 1024)}  # wide: with M = Na every weight tile has exactly one reader
import os
if os.environ.get("SHAPES"):
    shapes = {k: shapes[k] for k in os.environ["SHAPES"].split(",")}
cfgs = [(int(a), int(b)) for a, b in (x.split(",") for x in sys.argv[1:])] or [(0, 0)]
for name, (Nn, K) in shapes.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    ncopy = int(os.environ.get("COPIES", "0")) or (8 if Nn * K < 1e8 / 2 else 2)
    Ws = [torch.randn(Nn, K, device="cuda").bfloat16() for _ in range(ncopy)]
    if os.environ.get("RESIDLN"):
        out = torch.zeros(M, Nn, device="cuda")
        hln = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
        gain = torch.ones(Nn, device="cuda")
        lb = torch.zeros(Nn, device="cuda")
        ctr = torch.zeros(64, dtype=torch.int32, device="cuda")
        lnp = torch.zeros(M, 16, device="cuda")
        epi = N.Epilogue(N.EPI_RESID, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None,
                         0, None, 0, None, 0, 1, None, 0, None, 0, gain.data_ptr(), lb.data_ptr(),
                         1e-5, hln.data_ptr(), Nn, ctr.data_ptr())
    elif os.environ.get("SSRU"):  # SSRU cell epilogue, decode-loop double buffer at step 5
        out = torch.zeros(M, Nn // 2, device="cuda")
        cell = torch.zeros(2, M, Nn // 2, device="cuda")
        rows = torch.arange(M, dtype=torch.int32, device="cuda")
        stp = torch.tensor([5], dtype=torch.int32, device="cuda")
        epi = N.Epilogue(N.EPI_SSRU, None, out.data_ptr(), Nn // 2, N.F32, None, cell.data_ptr(),
                         rows.data_ptr(), Nn // 2, stp.data_ptr(), M * (Nn // 2))
    elif os.environ.get("LOGITS"):
        out = torch.zeros(M, Nn, device="cuda")
        part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda")
        epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None,
                         0, part.data_ptr(), part.shape[1] // 2, None, 0, 1, None, 0, None, 0)
    else:
        out = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
        epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.BF16, None, None, None, 0, None,
                         0, None, 0, None, 0, 1, None, 0, None, 0)
    if os.environ.get("LNIN"):  # input LayerNorm (prologue at small M)
        xin = torch.randn(M, K, device="cuda")
        gin, bin_ = torch.ones(K, device="cuda"), torch.zeros(K, device="cuda")
        epi.ln_in, epi.ln_in_ld, epi.ln_in_gain, epi.ln_in_bias, epi.ln_in_eps = (
            xin.data_ptr(), K, gin.data_ptr(), bin_.data_ptr(), 1e-5)
    epi.k_split = int(os.environ.get("KSPLIT", "0"))
    for na, cs in cfgs:
        pc = bool(os.environ.get("PC"))  # the persistent CTA-pair kernel (cs = pairs)
        if pc:
            N.call("skb_gemm_force_sw", 0, 0, 0)
            N.call("skb_gemm_force_pc", 2, na, cs)
        else:
            N.call("skb_gemm_force_sw", 2, na, cs)
        buf = (C.c_ulonglong * (1024 * 16))()
        for i in range(8):  # warm; the last launch is traced (its weights cold)
            if i == 7:
                torch.cuda.synchronize()
                N.call("skb_debug_gemm_trace", buf)  # clear
            N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, Ws[i % len(Ws)].data_ptr(), K,
                   C.byref(epi), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        N.call("skb_debug_gemm_trace", buf)
        t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        cols = [0, 2, 3, 5, 1, 8, 9, 10, 4, 11, 12, 13, 14, 6]
        labels = ["entry", "postwait", "stage0", "accready", "epi/partial", "csync", "recv",
                  "summed", "stored", "flushed", "stats", "ln_ticket/ln_in_done", "ln_rows/mma_xready", "exit"]
        if pc:  # k_gemm_pc's PC_STAMP slots
            cols = [0, 1, 2, 3, 4, 5, 6, 8, 9]
            labels = ["entry", "alloc+csync", "postwait", "stage0", "mma0 issued", "accready0",
                      "epi0 done", "stores drained", "exit"]
        rel = (t[:, cols] - t0) / 1e3
        print(f"{name} na={na} cs={cs} ctas={len(t)} sms={len(set(t[:, 7]))}")
        for j, lab in enumerate(labels):
            col = rel[:, j]
            col = col[(col > -1e6) & (col < 1e6)]
            if not len(col):
                continue
            print(f"   {lab:9s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
N.call("skb_gemm_force_sw", 0, 0, 0)
N.call("skb_gemm_force_pc", 0, 0, 0)
