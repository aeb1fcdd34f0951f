"""Per-CTA timeline of one persistent CTA-pair GEMM launch (build with
SKB_NVCC_EXTRA=-DSKB_GEMM_TRACE).  Slots, relative to the earliest CTA entry
(us, min/median/max over CTAs): 0 entry, 1 prologue done (barriers, TMEM,
cluster sync), 2 producer past griddepcontrol.wait, 3 first stage landed
(leader MMA), 4 first tile's MMAs committed, 5 first accumulator ready
(epilogue), 6 first tile stored, 8 epilogue done, 9 exit.

    M=640 SHAPES=qkv,out_proj python tools/pc_trace.py [na,pairs ...]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M = int(os.environ.get("M", "640"))
shapes = {"wo": (1024, 1024), "qkv": (3072, 1024), "ffn1": (4096, 1024), "out_proj": (32000, 1024)}
if os.environ.get("SHAPES"):
    shapes = {k: shapes[k] for k in os.environ["SHAPES"].split(",")}
cfgs = [(int(a), int(b)) for a, b in (x.split(",") for x in sys.argv[1:])] or [(0, 0)]
names = {0: "entry", 1: "prologue", 2: "pdl_wait", 3: "first_stage", 4: "tile0_mma",
         5: "tile0_acc", 6: "tile0_stored", 8: "epi_done", 9: "exit"}
for name, (Nn, K) in shapes.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    Ws = [torch.randn(Nn, K, device="cuda").bfloat16() for _ in range(8 if Nn * K < 1e8 / 2 else 2)]
    if os.environ.get("LOGITS"):
        out = torch.zeros(M, Nn, device="cuda")
        part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda")
        epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None,
                         0, part.data_ptr(), part.shape[1] // 2, None, 0, 1)
    else:
        out = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
        epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.BF16, None, None, None, 0)
    for na, pairs in cfgs:
        N.call("skb_gemm_force_pc", 2, na, pairs)
        buf = (C.c_ulonglong * (1024 * 16))()
        for i in range(8):
            if i == 7:
                torch.cuda.synchronize()
                N.call("skb_debug_gemm_trace", buf)  # clear
            N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, Ws[i % len(Ws)].data_ptr(), K,
                   C.byref(epi), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        N.call("skb_debug_gemm_trace", buf)
        t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
        live = t[:, 0] > 0
        t = t[live]
        t0 = t[:, 0].min()
        print(f"{name} M={M} na={na} pairs={pairs} ctas={live.sum()}")
        for sl, nm in names.items():
            v = t[:, sl]
            v = v[v > 0]
            if v.size == 0:
                continue
            r = (v - t0) / 1e3
            print(f"  {sl} {nm:13s} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")
    N.call("skb_gemm_force_pc", 0, 0, 0)
