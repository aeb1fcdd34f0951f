"""Sweep the tcgen05 GEMM tile configs on the decode-step shapes, the way the
decode step sees them: weights cold (rotating through copies > L2), the
activation matrix warm, launches back to back inside one CUDA graph (PDL
overlap included).  cuBLAS (torch.matmul, bf16 out) is timed beside it.

    python tools/gemm_sweep.py [M] > gpurun_out/gemm_sweep.txt
"""
import ctypes as C
import itertools
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 640
SHAPES = {"qkv": (3072, 1024), "wo": (1024, 1024), "ffn1": (4096, 1024), "ffn2": (1024, 4096),
          "ssru": (2048, 1024), "out_proj": (32000, 1024)}
import os
if os.environ.get("SHAPES"):
    SHAPES = {k: SHAPES[k] for k in os.environ["SHAPES"].split(",")}
REPS = 24
dev = "cuda"
ws = torch.empty(32 << 20, device=dev)
cnt = torch.zeros(1 << 16, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream
lib = N.lib()


def time_graph(fn, reps):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for r in range(reps):
                fn(r)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best * 1e3  # us


out_rows = []
for name, (Nn, K) in SHAPES.items():
    ncopy = max(2, min(REPS, int(160e6 // (Nn * K * 2)) + 1))
    A = torch.randn(M, K, device=dev).bfloat16()
    Ws = [torch.randn(Nn, K, device=dev).bfloat16() * 0.05 for _ in range(ncopy)]
    ref = (A.float() @ Ws[0].float().T)
    flops = 2.0 * M * Nn * K
    if os.environ.get("LOGITS") and name == "out_proj":  # the decode step's epilogue
        out = torch.zeros(M, Nn, device=dev)
        part = torch.zeros(M, 2 * ((Nn + 31) // 32), device=dev)
        epi = N.Epilogue(N.EPI_LOGITS, None, out.data_ptr(), Nn, N.F32, None, None, None, 0, None,
                         0, part.data_ptr(), part.shape[1] // 2, None, 0, 1)
    else:
        out = torch.zeros(M, Nn, device=dev, dtype=torch.bfloat16)
        epi = N.Epilogue(N.EPI_STORE, None, out.data_ptr(), Nn, N.BF16, None, None, None, 0, None,
                         0, None, 0, None, 0, 1, ws.data_ptr(), ws.numel(), cnt.data_ptr(),
                         cnt.numel())

    def ours(r=0):
        W = Ws[r % ncopy]
        N.call("skb_gemm", N.BF16, M, Nn, K, A.data_ptr(), K, W.data_ptr(), K, C.byref(epi),
               torch.cuda.current_stream().cuda_stream)

    cub_out = out if out.dtype == torch.bfloat16 else out.to(torch.bfloat16)

    def cublas(r=0):
        torch.matmul(A, Ws[r % ncopy].T, out=cub_out)

    us = time_graph(cublas, REPS)
    out_rows.append(dict(shape=name, M=M, cfg="cublas", us=round(us, 2),
                         tflops=round(flops / us / 1e6, 1)))
    print(json.dumps(out_rows[-1]), flush=True)
    cfgs = [("auto", 0, 0, 0), ("sw auto", 2, 0, 0)]
    if os.environ.get("SW_SWEEP"):
        cfgs.insert(1, ("tc auto", 1, 0, 0))
        for na in (32, 48, 64, 80, 96, 128, 160, 256):
            for cs in ((1, 2, 4) if K >= 4096 else tuple(int(x) for x in os.environ.get("SW_CS", "1").split(","))):
                if cs > 1 and na % (4 * cs):
                    continue
                cfgs.append((f"sw na{na} cs{cs}", 2, na, cs))
    # persistent CTA-pair kernel (mode 2 = forced), its tile and grid choices
    if not os.environ.get("NO_PC"):
        cfgs.append(("pc auto", -2, 0, 0))
        for na in (64, 96, 128, 160, 192, 224, 256):
            cfgs.append((f"pc na{na}", -2, na, 0))
        for pairs in (32, 48, 64):
            cfgs.append((f"pc pairs{pairs}", -2, 0, pairs))
    for label, mode, na, cs in cfgs:
        if mode == -2:
            lib.skb_gemm_force_sw(0, 0, 0)
            lib.skb_gemm_force_pc(2, na, cs)
        else:
            lib.skb_gemm_force_pc(1 if mode else 0, 0, 0)
            lib.skb_gemm_force_sw(mode, na, cs)
        try:
            out.zero_()
            ours()
            torch.cuda.synchronize()
            err = (out.float() - ref).abs().max().item()
            us = time_graph(ours, REPS)
        except Exception as e:  # noqa: BLE001
            print(json.dumps(dict(shape=name, cfg=label, error=str(e)[:80])))
            continue
        out_rows.append(dict(shape=name, M=M, cfg=label, us=round(us, 2),
                             tflops=round(flops / us / 1e6, 1), err=round(err, 4)))
        print(json.dumps(out_rows[-1]), flush=True)
    lib.skb_gemm_force_sw(0, 0, 0)
    lib.skb_gemm_force_pc(0, 0, 0)
