"""tc (M-major persistent) vs sw (swap-AB) GEMM kernels on the same inputs:
bitwise equality of the results and of the LOGITS partials, and timing
(20 back-to-back launches) at decode / encoder row counts."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2207_05851_b200 import _native as N, kern  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(3)
cases = [(M, Nn, K, kind) for M in (640, 1100, 2560, 3840)
         for (Nn, K, kind) in ((3072, 1024, N.EPI_STORE), (4096, 1024, N.EPI_RELU),
                               (1024, 4096, N.EPI_RESID), (32000, 1024, N.EPI_LOGITS))]
for (M, Nn, K, kind) in cases:
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(Nn, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(Nn, device="cuda", generator=g) if kind == N.EPI_RELU else None
    f32 = kind in (N.EPI_LOGITS, N.EPI_RESID)
    res, t = [], []
    for mode in (1, 2):
        N.call("skb_gemm_force_sw", mode, 0, 0)
        o = torch.zeros(M, Nn, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        part = torch.zeros(M, 2 * ((Nn + 31) // 32), device="cuda") if kind == N.EPI_LOGITS else None
        kern.gemm(A, W, o, kind, bias, lse_part=part)
        torch.cuda.synchronize()
        res.append((o.clone(), None if part is None else part.clone()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            kern.gemm(A, W, o, kind, bias, lse_part=part)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) / 20 * 1e3)
    N.call("skb_gemm_force_sw", 0, 0, 0)
    eq = torch.equal(res[0][0], res[1][0]) if kind != N.EPI_RESID else "n/a (accumulates)"
    peq = "" if kind != N.EPI_LOGITS else f" partials equal {torch.equal(res[0][1], res[1][1])}"
    print(f"M={M:5d} N={Nn:5d} K={K:5d} kind={kind}: tc {t[0]:7.1f} us  sw {t[1]:7.1f} us  "
          f"out equal {eq}{peq}")
