"""Caller-fixed K split (skb_epilogue.k_split, Model(gemm_split="latency")):
every projection is a sum of K-partials in partial order, so a row's result
must be bitwise the same whether the GEMM ran with 1 row (pull reduction over
distributed shared memory, prologue LayerNorm) or 640 rows (bulk-copy push
reduction, LayerNorm launch) — the batch-composition invariance of
test_search.py:400-405 for the latency configuration — and within the bf16
tolerance of an fp64 reference (kernels.py:167-195, 479-484)."""

import pytest
import torch

from paper_2207_05851_b200 import _native as N
from paper_2207_05851_b200 import kern

pytestmark = pytest.mark.gpu

BIG = 640
SMALL = (1, 5, 16, 40)


def _weights(Nn, K, seed, split):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W = (torch.randn(Nn, K, device="cuda", generator=g) * 0.05).bfloat16()
    W._skb_k_split = split
    bias = torch.randn(Nn, device="cuda", generator=g)
    return g, W, bias


@pytest.mark.parametrize("split", [2, 4, 8, 16])
@pytest.mark.parametrize("kind,Nn,K", [(N.EPI_STORE, 3072, 1024), (N.EPI_RELU, 4096, 1024),
                                       (N.EPI_RESID, 1024, 1024), (N.EPI_RESID, 1024, 4096),
                                       (N.EPI_STORE, 512, 512)])
def test_k_split_rows_independent_of_batch(split, kind, Nn, K):
    g, W, bias = _weights(Nn, K, Nn + K + split, split)
    A = torch.randn(BIG, K, device="cuda", generator=g).bfloat16()
    x0 = torch.randn(BIG, Nn, device="cuda", generator=g)

    def run(M):
        if kind == N.EPI_RESID:
            out = x0[:M].clone()
        else:
            out = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
        kern.gemm(A[:M], W, out, kind, bias)
        return out

    big = run(BIG)
    torch.cuda.synchronize()
    ref = A.double() @ W.double().T + bias.double()
    if kind == N.EPI_RELU:
        ref = ref.clamp_min(0)
    if kind == N.EPI_RESID:
        ref = ref + x0.double()
        assert (big.double() - ref).abs().max().item() <= 2e-3 * K ** 0.5
    else:
        assert (big.double() - ref).abs().max().item() <= 2e-2 * (K / 256) ** 0.5
    for M in SMALL:
        small = run(M)
        torch.cuda.synchronize()
        assert torch.equal(small, big[:M]), (M, (small.float() - big[:M].float()).abs().max().item())


@pytest.mark.parametrize("split", [4, 8])
@pytest.mark.parametrize("kind,Nn,K", [(N.EPI_STORE, 3072, 1024), (N.EPI_RELU, 4096, 1024)])
def test_k_split_input_layernorm(split, kind, Nn, K):
    """A = LN(x) in the GEMM prologue (each CTA normalises the whole row and
    keeps its own k-blocks) at <= 32 rows, a LayerNorm launch above: bitwise
    equal rows, and equal to the LayerNorm kernel + plain GEMM."""
    g, W, bias = _weights(Nn, K, 7 * split + Nn, split)
    x = torch.randn(BIG, K, device="cuda", generator=g) * 2 + 0.5
    gain = torch.rand(K, device="cuda", generator=g) + 0.5
    lb = torch.randn(K, device="cuda", generator=g)
    b = bias if kind == N.EPI_RELU else None

    def run(M):
        h = torch.zeros(M, K, device="cuda", dtype=torch.bfloat16)
        out = torch.zeros(M, Nn, device="cuda", dtype=torch.bfloat16)
        kern.gemm(h, W, out, kind, b, ln_in=(x[:M], gain, lb))
        return out

    big = run(BIG)
    h = torch.zeros(BIG, K, device="cuda", dtype=torch.bfloat16)
    kern.layernorm(x, gain, lb, h)
    sep = torch.zeros(BIG, Nn, device="cuda", dtype=torch.bfloat16)
    kern.gemm(h, W, sep, kind, b)
    torch.cuda.synchronize()
    assert torch.equal(big, sep)
    for M in (1, 5, 16, 32, 33):
        small = run(M)
        torch.cuda.synchronize()
        assert torch.equal(small, big[:M]), (M, (small.float() - big[:M].float()).abs().max().item())


def test_k_split_ssru_epilogue():
    """SSRU cell epilogue (model.py:268-272) under a K split of 4: small and
    large batches give the same cells and residual rows."""
    d = 1024
    g, W, bias = _weights(2 * d, d, 99, 4)
    A = torch.randn(BIG, d, device="cuda", generator=g).bfloat16()
    x0 = torch.randn(BIG, d, device="cuda", generator=g)
    outs = {}
    for M in (BIG, 5):
        x = x0[:M].clone()
        cn = torch.zeros(M, d, device="cuda")
        kern.gemm(A[:M], W, x, N.EPI_SSRU, bias, c_state=cn)
        outs[M] = (x, cn)
    torch.cuda.synchronize()
    assert torch.equal(outs[5][0], outs[BIG][0][:5])
    assert torch.equal(outs[5][1], outs[BIG][1][:5])


def test_k_split_rejects_bad_values():
    from paper_2207_05851_b200.errors import ConfigError
    A = torch.zeros(4, 256, device="cuda", dtype=torch.bfloat16)
    W = torch.zeros(128, 256, device="cuda", dtype=torch.bfloat16)
    W._skb_k_split = 3
    out = torch.zeros(4, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ConfigError):
        kern.gemm(A, W, out)
