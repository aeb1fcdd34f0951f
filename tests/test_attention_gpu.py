"""Attention kernels vs a torch fp32 reference of the same op
(kernels.py:510-517; model.py:559-573): incremental self-attention over the
ancestor-indexed KV cache (grouped and per-row kernels), cross-attention and
encoder attention."""

import math

import pytest
import torch

from paper_2207_05851_b200 import kern

pytestmark = pytest.mark.gpu


def _ref_self(qkv, kc, vc, anc_cur, t, H, dh):
    R = qkv.shape[0]
    D = H * dh
    q = qkv[:, :D].float().view(R, H, dh)
    knew = qkv[:, D:2 * D].float().view(R, H, dh)
    vnew = qkv[:, 2 * D:].float().view(R, H, dh)
    out = torch.zeros(R, H, dh, device=qkv.device)
    for r in range(R):
        ks, vs = [], []
        for p in range(t):
            s = int(anc_cur[r, p])
            ks.append(kc[s, p].float())
            vs.append(vc[s, p].float())
        ks.append(knew[r])
        vs.append(vnew[r])
        K = torch.stack(ks, 1)  # H, t+1, dh
        V = torch.stack(vs, 1)
        sc = torch.einsum("hd,hpd->hp", q[r], K) / math.sqrt(dh)
        out[r] = torch.einsum("hp,hpd->hd", torch.softmax(sc, -1), V)
    return out.view(R, D)


@pytest.mark.parametrize("G,t,dh,H", [(5, 0, 64, 4), (5, 7, 64, 4), (5, 45, 64, 4), (4, 70, 32, 4),
                                      (3, 33, 128, 4), (1, 40, 64, 4), (8, 79, 64, 8),
                                      (16, 63, 64, 4), (5, 60, 64, 16), (2, 79, 64, 6)])
@pytest.mark.parametrize("tree", [False, True])
def test_self_attention_grouped_matches_reference(G, t, dh, H, tree):
    """Cache layout [slot][pos][head][dh]; the beam rows of a group reference
    ancestor slots of their own group.  `tree` draws them from a beam tree
    (mostly shared history, the tensor-core kernel's common case); otherwise
    uniformly (mostly distinct entries: several staging passes)."""
    g = torch.Generator(device="cuda").manual_seed(t * 10 + G + H)
    B, S = 6, 80
    R, D = B * G, H * dh
    qkv = torch.randn(R, 3 * D, device="cuda", generator=g).bfloat16()
    kc = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    vc = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    anc = torch.zeros(2, R, S, dtype=torch.int32, device="cuda")
    grp = torch.arange(R, device="cuda") // G
    if tree:
        hist = torch.arange(R, device="cuda")[:, None].repeat(1, S)
        for p in range(1, S):
            par = grp * G + torch.randint(0, max(1, G // 2), (R,), device="cuda", generator=g)
            hist[:, :p] = hist[par, :p]
        anc[t & 1] = hist.int()
    else:
        anc[t & 1] = (grp[:, None] * G + torch.randint(0, G, (R, S), device="cuda", generator=g)).int()
    step = torch.tensor([t], dtype=torch.int32, device="cuda")
    ref = _ref_self(qkv, kc, vc, anc[t & 1], t, H, dh)
    ctx = torch.zeros(R, D, device="cuda", dtype=torch.bfloat16)
    kern.self_attention_step(qkv, kc, vc, anc, step, ctx, R, H, dh, S, group=G)
    torch.cuda.synchronize()
    assert (ctx.float() - ref).abs().max().item() < 2e-2
    # the fresh k/v landed in slot (r, t)
    assert torch.equal(kc[:, t].reshape(R, D), qkv[:, D:2 * D])
    assert torch.equal(vc[:, t].reshape(R, D), qkv[:, 2 * D:])


@pytest.mark.parametrize("G,t,H", [(5, 0, 16), (5, 35, 16), (5, 69, 16), (1, 40, 8), (8, 79, 8),
                                   (16, 63, 4), (3, 31, 4), (2, 32, 4)])
@pytest.mark.parametrize("tree", [False, True])
def test_self_attention_planned_bitwise(G, t, H, tree):
    """One skb_attn_plan per step replaces every layer's ancestor walk: the
    planned kernel stages the same entries in the same order, so its output
    is bitwise equal to the unplanned one (and the cache write identical)."""
    dh = 64
    g = torch.Generator(device="cuda").manual_seed(t * 7 + G + H)
    B, S = 7, 80
    R, D = B * G, H * dh
    qkv = torch.randn(R, 3 * D, device="cuda", generator=g).bfloat16()
    kc0 = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    vc0 = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    anc = torch.zeros(2, R, S, dtype=torch.int32, device="cuda")
    grp = torch.arange(R, device="cuda") // G
    if tree:
        hist = torch.arange(R, device="cuda")[:, None].repeat(1, S)
        for p in range(1, S):
            par = grp * G + torch.randint(0, max(1, G // 2), (R,), device="cuda", generator=g)
            hist[:, :p] = hist[par, :p]
        anc[t & 1] = hist.int()
    else:
        anc[t & 1] = (grp[:, None] * G + torch.randint(0, G, (R, S), device="cuda", generator=g)).int()
    step = torch.tensor([t], dtype=torch.int32, device="cuda")
    plan = torch.zeros(kern.attn_plan_bytes(R, G, S), dtype=torch.uint8, device="cuda")
    kern.attn_plan(anc, step, plan, R, S, G)
    outs = []
    for use_plan in (False, True):
        kc, vc = kc0.clone(), vc0.clone()
        ctx = torch.zeros(R, D, device="cuda", dtype=torch.bfloat16)
        kern.self_attention_step(qkv, kc, vc, anc, step, ctx, R, H, dh, S, group=G,
                                 plan=plan if use_plan else None)
        torch.cuda.synchronize()
        outs.append((ctx, kc, vc))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])


@pytest.mark.parametrize("G,L", [(5, 30), (1, 17), (4, 90)])
def test_cross_attention_matches_reference(G, L):
    g = torch.Generator(device="cuda").manual_seed(L)
    B, H, dh = 7, 16, 64
    R, D = B * G, H * dh
    q = torch.randn(R, D, device="cuda", generator=g).bfloat16()
    kv = torch.randn(B * L, 2 * D, device="cuda", generator=g).bfloat16()
    lengths = torch.randint(1, L + 1, (B,), device="cuda", generator=g).int()
    row_sent = (torch.arange(R, device="cuda") // G).int()
    ctx = torch.zeros(R, D, device="cuda", dtype=torch.bfloat16)
    kern.cross_attention_step(q, kv, 0, D, L, row_sent, lengths, ctx, R, H, dh, G)
    torch.cuda.synchronize()
    K = kv[:, :D].float().view(B, L, H, dh)
    V = kv[:, D:].float().view(B, L, H, dh)
    ref = torch.zeros(R, H, dh, device="cuda")
    for r in range(R):
        b = int(row_sent[r])
        n = int(lengths[b])
        sc = torch.einsum("hd,lhd->hl", q[r].float().view(H, dh), K[b, :n]) / math.sqrt(dh)
        ref[r] = torch.einsum("hl,lhd->hd", torch.softmax(sc, -1), V[b, :n])
    assert (ctx.float() - ref.view(R, D)).abs().max().item() < 2e-2


@pytest.mark.parametrize("B,G,t", [(1, 5, 35), (1, 1, 69), (7, 5, 20), (128, 5, 40)])
def test_self_attention_heads_per_cta_bitwise(B, G, t):
    """Heads per CTA (one warp per head; 2 automatically for batch-1 grids,
    else 4) only changes which CTA computes a head, never its numbers."""
    from paper_2207_05851_b200 import _native as N
    dh, H, S = 64, 16, 80
    g = torch.Generator(device="cuda").manual_seed(B + t)
    R, D = B * G, H * dh
    qkv = torch.randn(R, 3 * D, device="cuda", generator=g).bfloat16()
    kc0 = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    vc0 = torch.randn(R, S, H, dh, device="cuda", generator=g).bfloat16()
    anc = torch.zeros(2, R, S, dtype=torch.int32, device="cuda")
    grp = torch.arange(R, device="cuda") // G
    anc[t & 1] = (grp[:, None] * G + torch.randint(0, G, (R, S), device="cuda", generator=g)).int()
    step = torch.tensor([t], dtype=torch.int32, device="cuda")
    plan = torch.zeros(kern.attn_plan_bytes(R, G, S), dtype=torch.uint8, device="cuda")
    kern.attn_plan(anc, step, plan, R, S, G)
    outs = []
    try:
        for hg in (0, 2, 4, 8):
            N.call("skb_attn_force_heads", hg)
            kc, vc = kc0.clone(), vc0.clone()
            ctx = torch.zeros(R, D, device="cuda", dtype=torch.bfloat16)
            kern.self_attention_step(qkv, kc, vc, anc, step, ctx, R, H, dh, S, group=G, plan=plan)
            torch.cuda.synchronize()
            outs.append(ctx)
    finally:
        N.call("skb_attn_force_heads", 0)
    for o in outs[1:]:
        assert torch.equal(outs[0], o)
