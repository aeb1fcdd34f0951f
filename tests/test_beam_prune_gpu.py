"""The pruned beam scan (only 32-column groups whose partial max can reach
the top K) must pick exactly what the full scan picks from the same logits
and the same fused log-softmax partials — including exact ties, 1-ulp
near-ties and top-K clusters inside one group."""

import numpy as np
import pytest
import torch

from paper_2207_05851_b200 import _native as N
from paper_2207_05851_b200 import kern

pytestmark = pytest.mark.gpu


def _state(B, K, U, logits, prune, lse_part, mask=None, t=3, max_len=40):
    dev = "cuda"
    R = B * K
    z = lambda n, dt=torch.int32: torch.zeros(n, dtype=dt, device=dev)  # noqa: E731
    bufs = dict(len_pen=torch.ones(max_len + 1, dtype=torch.float64, device=dev),
                step=torch.full((1,), t, dtype=torch.int32, device=dev),
                max_len=torch.full((B,), max_len, dtype=torch.int32, device=dev),
                prefix_len=z(B), prefix_col=torch.full((B,), -1, dtype=torch.int32, device=dev),
                n_alive=torch.full((B,), K, dtype=torch.int32, device=dev), done=z(B),
                score=(torch.arange(R, device=dev, dtype=torch.float64) % 3) * -0.25,
                tok=z(R), ftok=z(R), parent=z(R), tok_hist=z(max_len * R), par_hist=z(max_len * R),
                fac_hist=z(max_len * R), cand_score=z(R * K, torch.float64),
                cand_lp=z(R * K, torch.float32), cand_col=z(R * K), cand_cnt=z(R),
                row_argmax=z(R), fac_choice=z(R), counter=z(B),
                best_norm=z(B, torch.float64), best_logprob=z(B, torch.float64),
                best_steps=z(B), best_forced=z(B), best_parent=z(B), best_fac=z(B), n_done=z(1))
    b = bufs
    st = N.BeamState(B, K, U, max_len, 0, b["len_pen"].data_ptr(), b["step"].data_ptr(), None,
                     N.ptr(mask), 3, b["max_len"].data_ptr(), b["prefix_len"].data_ptr(),
                     b["prefix_col"].data_ptr(), 1, None, b["n_alive"].data_ptr(),
                     b["done"].data_ptr(), b["score"].data_ptr(), b["tok"].data_ptr(),
                     b["ftok"].data_ptr(), b["parent"].data_ptr(), b["tok_hist"].data_ptr(),
                     b["par_hist"].data_ptr(), b["fac_hist"].data_ptr(), None, 1, None,
                     lse_part.data_ptr(), lse_part.shape[1] // 2, prune, 0,
                     b["cand_score"].data_ptr(), b["cand_lp"].data_ptr(), b["cand_col"].data_ptr(),
                     b["cand_cnt"].data_ptr(), b["row_argmax"].data_ptr(),
                     b["fac_choice"].data_ptr(), b["counter"].data_ptr(), b["best_norm"].data_ptr(),
                     b["best_logprob"].data_ptr(), b["best_steps"].data_ptr(),
                     b["best_forced"].data_ptr(), b["best_parent"].data_ptr(),
                     b["best_fac"].data_ptr(), b["n_done"].data_ptr())
    return st, b


def _partials(x, U):
    """(max, sum exp) per 32-column group, as the GEMM LOGITS epilogue writes."""
    R = x.shape[0]
    G = (U + 31) // 32
    xp = torch.full((R, G * 32), float("-inf"), device=x.device)
    xp[:, :U] = x
    g = xp.view(R, G, 32)
    m = g.max(-1).values
    s = torch.exp(g - m[..., None]).sum(-1)
    return torch.stack([m, s], -1).reshape(R, 2 * G).contiguous()


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("K", [1, 4, 5, 12])
@pytest.mark.parametrize("final", [False, True])
def test_pruned_equals_full_scan(seed, K, final):
    B, U = 6, 3000 + 7 * seed
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B * K, U, device="cuda", generator=g) * 2
    # exact ties and one-ulp near-ties around the top; a cluster in one group
    top = x.max(1, keepdim=True).values
    x[:, 100:110] = top + 0.5
    x[:, 2000] = top[:, 0] + 0.5
    x[:, 37] = torch.nextafter(top[:, 0] + 0.5, torch.tensor(-1e9, device="cuda"))
    x[:, 64:96] = top + 0.25
    x = x.contiguous()
    part = _partials(x, U)
    t, max_len = (39, 40) if final else (3, 40)
    picks = []
    for prune in (0, 1):
        st, b = _state(B, K, U, x, prune, part, t=t, max_len=max_len)
        kern.beam_step(x, st)
        torch.cuda.synchronize()
        picks.append({k: b[k].cpu().numpy().copy() for k in
                      ("tok", "parent", "score", "n_alive", "best_logprob", "best_forced",
                       "row_argmax", "best_parent")})
    for k in picks[0]:
        np.testing.assert_array_equal(picks[0][k], picks[1][k], err_msg=k)
