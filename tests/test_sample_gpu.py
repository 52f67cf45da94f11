"""Rollout token sampling (csrc/sample.cu): determinism, distribution,
and consistency of the behaviour log-probs with the learner's kernel."""

import numpy as np
import pytest

from oracle import grpo_oracle as O

pytestmark = pytest.mark.gpu


def test_sampling_is_deterministic_per_seed(dev):
    import torch
    from paper_2605_13276_b200.rollout import sample_action_tokens
    x = (torch.randn(448, 4096, device=dev) * 2).to(torch.bfloat16)
    a = sample_action_tokens(x, 56, seed=7)
    b = sample_action_tokens(x, 56, seed=7)
    c = sample_action_tokens(x, 56, seed=8)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert not torch.equal(a[0], c[0])
    assert int(a[0].min()) >= 0 and int(a[0].max()) < 4096


def test_sampled_distribution_matches_softmax(dev):
    """Chi-square goodness of fit: 200k rows of the same 16-way logits."""
    import torch
    from paper_2605_13276_b200.rollout import sample_action_tokens
    logits = torch.tensor([0.5, -1.0, 2.0, 0.0, 1.5, -3.0, 0.25, 1.0,
                           -0.5, 0.75, -2.0, 1.25, 0.1, -0.2, 0.9, -1.5], device=dev)
    R = 200_000
    x = logits.repeat(R, 1).contiguous()
    tok, _, _ = sample_action_tokens(x, 1, seed=123)
    counts = np.bincount(tok.cpu().numpy(), minlength=16)
    p = torch.softmax(logits.double(), 0).cpu().numpy()
    chi2 = float((((counts - R * p) ** 2) / (R * p)).sum())
    assert chi2 < 45.0, (chi2, counts)  # 15 dof: p ~ 1e-4


def test_behaviour_logprobs_match_oracle_and_learner(dev):
    import torch
    from paper_2605_13276_b200 import grpo
    from paper_2605_13276_b200.rollout import sample_action_tokens
    n_groups, G, C, T, V = 4, 8, 1, 56, 32064
    R = n_groups * G * C * T
    x = (torch.randn(R, V, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
         * 2).to(torch.bfloat16)
    tok, blp, lp_chunk, lp_tok = sample_action_tokens(x, T, seed=3, want_lp_tok=True)
    # oracle: f64 log-softmax gather of the sampled tokens
    lse, olp = O.token_row_stats(x.float().cpu().numpy(), tok.cpu().numpy())
    np.testing.assert_allclose(lp_tok.cpu().numpy(), olp, rtol=1e-9, atol=1e-6)
    np.testing.assert_allclose(lp_chunk.cpu().numpy(),
                               olp.reshape(-1, T).sum(axis=1), rtol=1e-9, atol=1e-5)
    assert torch.equal(blp, lp_chunk.float())
    # the learner's fused kernel sees the same log-probs: ratios ~ 1
    rw = torch.randint(0, 2, (n_groups * G,), device=dev).float()
    tl = grpo.TokenLoss(n_groups, G, C, T, V, grpo.GrpoConfig(group_size=G))
    dl = torch.empty_like(x)
    tl.launch(x, tok, blp, rw, dl)
    st = tl.stats(rw)
    assert abs(st["mean_ratio"] - 1.0) < 1e-4
    assert st["clip_fraction"] <= 1.0


@pytest.mark.parametrize("dtype_name", ["bfloat16", "float32"])
def test_wide_rows_walk_every_granule_block(dev, dtype_name):
    """V = 131,072: each thread owns 64 (bf16) / 128 (f32) granules, so the
    winner's warp walks its elements in several 32-granule blocks.  Mass sits
    on 16 columns spread over the row (many in the later blocks); one-hot rows
    must return their column exactly."""
    import torch
    from paper_2605_13276_b200.rollout import sample_action_tokens
    dt = getattr(torch, dtype_name)
    V, R = 131072, 40_000
    cols = torch.tensor([5, 2047, 9000, 40000, 65535, 65536, 70001, 81920,
                         90000, 100003, 110000, 120000, 125000, 130000, 131000, 131071],
                        device=dev)
    w = torch.tensor([0.5, -1.0, 2.0, 0.0, 1.5, -3.0, 0.25, 1.0,
                      -0.5, 0.75, -2.0, 1.25, 0.1, -0.2, 0.9, -1.5], device=dev)
    x = torch.full((R, V), -80.0, device=dev, dtype=dt)
    x[:, cols] = w.to(dt)
    tok, _, _ = sample_action_tokens(x, 1, seed=5)
    hit = (tok.unsqueeze(1) == cols.unsqueeze(0).int())
    assert bool(hit.any(dim=1).all())
    counts = hit.sum(dim=0).cpu().numpy()
    p = torch.softmax(w.to(dt).double(), 0).cpu().numpy()
    chi2 = float((((counts - R * p) ** 2) / (R * p)).sum())
    assert chi2 < 45.0, (chi2, counts)
    # one-hot rows: the only finite column wins, wherever it sits
    oh = torch.full((len(cols), V), float("-inf"), device=dev, dtype=dt)
    oh[torch.arange(len(cols), device=dev), cols] = 0.0
    t1, _, lp1 = sample_action_tokens(oh, 1, seed=9)
    assert torch.equal(t1, cols.int())
    assert torch.all(lp1 == 0.0)
