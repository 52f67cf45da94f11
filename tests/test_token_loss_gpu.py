"""GPU parity of the fused action-token GRPO loss (csrc/token_loss.cu) against
the numpy oracle (oracle/grpo_oracle.py), through the C-ABI.

Tolerances (north star): loss and gradients within 1e-5 relative in fp32,
1e-2 in bf16; chunk indexing / advantage grouping / canonical order exact.
"""

import numpy as np
import pytest

from oracle import grpo_oracle as O
from oracle.check import assert_dlogits_close, coeff_term_scale, row_condition

pytestmark = pytest.mark.gpu


def _case(seed, n_groups, G, C, T, V, dtype, spread=0.05, binary=True, ids=None):
    import torch
    rng = np.random.default_rng(seed)
    x = rng.normal(0.0, 2.0, (n_groups, G, C, T, V)).astype(np.float32)
    if dtype == torch.bfloat16:
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()  # exact bf16 values
    tokens = rng.integers(0, V, (n_groups, G, C, T)).astype(np.int32)
    # behaviour log-probs near the current policy (ratios inside the clip box)
    _, _, st0 = O.grpo_token_grad(x, tokens, np.zeros((n_groups, G, C), np.float32),
                                  np.tile(np.arange(G, dtype=np.float32), (n_groups, 1)),
                                  np.arange(n_groups), want_dlogits=False)
    blp = (st0["lp_chunk"] + rng.uniform(-spread, spread, (n_groups, G, C))).astype(np.float32)
    if binary:
        rewards = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
    else:
        rewards = rng.uniform(0, 1, (n_groups, G)).astype(np.float32)
    if ids is None:
        ids = rng.permutation(n_groups * 3)[:n_groups]
    return x, tokens, blp, rewards, np.asarray(ids)


def _assert_coeff_close(got, ost, blp, rewards, rtol, clip_eps=0.2, kl_coeff=0.0):
    """Per-chunk coefficients equal the oracle's to rtol of max(|coeff|, the
    magnitude of the terms it is built from) -- the KL term can cancel the
    surrogate term -- except chunks whose ratio sits within 1e-4 of a clip
    edge (the lp tolerance may flip the branch there; the clip count then
    differs by those chunks at most).  Returns (n_edge, per-row condition)."""
    want = ost["coeff"]
    rho = np.exp(ost["lp_chunk"] - np.asarray(blp, np.float32).astype(np.float64))
    edge = (np.abs(rho - (1 - clip_eps)) < 1e-4) | (np.abs(rho - (1 + clip_eps)) < 1e-4)
    got = np.asarray(got).reshape(want.shape)
    scale = np.maximum(np.abs(want), coeff_term_scale(ost["lp_chunk"], blp, rewards,
                                                      clip_eps, kl_coeff=kl_coeff))
    err = np.abs(got - want)
    bad = (err > rtol * scale) & ~edge
    assert not bad.any(), (f"{int(bad.sum())} coefficients off: max err/scale "
                           f"{float((err / scale)[~edge].max()):.3g} > {rtol:g}")
    T = ost["lp_tok"].size // want.size
    cond = row_condition(want, np.where(edge, np.abs(want), scale), T)
    return int(edge.sum()), cond


def _run_gpu(x, tokens, blp, rewards, ids, dtype, fused=True, cfg=None):
    import torch
    from paper_2605_13276_b200 import grpo
    cfg = cfg or grpo.GrpoConfig(group_size=x.shape[1])
    dev = torch.device("cuda", 0)
    lg = torch.from_numpy(x).to(dev, dtype)
    loss, dl, st = grpo.grpo_token_grad(
        lg, torch.from_numpy(tokens).to(dev), torch.from_numpy(blp).to(dev),
        torch.from_numpy(rewards).to(dev), ids, cfg, fused=fused)
    torch.cuda.synchronize()
    return loss, dl.float().cpu().numpy(), st


def _check(x, tokens, blp, rewards, ids, dtype, fused, rtol, cfg_kw=None):
    from paper_2605_13276_b200 import grpo
    cfg = grpo.GrpoConfig(group_size=x.shape[1], **(cfg_kw or {}))
    loss, dl, st = _run_gpu(x, tokens, blp, rewards, ids, dtype, fused, cfg)
    oloss, odl, ost = O.grpo_token_grad(x, tokens, blp, rewards, ids, clip_eps=cfg.clip_eps,
                                        kl_coeff=cfg.kl_coeff)
    # chunk log-probs (f64 accumulate on both sides)
    lp = st["lp_chunk"].cpu().numpy()
    # |lp| ~ 600: an absolute 1e-5 keeps rho = exp(lp - blp) within 1e-5 relative
    np.testing.assert_allclose(lp, ost["lp_chunk"], rtol=1e-9, atol=1e-5)
    assert st["group_ids"] == ost["group_ids"]            # canonical order, exact
    assert st["n_chunks"] == ost["n_chunks"]
    scale = sum(abs(v) for v in ost["coeff"].ravel()) / max(ost["coeff"].size, 1)
    assert abs(loss - oloss) <= 1e-5 * max(abs(oloss), scale, 1e-12)
    assert st["mean_ratio"] == pytest.approx(ost["mean_ratio"], rel=1e-5)
    # per-chunk coefficients d loss / d lp (w included) and per-token lp
    n_edge, cond = _assert_coeff_close(st["coeff"].cpu().numpy(), ost, blp, rewards, rtol,
                                       cfg.clip_eps, cfg.kl_coeff)
    assert abs(st["clip_fraction"] - ost["clip_fraction"]) <= (n_edge + 0.5) / ost["n_chunks"]
    np.testing.assert_allclose(st["lp_tok"].cpu().numpy().reshape(-1), ost["lp_tok"],
                               rtol=0, atol=1e-6)
    # row-wise relative L2 + element-wise rtol on entries >= 1e-3 row max
    # (widened only for rows whose chunk coefficient cancels, KL runs)
    assert_dlogits_close(dl, odl.reshape(dl.shape), rtol, row_cond=cond)
    return st, ost


def test_f32_unfused_odd_vocab_matches_oracle():
    import torch
    case = _case(0, 3, 4, 2, 3, 257, torch.float32)
    _check(*case, torch.float32, fused=False, rtol=1e-5)


def test_f32_vectorised_rows_match_oracle():
    import torch
    case = _case(1, 2, 4, 2, 5, 1024, torch.float32, binary=False)
    _check(*case, torch.float32, fused=True, rtol=1e-5)   # fused f32, one piece per row


def test_bf16_fused_matches_oracle():
    import torch
    case = _case(2, 4, 8, 1, 56, 4096, torch.bfloat16)
    _check(*case, torch.bfloat16, fused=True, rtol=1e-2)


def test_bf16_fused_multi_chunk_kl_matches_oracle():
    import torch
    case = _case(3, 5, 4, 3, 7, 2048, torch.bfloat16, spread=0.5, binary=False)
    _check(*case, torch.bfloat16, fused=True, rtol=1e-2, cfg_kw={"kl_coeff": 0.3})


def test_bf16_unfused_matches_oracle():
    import torch
    case = _case(4, 2, 8, 1, 56, 4096, torch.bfloat16)
    _check(*case, torch.bfloat16, fused=False, rtol=1e-2)


def test_bf16_openvla_vocab_rows():
    """V = 32,064 (OpenVLA/Llama-2 padded vocab): the C2 row shape."""
    import torch
    case = _case(5, 2, 8, 1, 56, 32064, torch.bfloat16)
    _check(*case, torch.bfloat16, fused=True, rtol=1e-2)


def test_group_order_is_canonicalised_bitwise():
    import torch
    x, tokens, blp, rewards, ids = _case(6, 4, 8, 1, 56, 2048, torch.bfloat16)
    perm = np.array([2, 0, 3, 1])
    loss_a, dl_a, st_a = _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16)
    loss_b, dl_b, st_b = _run_gpu(x[perm], tokens[perm], blp[perm], rewards[perm], ids[perm],
                                  torch.bfloat16)
    assert loss_a == loss_b
    assert st_a["group_ids"] == st_b["group_ids"] == sorted(ids.tolist())
    R = dl_a.shape[0] // 4
    assert np.array_equal(dl_a.reshape(4, R, -1)[perm], dl_b.reshape(4, R, -1))


def test_fused_equals_unfused_forward_stats():
    import torch
    case = _case(7, 3, 8, 2, 9, 4096, torch.bfloat16, binary=False)
    la, _, sa = _run_gpu(*case, torch.bfloat16, fused=True)
    lb, _, sb = _run_gpu(*case, torch.bfloat16, fused=False)
    # different lse summation trees: ~1e-8 on lp, cancellation-amplified in the loss
    assert la == pytest.approx(lb, rel=1e-5, abs=1e-9)
    np.testing.assert_allclose(sa["lp_chunk"].cpu().numpy(), sb["lp_chunk"].cpu().numpy(),
                               rtol=1e-9, atol=1e-5)


def test_abort_on_nonfinite_reward_names_group():
    import torch
    from paper_2605_13276_b200.grpo import GrpoAbort
    x, tokens, blp, rewards, ids = _case(8, 3, 4, 1, 4, 512, torch.bfloat16, ids=[7, 3, 5])
    rewards[2, 1] = np.nan
    with pytest.raises(GrpoAbort, match="group 5.*non-finite reward") as exc:
        _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16)
    assert exc.value.group_id == 5


def test_abort_on_overflowing_ratio():
    import torch
    from paper_2605_13276_b200.grpo import GrpoAbort
    x, tokens, blp, rewards, ids = _case(9, 3, 4, 1, 4, 512, torch.bfloat16, ids=[7, 3, 5])
    blp[0, :, :] = -1e6
    with pytest.raises(GrpoAbort, match="group 7.*non-finite importance ratio"):
        _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16)


def test_abort_on_nonfinite_logit():
    import torch
    from paper_2605_13276_b200.grpo import GrpoAbort
    x, tokens, blp, rewards, ids = _case(10, 3, 4, 1, 4, 512, torch.float32, ids=[7, 3, 5])
    x[1, 2, 0, 1, 5] = np.inf
    with pytest.raises(GrpoAbort, match="group 3.*non-finite log-prob"):
        _run_gpu(x, tokens, blp, rewards, ids, torch.float32)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_bf16_abort_on_nonfinite_logit(bad, fused):
    """A NaN or +inf logit anywhere in a row poisons that row's lse in the
    fused bf16 path too (the reference's log-prob check, grpo.py:255-256)."""
    import torch
    from paper_2605_13276_b200.grpo import GrpoAbort
    x, tokens, blp, rewards, ids = _case(12, 3, 4, 1, 4, 4096, torch.bfloat16, ids=[7, 3, 5])
    x[1, 2, 0, 1, 3001] = bad   # not the target column, deep inside one warp's slice
    tokens[1, 2, 0, 1] = 17
    with pytest.raises(GrpoAbort, match="group 3.*non-finite log-prob"):
        _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16, fused=fused)


def test_fused_bf16_masked_logits_match_oracle():
    """-inf (masked) logits, including whole warp slices of -inf and rows
    with a large dynamic range, stay finite and match the oracle."""
    import torch
    x, tokens, blp, rewards, ids = _case(13, 2, 4, 1, 4, 4096, torch.bfloat16)
    x[0, 1, 0, 2, 1024:3072] = -np.inf
    x[1, 0, 0, 0, :] += 70.0            # beyond the speculative exp frame
    x[1, 3, 0, 3, :] -= 90.0
    x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()  # exact bf16 values again
    tokens[0, 1, 0, 2] = 5
    _, _, st0 = O.grpo_token_grad(x, tokens, np.zeros(blp.shape, np.float32),
                                  np.tile(np.arange(4, dtype=np.float32), (2, 1)),
                                  np.arange(2), want_dlogits=False)
    blp = (st0["lp_chunk"] + 0.01).astype(np.float32)
    _check(x, tokens, blp, rewards, ids, torch.bfloat16, True, 1e-2)


def test_token_out_of_range_is_usage_error():
    import torch
    from paper_2605_13276_b200.core import UsageError
    x, tokens, blp, rewards, ids = _case(11, 2, 4, 1, 4, 512, torch.bfloat16)
    tokens[0, 0, 0, 0] = 512
    with pytest.raises(UsageError, match="token"):
        _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16)


def _full_c2(dtype, seed, spread):
    """BASELINE config 2 at full size: 64 groups x G=8 x C=1 x T=56 x
    V=32,064 -- every chunk's lp and coefficient, the loss and the stats
    against the oracle; d loss / d logits on 1,024 sampled rows (all 512
    chunks' first rows + 512 random rows) with the row-wise criterion;
    size-independent properties on all 28,672 rows."""
    import torch
    from paper_2605_13276_b200 import grpo
    from oracle.check import dlogits_rows
    n_groups, G, C, T, V = 64, 8, 1, 56, 32064
    R = n_groups * G * C * T
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(seed)
    logits = (torch.randn(R, V, device=dev, generator=g) * 2).to(dtype)
    tokens = torch.randint(31744, 32000, (R,), device=dev, generator=g, dtype=torch.int32)
    rewards = torch.randint(0, 2, (n_groups * G,), device=dev, generator=g).float()
    rewards[: 2 * G] = torch.rand(2 * G, device=dev, generator=g)   # 2 groups of U(0,1)
    ids = np.random.default_rng(seed).permutation(4 * n_groups)[:n_groups]
    cfg = grpo.GrpoConfig(group_size=G)
    tl = grpo.TokenLoss(n_groups, G, C, T, V, cfg, dtype=dtype)
    tl.set_groups(ids)
    tl.launch(logits, tokens, torch.zeros(n_groups * G * C, device=dev), rewards, None)
    lp0 = tl.lp_chunk.clone()
    noise = (torch.rand(lp0.shape, device=dev, generator=g, dtype=torch.float64) - 0.5) * 2 * spread
    blp = (lp0 + noise).float()
    dl = torch.empty_like(logits)
    tl.launch(logits, tokens, blp, rewards, dl)
    st = tl.stats(rewards)
    torch.cuda.synchronize()
    # ---- oracle over the whole batch (forward: every row's lse and lp)
    x = logits.float().cpu().numpy().reshape(n_groups, G, C, T, V)
    tk = tokens.cpu().numpy().reshape(n_groups, G, C, T)
    bl = blp.cpu().numpy().reshape(n_groups, G, C)
    rw = rewards.cpu().numpy().reshape(n_groups, G)
    oloss, _, ost = O.grpo_token_grad(x, tk, bl, rw, ids, want_dlogits=False)
    assert st["n_chunks"] == ost["n_chunks"] == n_groups * G * C
    assert st["group_ids"] == ost["group_ids"]
    lp = tl.lp_chunk.cpu().numpy().reshape(n_groups, G, C)
    np.testing.assert_allclose(lp, ost["lp_chunk"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(tl.lp_tok.cpu().numpy(), ost["lp_tok"], rtol=0, atol=1e-6)
    co = tl.coeff.cpu().numpy().reshape(n_groups, G, C)
    rtol = 1e-5 if dtype == torch.float32 else 1e-2
    # coefficients: w * d_drho * rho (+ KL); rho = exp(lp - blp) carries the
    # lp error (<= 1e-5 absolute) as a relative error
    n_edge, _ = _assert_coeff_close(co, ost, bl, rw, 2e-5)
    scale = float(np.abs(ost["coeff"]).mean())
    assert abs(st["loss"] - oloss) <= 1e-5 * max(abs(oloss), scale), (st["loss"], oloss)
    assert st["mean_ratio"] == pytest.approx(ost["mean_ratio"], rel=1e-5)
    assert abs(st["clip_fraction"] - ost["clip_fraction"]) <= (n_edge + 0.5) / ost["n_chunks"]
    assert st["mean_reward"] == pytest.approx(float(np.mean([rw[k].mean() for k in range(n_groups)])),
                                              rel=1e-12)
    # ---- dlogits: 1,024 sampled rows against the oracle, row-wise
    rng = np.random.default_rng(seed + 1)
    rows = np.unique(np.concatenate([np.arange(0, R, T), rng.choice(R, 512, replace=False)]))
    want = dlogits_rows(x.reshape(R, V)[rows], tk.reshape(R)[rows], ost["lse"][rows],
                        np.repeat(ost["coeff"].reshape(-1), T)[rows])
    got = dl[torch.from_numpy(rows).to(dev)].float().cpu().numpy()
    err = assert_dlogits_close(got, want, rtol)
    # ---- all rows: the softmax Jacobian's rows sum to 0 (storage rounding
    # only), and rows of zero-coefficient chunks are exactly zero
    rs = dl.float().sum(dim=1).abs().max().item()
    assert rs <= (1e-2 if dtype == torch.bfloat16 else 1e-5) * dl.float().abs().max().item()
    zero_rows = torch.from_numpy(np.repeat(ost["coeff"].reshape(-1) == 0.0, T)).to(dev)
    assert int((dl[zero_rows] != 0).sum().item()) == 0
    return err


@pytest.mark.parametrize("spread", [0.05, 0.5])
def test_full_c2_bf16_matches_oracle(spread):
    import torch
    _full_c2(torch.bfloat16, 0, spread)


def test_full_c2_f32_matches_oracle():
    import torch
    _full_c2(torch.float32, 1, 0.05)


def test_long_chunks_fall_back_to_unfused_kernels():
    """T > 128 tokens per chunk exceeds the fused warp-pairwise path."""
    import torch
    case = _case(12, 2, 4, 1, 160, 1024, torch.bfloat16)
    _check(*case, torch.bfloat16, fused=True, rtol=1e-2)


def test_f32_openvla_vocab_matches_oracle():
    import torch
    case = _case(13, 2, 4, 1, 8, 32064, torch.float32, binary=False)
    _check(*case, torch.float32, fused=True, rtol=1e-5)


@pytest.mark.parametrize("dtype_name,V", [("float32", 32064), ("bfloat16", 65536),
                                          ("bfloat16", 128256)])
def test_fused_rows_split_into_pieces_match_oracle(dtype_name, V):
    """Rows longer than one SMEM stage stream as 2 or 4 pieces (f32 at the
    C2 vocabulary; bf16 at 64K / Llama-3's 128,256): the tail warp combines
    the pieces' partials, the target may sit in any piece."""
    import torch
    dtype = getattr(torch, dtype_name)
    x, tokens, blp, rewards, ids = _case(21, 2, 4, 2, 6, V, dtype, binary=False)
    tokens[0, 0, 0, :] = [0, V // 2 - 1, V // 2, V - 1, V // 4, 3 * V // 4]  # piece edges
    _, _, st0 = O.grpo_token_grad(x, tokens, np.zeros(blp.shape, np.float32),
                                  np.tile(np.arange(4, dtype=np.float32), (2, 1)),
                                  np.arange(2), want_dlogits=False)
    blp = (st0["lp_chunk"] + 0.02).astype(np.float32)
    case = (x, tokens, blp, rewards, ids)
    rtol = 1e-5 if dtype == torch.float32 else 1e-2
    _check(*case, dtype, fused=True, rtol=rtol)
    la, _, sa = _run_gpu(*case, dtype, fused=True)
    lb, _, sb = _run_gpu(*case, dtype, fused=False)
    np.testing.assert_allclose(sa["lp_chunk"].cpu().numpy(), sb["lp_chunk"].cpu().numpy(),
                               rtol=1e-9, atol=1e-5)
    # forward-only (loss evaluation) through the same pieces
    from paper_2605_13276_b200 import grpo
    dev = torch.device("cuda", 0)
    lf, dlf, sf = grpo.grpo_token_grad(
        torch.from_numpy(x).to(dev, dtype), torch.from_numpy(tokens).to(dev),
        torch.from_numpy(blp).to(dev), torch.from_numpy(rewards).to(dev), ids,
        grpo.GrpoConfig(group_size=4), write_dlogits=False)
    assert dlf is None
    np.testing.assert_allclose(sf["lp_chunk"].cpu().numpy(), sa["lp_chunk"].cpu().numpy(),
                               rtol=0, atol=1e-12)
    assert lf == pytest.approx(la, rel=1e-12, abs=1e-15)


def test_misaligned_logits_take_the_scalar_path():
    """A logits view starting one element into its storage (not 16-byte
    aligned) must still be exact: the C-ABI picks the scalar kernels."""
    import torch
    from paper_2605_13276_b200 import grpo
    x, tokens, blp, rewards, ids = _case(14, 2, 4, 1, 3, 256, torch.float32)
    dev = torch.device("cuda", 0)
    R, V = x.reshape(-1, 256).shape
    store = torch.empty(R * V + 1, dtype=torch.float32, device=dev)
    lg = store[1:].view(R, V)
    lg.copy_(torch.from_numpy(x.reshape(R, V)).to(dev))
    cfg = grpo.GrpoConfig(group_size=4)
    tl = grpo.TokenLoss(2, 4, 1, 3, V, cfg, dtype=torch.float32)
    tl.set_groups(ids)
    dl = torch.empty(R * V + 1, dtype=torch.float32, device=dev)[1:].view(R, V)
    tl.launch(lg, torch.from_numpy(tokens.reshape(-1)).to(dev),
              torch.from_numpy(blp.reshape(-1)).to(dev), torch.from_numpy(rewards.reshape(-1)).to(dev),
              dl)
    st = tl.stats(torch.from_numpy(rewards.reshape(-1)))
    oloss, odl, ost = O.grpo_token_grad(x, tokens, blp, rewards, ids)
    scale = np.abs(ost["coeff"]).mean()
    assert abs(st["loss"] - oloss) <= 1e-5 * max(abs(oloss), scale)
    assert_dlogits_close(dl.cpu().numpy(), odl.reshape(R, V), 1e-5)


def test_zero_advantage_groups_give_zero_gradient_rows():
    """All-success / all-fail groups have A = 0 -> coefficient 0 -> the fused
    kernel's zero-row fast path must write exact zeros (and count them as
    clipped, reference grpo.py:272-273)."""
    import torch
    x, tokens, blp, rewards, ids = _case(15, 3, 8, 1, 56, 4096, torch.bfloat16)
    rewards[:] = 1.0
    loss, dl, st = _run_gpu(x, tokens, blp, rewards, ids, torch.bfloat16)
    assert np.all(dl == 0.0)
    assert st["clip_fraction"] == 1.0 and loss == 0.0


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_match_oracle(seed):
    """Randomised batch shapes, dtypes, vocabularies (incl. ones that are not
    16-byte row multiples), group ids and KL settings against the oracle,
    through whichever kernel path the C-ABI selects."""
    import torch
    rng = np.random.default_rng(1000 + seed)
    n_groups = int(rng.integers(1, 6))
    G = int(rng.integers(2, 10))
    C = int(rng.integers(1, 4))
    T = int(rng.integers(1, 21))
    V = int(rng.choice([8, 24, 200, 1000, 2048, 3001, 4096 + 8]))
    dtype = torch.bfloat16 if rng.random() < 0.6 else torch.float32
    fused = bool(rng.random() < 0.8)
    kl = float(rng.choice([0.0, 0.0, 0.2]))
    ids = rng.permutation(n_groups * 5)[:n_groups]
    case = _case(2000 + seed, n_groups, G, C, T, V, dtype, spread=float(rng.choice([0.05, 0.5])),
                 binary=bool(rng.random() < 0.5), ids=ids)
    rtol = 1e-5 if dtype == torch.float32 else 1e-2
    _check(*case, dtype, fused=fused, rtol=rtol, cfg_kw={"kl_coeff": kl})


def test_back_to_back_launches_see_their_own_inputs():
    """The fused kernel and the epilogue are launched with programmatic
    dependent launch: three calls queued back to back on one stream (no
    host sync between them) with different rewards / behaviour log-probs /
    logits must each match the oracle on their own inputs -- no call may
    read the previous call's advantages, pending markers or chunk lps."""
    import torch
    from paper_2605_13276_b200 import grpo
    dev = torch.device("cuda", 0)
    n_groups, G, C, T, V = 6, 4, 1, 8, 4096
    cases = [_case(40 + k, n_groups, G, C, T, V, torch.bfloat16, ids=np.arange(n_groups))
             for k in range(3)]
    tl = grpo.TokenLoss(n_groups, G, C, T, V, grpo.GrpoConfig(group_size=G),
                        dtype=torch.bfloat16, device=dev)
    tl.set_groups(np.arange(n_groups))
    outs = []
    for x, tokens, blp, rewards, _ in cases:
        lg = torch.from_numpy(x).to(dev, torch.bfloat16).reshape(-1, V)
        dl = torch.empty_like(lg)
        rw = torch.from_numpy(rewards.reshape(-1)).to(dev)
        tl.launch(lg, torch.from_numpy(tokens.reshape(-1)).to(dev),
                  torch.from_numpy(blp.reshape(-1)).to(dev), rw, dl)
        outs.append((dl, tl.lp_chunk.clone(), tl.stats_dev.clone(), rw))
    torch.cuda.synchronize()
    from paper_2605_13276_b200 import _lib
    for (x, tokens, blp, rewards, ids), (dl, lp, st, _) in zip(cases, outs):
        oloss, odl, ost = O.grpo_token_grad(x, tokens, blp, rewards, ids)
        np.testing.assert_allclose(lp.cpu().numpy(), ost["lp_chunk"].reshape(-1),
                                   rtol=1e-9, atol=1e-5)
        sv = st.cpu().numpy()
        assert sv[_lib.ST_ABORT] == 0 and sv[_lib.ST_KERNEL_ERR] == 0
        assert sv[_lib.ST_CHUNK_COUNT] == ost["n_chunks"]
        scale = sum(abs(v) for v in ost["coeff"].ravel()) / max(ost["coeff"].size, 1)
        assert abs(sv[_lib.ST_LOSS] - oloss) <= 1e-5 * max(abs(oloss), scale, 1e-12)
        assert_dlogits_close(dl.float().cpu().numpy(), odl.reshape(dl.shape), 1e-2)


@pytest.mark.parametrize("priority", [-1, 0])
def test_fused_kernel_beside_gemms_on_another_stream(priority):
    """The fused kernel's CTAs wait on each other's published token
    log-probs, so it needs all of its CTAs resident.  Launched while another
    stream's GEMMs hold the SMs (the swimlane's sampler beside the trainer),
    it must still finish -- its CTAs become resident as the GEMM CTAs retire
    (no deadlock: resident fused CTAs never wait on the GEMM) -- without the
    spin timeout (ST_KERNEL_ERR) and with the oracle's result, on a
    high-priority stream (the trainer's) and a default-priority one."""
    import torch
    from paper_2605_13276_b200 import grpo
    dev = torch.device("cuda", 0)
    x, tokens, blp, rewards, ids = _case(41, 4, 8, 1, 56, 32064, torch.bfloat16)
    cfg = grpo.GrpoConfig(group_size=8)
    R, V = 4 * 8 * 56, 32064
    tl = grpo.TokenLoss(4, 8, 1, 56, V, cfg, dtype=torch.bfloat16, device=dev)
    tl.set_groups(ids)
    lg = torch.from_numpy(x.reshape(R, V)).to(dev, torch.bfloat16)
    tk = torch.from_numpy(tokens.reshape(-1)).to(dev)
    bl = torch.from_numpy(blp.reshape(-1)).to(dev)
    rw = torch.from_numpy(rewards.reshape(-1)).to(dev)
    dl = torch.empty_like(lg)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    side = torch.cuda.Stream(device=dev)
    mine = torch.cuda.Stream(device=dev, priority=priority)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    started = torch.cuda.Event()
    with torch.cuda.stream(side):
        torch.mm(a, b)
        started.record(side)
        for _ in range(11):                          # ~10 ms more GEMM CTAs on every SM
            torch.mm(a, b)
    with torch.cuda.stream(mine):
        mine.wait_event(started)                     # launched while the GEMMs run
        e0.record(mine)
        tl.launch(lg, tk, bl, rw, dl, stream=mine)
        e1.record(mine)
    torch.cuda.synchronize()
    st = tl.stats(rewards)                           # raises on ST_KERNEL_ERR (timeout)
    oloss, odl, ost = O.grpo_token_grad(x, tokens, blp, rewards, ids)
    scale = float(np.abs(ost["coeff"]).mean())
    assert abs(st["loss"] - oloss) <= 1e-5 * max(abs(oloss), scale)
    assert_dlogits_close(dl.float().cpu().numpy(), odl.reshape(R, V), 1e-2)
    print(f"fused loss beside GEMMs (priority {priority}): {e0.elapsed_time(e1):.2f} ms")
