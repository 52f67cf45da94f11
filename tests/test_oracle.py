"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import grpo_oracle as O


def test_oracle_advantages_bitwise_against_reference():
    g = golden("advantages")
    offs = g["offsets"]
    for a, b in zip(offs[:-1], offs[1:]):
        got = O.compute_advantages(g["rewards"][a:b], float(g["delta"]))
        assert np.array_equal(got, g["adv"][a:b]), (a, b)


def test_oracle_reproduces_nondyadic_constant_quirk():
    # three identical non-dyadic rewards give A != 0
    g = golden("advantages")
    kinds = g["kinds"]
    idx = int(np.flatnonzero(kinds == 9)[0])
    a, b = g["offsets"][idx], g["offsets"][idx + 1]
    adv = g["adv"][a:b]
    assert np.all(adv != 0.0) and np.all(np.abs(adv) < 1e-4)


@pytest.mark.parametrize("ratio,adv,eps,want", [
    (1.3, 1.0, 0.2, (-1.2, 0.0)),
    (0.7, -1.0, 0.2, (0.8, 0.0)),
    (0.95, 2.0, 0.2, (-1.9, -2.0)),
    (1.0, 1.5, 0.2, (-1.5, -1.5)),
    (1.0, -1.5, 0.2, (1.5, 1.5)),
])
def test_oracle_surrogate_kats(ratio, adv, eps, want):
    loss, d = O.clipped_surrogate(ratio, adv, eps)
    assert loss == pytest.approx(want[0]) and d == want[1]


def _gauss_case(g, tag):
    return dict(w1=g[f"{tag}_w1"], b1=g[f"{tag}_b1"], w2=g[f"{tag}_w2"], b2=g[f"{tag}_b2"],
                log_std=g[f"{tag}_log_std"], group_ids=g[f"{tag}_group_ids"],
                obs=g[f"{tag}_obs"], actions=g[f"{tag}_actions"], blp=g[f"{tag}_blp"],
                rewards=g[f"{tag}_rewards"])


def test_oracle_grpo_grad_gauss_matches_reference():
    g = golden("grpo_gauss")
    tags = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_loss")})
    assert len(tags) == 12
    for tag in tags:
        case = _gauss_case(g, tag)
        loss, grad, st = O.grpo_grad_gauss(**case, kl_coeff=float(g[f"{tag}_kl"]))
        # The reference's default numba backend evaluates float(x) of f32
        # array elements in f32 (its jitted chunk_log_prob differs from its own
        # py_func by ~4e-8 rel), its numpy backend in f64; the two agree only
        # to rtol 1e-6 (reference tests/test_kernels.py:59,79).  The oracle
        # follows the documented f64 contract, so the pin is that tolerance.
        assert loss == pytest.approx(float(g[f"{tag}_loss"]), abs=1e-6)
        ref = g[f"{tag}_grad"]
        assert np.abs(grad - ref).max() <= 1e-5 * np.abs(ref).max()
        rs = g[f"{tag}_stats"]
        assert st["mean_ratio"] == pytest.approx(rs[1], rel=1e-6)
        assert st["clip_fraction"] == rs[2] and st["n_chunks"] == rs[3]


def test_oracle_adam_matches_reference_update():
    g = golden("grpo_gauss")
    for seed in range(10):
        tag = f"s{seed}_kl0"
        case = _gauss_case(g, tag)
        _, grad, _ = O.grpo_grad_gauss(**case)
        flat = np.concatenate([case[k].ravel() for k in ("w1", "b1", "w2", "b2", "log_std")])
        norm, grad = O.clip_grad_norm(grad, None)
        assert norm == pytest.approx(float(g[f"{tag}_grad_norm"]), rel=1e-6)
        new, *_ = O.adam_step(flat, g[f"{tag}_grad"], np.zeros(flat.size), np.zeros(flat.size),
                              0, 1e-3, 0.9, 0.999, 1e-8)
        assert np.array_equal(new, g[f"{tag}_updated"])  # bitwise on the reference grad


def test_oracle_kernels_match_reference_backend():
    g = golden("kernels")
    lp = O.chunk_log_prob(g["means"], g["log_std"], g["actions"])
    np.testing.assert_allclose(lp, g["lp"], rtol=1e-6)
    mf = O.mlp_forward(g["w1"], g["b1"], g["w2"], g["b2"], g["obs"])
    np.testing.assert_allclose(mf, g["mlp_out"], rtol=1e-6, atol=1e-7)
    out = np.zeros_like(g["backward"])
    O.policy_backward(g["w1"], g["b1"], g["w2"], g["b2"], g["ls2"], g["obs"], g["act"],
                      g["coeffs"], out)
    np.testing.assert_allclose(out, g["backward"], rtol=1e-5, atol=1e-6 * np.abs(out).max())


def test_token_oracle_epilogue_equals_gaussian_epilogue():
    """Cross-check of the unpinned token head: feed the token
    restatement's epilogue the Gaussian chunk log-probs of a pinned case and
    require the reference loss/stats."""
    g = golden("grpo_gauss")
    tag = "s2_kl0"
    case = _gauss_case(g, tag)
    n_groups, G, C = case["blp"].shape
    lp = np.zeros((n_groups, G, C))
    for k in range(n_groups):
        for i in range(G):
            means = O.mlp_forward(case["w1"], case["b1"], case["w2"], case["b2"], case["obs"][k, i])
            lp[k, i] = O.chunk_log_prob(means, case["log_std"], case["actions"][k, i])
    order, entries = O._entries(case["group_ids"], case["rewards"], case["blp"], G, 1e-8)
    loss, ratio_sum, clip, n, _ = O._epilogue(lambda key: lp[key], entries, n_groups * G, 0.2, 0.0)
    assert loss == pytest.approx(float(g[f"{tag}_loss"]), abs=1e-6)
    assert n == int(g[f"{tag}_stats"][3])


def test_token_oracle_small_case_properties():
    rng = np.random.default_rng(0)
    n_groups, G, C, T, V = 2, 4, 2, 3, 17
    logits = rng.normal(0, 2, (n_groups, G, C, T, V)).astype(np.float32)
    tokens = rng.integers(0, V, (n_groups, G, C, T))
    blp = rng.normal(-8, 1, (n_groups, G, C)).astype(np.float32)
    rewards = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
    loss, dl, st = O.grpo_token_grad(logits, tokens, blp, rewards, np.array([5, 2]))
    assert st["group_ids"] == [2, 5]
    # each dlogits row sums to zero (softmax Jacobian rows) times coeff
    np.testing.assert_allclose(dl.sum(axis=-1), 0.0, atol=1e-12)
    # lp_tok <= 0 and lp_chunk is the per-chunk sum
    assert np.all(st["lp_tok"] <= 0)
    np.testing.assert_allclose(st["lp_chunk"].reshape(-1), st["lp_tok"].reshape(-1, T).sum(1),
                               rtol=1e-13)


def _pairwise(a):
    """numpy pairwise_sum restated (loops_utils.h) -- used by the GPU kernels."""
    n = len(a)
    if n < 8:
        s = 0.0
        for x in a:
            s += x
        return s
    if n <= 128:
        r = list(a[:8])
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for x in a[i:]:
            s += x
        return s
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a[:n2]) + _pairwise(a[n2:])


@pytest.mark.parametrize("T", [1, 3, 7, 8, 9, 15, 16, 56, 57, 100, 128, 129, 300])
def test_row_sum_is_numpy_pairwise_bitwise(T):
    """The chunk-lp order the kernels implement (numpy pairwise) is what
    ndarray.sum(axis=1) computes on contiguous rows."""
    x = np.random.default_rng(T).normal(-10, 3, (5, T))
    got = x.sum(axis=1)
    for i in range(5):
        assert got[i] == _pairwise(list(x[i])), T


def test_oracle_alloc_trace_matches_reference_golden_bitwise():
    """The C restatement of alloc_trace_run (oracle/arena_oracle.c) against
    the reference's own traces (tests/golden/alloc_traces.npz)."""
    from oracle.arena import alloc_trace
    from paper_2605_13276_b200.pools import random_workload
    g = golden("alloc_traces")
    for seed in (0, 1, 11, 17, 5):
        cap, n = int(g[f"s{seed}_cap"]), int(g[f"s{seed}_n"])
        ok, off, fin = alloc_trace(cap, *random_workload(seed, n, cap))
        assert np.array_equal(ok, g[f"s{seed}_ok"]), seed
        assert np.array_equal(off, g[f"s{seed}_off"]), seed
        assert fin == tuple(int(x) for x in g[f"s{seed}_final"]), seed


def test_oracle_alloc_trace_edge_cases():
    from oracle.arena import alloc_trace
    # free with nothing live, exact fit, no fit, and a full coalesce back to one extent
    ok, off, fin = alloc_trace(256, [0, 1, 1, 1, 0, 0], [0, 128, 128, 1, 0, 0],
                               [1, 64, 1, 1, 1, 1], [0, 0, 0, 0, 5, 0])
    assert ok.tolist() == [2, 1, 1, 0, 3, 3]
    assert off.tolist() == [-1, 0, 128, -1, 128, 0]
    assert fin == (256, 256, 1)
    ok, off, fin = alloc_trace(100, [], [], [], [])
    assert len(ok) == 0 and fin == (100, 100, 1)


def test_dlogits_criterion_sees_off_target_errors():
    """The row-wise criterion (oracle/check.py) must reject a systematic
    10 % error on every off-target softmax entry at V = 32,064 -- the error a
    max-scaled tolerance cannot see -- and accept the exact gradient."""
    from oracle.check import dlogits_errors, dlogits_rows
    rng = np.random.default_rng(0)
    V = 32064
    x = rng.normal(0, 2, (4, V))
    tok = rng.integers(0, V, 4)
    lse = np.log(np.exp(x).sum(axis=1))
    want = dlogits_rows(x, tok, lse, np.array([1e-3, -2e-3, 0.0, 5e-4]))
    assert dlogits_errors(want, want) == (0.0, 0.0, 0)
    bad = want.copy()
    off = np.ones_like(bad, dtype=bool)
    off[np.arange(4), tok] = False
    bad[off] *= 1.1
    row_l2, elem, nz = dlogits_errors(bad, want)
    assert nz == 0 and elem > 0.05
    # max-scaled check would pass this
    assert np.all(np.abs(bad - want) <= 1e-2 * (np.abs(want) + np.abs(want).max()))
    # a nonzero value in a zero-coefficient row is counted
    bad2 = want.copy()
    bad2[2, 0] = 1e-30
    assert dlogits_errors(bad2, want)[2] == 1


def test_coefficient_condition_widens_only_cancelling_rows():
    from oracle.check import coeff_term_scale, row_condition
    lp = np.full((1, 2, 1), -10.0)
    blp = np.array([[[-10.0], [-10.0]]], np.float32)
    rw = np.array([[0.0, 1.0]], np.float32)
    s = coeff_term_scale(lp, blp, rw, kl_coeff=0.0)
    # w = 1/2; A = -+1/(0.5 + 1e-8); rho = 1
    np.testing.assert_allclose(s.ravel(), 0.5 * 0.5 / (0.5 + 1e-8))
    coeff = np.array([s.ravel()[0], 1e-6 * s.ravel()[1]])
    rc = row_condition(coeff, s, 3)
    assert rc.shape == (6,) and np.all(rc[:3] == 1.0) and np.allclose(rc[3:], 1e6)


def test_mean_reward_matches_the_per_group_definition():
    """grpo._mean_reward (one row-wise reduction) is bit-identical to the
    reference's float(np.mean([b.rewards.mean() for b in batches]))
    (grpo.py:291) in canonical order, for many group sizes."""
    from paper_2605_13276_b200.grpo import _mean_reward
    rng = np.random.default_rng(5)
    for G in list(range(2, 40)) + [64, 127, 128, 129, 300]:
        for n_groups in (1, 3, 64):
            r = (rng.standard_normal((n_groups, G)) * rng.uniform(0.01, 100)).astype(np.float32)
            order = rng.permutation(n_groups)
            want = float(np.mean([r[k].mean() for k in order]))
            assert _mean_reward(r, order) == want, (G, n_groups)
