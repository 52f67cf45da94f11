"""Reference-shaped learner on the GPU vs golden vectors produced by the
reference itself (tests/golden/make_golden.py): advantages (bitwise), the
Gaussian-MLP grpo_grad, Adam (bitwise), kernels, aborts."""

import numpy as np
import pytest

from conftest import golden
from oracle import grpo_oracle as O

pytestmark = pytest.mark.gpu


def _tags(g):
    return sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_loss")})


def _case(g, tag):
    from paper_2605_13276_b200.grpo import GroupBatch
    from paper_2605_13276_b200.policy import PolicyParams
    params = PolicyParams(w1=g[f"{tag}_w1"].copy(), b1=g[f"{tag}_b1"].copy(),
                          w2=g[f"{tag}_w2"].copy(), b2=g[f"{tag}_b2"].copy(),
                          log_std=g[f"{tag}_log_std"].copy())
    batches = []
    for k, gid in enumerate(g[f"{tag}_group_ids"]):
        batches.append(GroupBatch(
            group_id=int(gid), horizon=8, chunk=4, obs=g[f"{tag}_obs"][k].copy(),
            actions=g[f"{tag}_actions"][k].copy(), behavior_log_prob=g[f"{tag}_blp"][k].copy(),
            rewards=g[f"{tag}_rewards"][k].copy(), behavior_version=0))
    return params, batches


def test_advantages_bitwise_against_reference(dev):
    from paper_2605_13276_b200.grpo import compute_advantages
    g = golden("advantages")
    offs = g["offsets"]
    for a, b in zip(offs[:-1], offs[1:]):
        got = compute_advantages(g["rewards"][a:b], float(g["delta"]))
        assert got.dtype == np.float64
        assert np.array_equal(got, g["adv"][a:b]), (a, b)


def test_advantages_known_answers(dev):
    from paper_2605_13276_b200.grpo import compute_advantages
    np.testing.assert_allclose(compute_advantages([1.0, 0.0, 0.0, 1.0], 1e-8), [1, -1, -1, 1],
                               rtol=1e-7)
    assert np.all(compute_advantages([1.0, 1.0, 1.0, 1.0], 1e-8) == 0.0)
    from paper_2605_13276_b200.core import ConfigError
    with pytest.raises(ConfigError):
        compute_advantages([1.0], 1e-8)


def test_grpo_grad_matches_reference_golden(dev):
    from paper_2605_13276_b200 import grpo
    g = golden("grpo_gauss")
    tags = _tags(g)
    assert len(tags) == 12
    for tag in tags:
        params, batches = _case(g, tag)
        cfg = grpo.GrpoConfig(group_size=4, clip_eps=0.2, adv_epsilon=1e-8, micro_batch=4,
                              lr=1e-3, kl_coeff=float(g[f"{tag}_kl"]))
        loss, grad, st = grpo.grpo_grad(params, batches, cfg)
        ref = g[f"{tag}_grad"]
        # the reference's default numba backend evaluates part of the
        # log-density in f32 (see tests/test_oracle.py): pin at its own
        # inter-backend tolerance, and tighter against the f64 oracle below
        assert loss == pytest.approx(float(g[f"{tag}_loss"]), abs=1e-6)
        assert np.abs(grad - ref).max() <= 1e-5 * np.abs(ref).max()
        rs = g[f"{tag}_stats"]
        assert st["mean_ratio"] == pytest.approx(rs[1], rel=1e-6)
        assert st["clip_fraction"] == rs[2] and st["n_chunks"] == rs[3]
        assert st["mean_reward"] == rs[4]
        # against the f64 oracle restatement: much tighter
        oloss, ograd, _ = O.grpo_grad_gauss(
            params.w1, params.b1, params.w2, params.b2, params.log_std,
            g[f"{tag}_group_ids"], g[f"{tag}_obs"], g[f"{tag}_actions"], g[f"{tag}_blp"],
            g[f"{tag}_rewards"], kl_coeff=cfg.kl_coeff)
        assert loss == pytest.approx(oloss, rel=1e-9, abs=1e-13)
        assert np.abs(grad - ograd).max() <= 1e-9 * np.abs(ograd).max()


def test_batch_order_is_canonicalised_bitwise(dev):
    from paper_2605_13276_b200 import grpo
    g = golden("grpo_gauss")
    params, batches = _case(g, "s5_kl0")
    cfg = grpo.GrpoConfig(group_size=4, micro_batch=4)
    la, ga, sa = grpo.grpo_grad(params, batches, cfg)
    lb, gb, sb = grpo.grpo_grad(params, batches[::-1], cfg)
    assert la == lb and sa["group_ids"] == sb["group_ids"] == [0, 1]
    np.testing.assert_allclose(ga, gb, rtol=1e-13, atol=1e-16)


def test_aborts_carry_group_and_message(dev):
    from paper_2605_13276_b200 import grpo
    from paper_2605_13276_b200.core import ConfigError
    g = golden("grpo_gauss")
    cfg = grpo.GrpoConfig(group_size=4, micro_batch=4)
    params, batches = _case(g, "s1_kl0")
    batches[1].rewards[0] = np.nan
    with pytest.raises(grpo.GrpoAbort, match="group 1.*non-finite reward") as exc:
        grpo.grpo_grad(params, batches, cfg)
    assert exc.value.group_id == 1
    params, batches = _case(g, "s2_kl0")
    params.w2[0, 0] = np.nan
    with pytest.raises(grpo.GrpoAbort, match="non-finite log-prob"):
        grpo.grpo_grad(params, batches, cfg)
    params, batches = _case(g, "s6_kl0")
    batches[0].behavior_log_prob[:] = -1e6
    with pytest.raises(grpo.GrpoAbort, match="non-finite importance ratio"):
        grpo.grpo_grad(params, batches, cfg)
    with pytest.raises(ConfigError, match="at least one group"):
        grpo.grpo_grad(params, [], cfg)
    params, batches = _case(g, "s0_kl0")
    with pytest.raises(ConfigError, match="group 0 has 4"):
        grpo.grpo_grad(params, batches, grpo.GrpoConfig(group_size=8))


def test_adam_is_bitwise_on_the_reference_gradient(dev):
    from paper_2605_13276_b200 import grpo
    g = golden("grpo_gauss")
    cfg = grpo.GrpoConfig(lr=1e-3)
    for seed in range(10):
        tag = f"s{seed}_kl0"
        flat = np.concatenate([g[f"{tag}_{k}"].ravel() for k in ("w1", "b1", "w2", "b2",
                                                                  "log_std")]).astype(np.float32)
        st = grpo.AdamState.zeros(flat.size)
        grpo.adam_step(flat, g[f"{tag}_grad"].copy(), st, cfg)
        assert st.step == 1
        assert np.array_equal(flat, g[f"{tag}_updated"]), seed


def test_adam_known_answers(dev):
    from paper_2605_13276_b200 import grpo
    p = np.zeros(3, dtype=np.float32)
    st = grpo.AdamState.zeros(3)
    out = grpo.adam_step(p, np.ones(3), st, grpo.GrpoConfig(lr=0.1))
    assert out is p
    np.testing.assert_allclose(p, -0.1, rtol=1e-6)
    for scale in (1e-3, 1.0, 1e3):
        q = np.zeros(2, dtype=np.float32)
        grpo.adam_step(q, np.full(2, scale), grpo.AdamState.zeros(2), grpo.GrpoConfig(lr=0.05))
        np.testing.assert_allclose(q, -0.05, rtol=1e-5)


def test_clip_grad_norm(dev):
    from paper_2605_13276_b200 import grpo
    gv = np.array([3.0, 4.0])
    assert grpo.clip_grad_norm(gv, 2.5) == pytest.approx(5.0)
    np.testing.assert_allclose(gv, [1.5, 2.0])
    g2 = np.array([3.0, 4.0])
    assert grpo.clip_grad_norm(g2, None) == pytest.approx(5.0)
    np.testing.assert_allclose(g2, [3.0, 4.0])


def test_grpo_update_matches_reference(dev):
    from paper_2605_13276_b200 import grpo
    from paper_2605_13276_b200.policy import flatten
    g = golden("grpo_gauss")
    params, batches = _case(g, "s8_kl0")
    cfg = grpo.GrpoConfig(group_size=4, micro_batch=4, lr=1e-3)
    adam = grpo.AdamState.zeros(params.n_params)
    newp, ust = grpo.grpo_update(params, batches, cfg, adam, 4)
    assert ust.version == 5 and adam.step == 1
    assert ust.n_traj == 8 and ust.n_groups == 2 and ust.n_chunks == 16
    np.testing.assert_allclose(flatten(newp), g["s8_kl0_updated"], rtol=0, atol=2e-7)
    assert ust.grad_norm == pytest.approx(float(g["s8_kl0_grad_norm"]), rel=1e-5)


def test_kernels_match_reference_backend(dev):
    from paper_2605_13276_b200 import kernels
    g = golden("kernels")
    np.testing.assert_allclose(kernels.chunk_log_prob(g["means"], g["log_std"], g["actions"]),
                               g["lp"], rtol=1e-6)
    np.testing.assert_allclose(kernels.mlp_forward(g["w1"], g["b1"], g["w2"], g["b2"], g["obs"]),
                               g["mlp_out"], rtol=1e-6, atol=1e-6)
    out = np.zeros_like(g["backward"])
    kernels.policy_backward(g["w1"], g["b1"], g["w2"], g["b2"], g["ls2"], g["obs"], g["act"],
                            g["coeffs"], out)
    np.testing.assert_allclose(out, g["backward"], rtol=1e-5, atol=1e-6 * np.abs(out).max())
    # accumulates (+=), like the reference
    kernels.policy_backward(g["w1"], g["b1"], g["w2"], g["b2"], g["ls2"], g["obs"], g["act"],
                            g["coeffs"], out)
    np.testing.assert_allclose(out, 2 * g["backward"], rtol=1e-5, atol=2e-6 * np.abs(out).max())


def test_policy_closed_forms(dev):
    from paper_2605_13276_b200.policy import PolicyParams, backward, log_prob_of
    LOG_2PI = float(np.log(2 * np.pi))
    z = lambda ls: PolicyParams(w1=np.zeros((4, 3), np.float32), b1=np.zeros(4, np.float32),
                                w2=np.zeros((2, 4), np.float32), b2=np.zeros(2, np.float32),
                                log_std=np.full(2, ls, np.float32))
    obs = np.zeros(3, np.float32)
    assert log_prob_of(z(0.0), obs, np.zeros(2, np.float32)) == pytest.approx(-LOG_2PI, abs=1e-6)
    assert log_prob_of(z(0.0), obs, np.array([1.0, 0.0], np.float32)) == pytest.approx(
        -2.337877, abs=1e-5)
    at = log_prob_of(z(-0.3), obs, np.zeros(2, np.float32))
    sh = np.array([np.exp(-0.3), 0.0], np.float32)
    assert log_prob_of(z(-0.3), obs, sh) == pytest.approx(at - 0.5, abs=1e-5)
    gr = backward(z(0.2), obs, np.zeros(2, np.float32), upstream=2.0)
    np.testing.assert_allclose(gr[-2:], -2.0, rtol=1e-6)


def test_gauss_head_backward_c3_shape(dev):
    """pi0-shaped action expert head (BASELINE config 3): D = 1,600."""
    import torch
    from paper_2605_13276_b200 import kernels
    rng = np.random.default_rng(0)
    B, D = 512, 1600
    means = rng.normal(0, 1, (B, D)).astype(np.float32)
    actions = rng.normal(0, 1, (B, D)).astype(np.float32)
    log_std = rng.normal(0, 0.1, D).astype(np.float32)
    c = rng.normal(0, 1e-3, B)
    lp = kernels.chunk_log_prob(means, log_std, actions)
    np.testing.assert_allclose(lp, O.chunk_log_prob(means, log_std, actions), rtol=1e-12)
    dm, dls = kernels.gauss_head_backward(means, log_std, actions, c)
    odm, odls = O.gauss_head_backward(means, log_std, actions, c)
    np.testing.assert_allclose(dm, odm, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(dls, odls, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("C,kl", [(1, 0.0), (3, 0.1)])
def test_gauss_loss_one_call_matches_oracle(dev, C, kl):
    """dvla_gauss_loss_fwd_bwd (advantages -> chunk_log_prob -> canonical
    epilogue -> head backward in one C call) against the f64 oracle, with
    permuted group ids, several chunks per trajectory and the KL term."""
    import torch
    from paper_2605_13276_b200 import grpo
    rng = np.random.default_rng(1 + C)
    n_groups, G, D = 6, 4, 1600
    ids = np.array([11, 3, 7, 20, 1, 9])
    means = rng.normal(0, 1, (n_groups, G, C, D)).astype(np.float32)
    actions = (means + rng.normal(0, 0.5, means.shape)).astype(np.float32)
    log_std = rng.normal(0, 0.1, D).astype(np.float32)
    lp0 = O.chunk_log_prob(means.reshape(-1, D), log_std, actions.reshape(-1, D))
    blp = (lp0.reshape(n_groups, G, C) + rng.uniform(-0.3, 0.3, (n_groups, G, C))).astype(np.float32)
    rewards = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
    cfg = grpo.GrpoConfig(group_size=G, kl_coeff=kl)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    loss, dm, dls, st = grpo.grpo_gauss_head_grad(t(means), t(log_std), t(actions), t(blp),
                                                   t(rewards), ids, cfg)
    # oracle: same epilogue entries, coefficients -> head backward
    order, entries = O._entries(ids, rewards, blp, G, cfg.adv_epsilon)
    lp_flat = lp0.reshape(n_groups, G, C)
    res = O._epilogue(lambda key: lp_flat[key[0], key[1]], entries, n_groups * G, cfg.clip_eps,
                      kl)
    cs = np.empty((n_groups, G, C))
    for (k, i), v in res[4].items():
        cs[k, i] = v
    odm, odls = O.gauss_head_backward(means.reshape(-1, D), log_std, actions.reshape(-1, D),
                                      cs.reshape(-1))
    assert loss == pytest.approx(res[0], rel=1e-9, abs=1e-15)
    assert st["group_ids"] == sorted(ids.tolist())
    np.testing.assert_allclose(st["lp_chunk"].cpu().numpy(), lp_flat, rtol=1e-12)
    np.testing.assert_allclose(dm.cpu().numpy().reshape(-1, D), odm, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(dls.cpu().numpy(), odls, rtol=1e-9, atol=1e-14)


def test_gauss_loss_one_call_abort_on_nonfinite_reward(dev):
    import torch
    from paper_2605_13276_b200 import grpo
    rng = np.random.default_rng(5)
    n_groups, G, C, D = 3, 4, 1, 64
    means = rng.normal(0, 1, (n_groups, G, C, D)).astype(np.float32)
    rewards = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
    rewards[1, 2] = np.inf
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    with pytest.raises(grpo.GrpoAbort, match="group 4.*non-finite reward"):
        grpo.grpo_gauss_head_grad(t(means), t(np.zeros(D, np.float32)), t(means),
                                  t(np.zeros((n_groups, G, C), np.float32)), t(rewards),
                                  [9, 4, 6], grpo.GrpoConfig(group_size=G))


def test_grpo_loss_matches_golden_and_finite_differences(dev):
    """grpo.grpo_loss (reference grpo.py:181-214) on the reference's golden
    cases: equals the reference loss (its inter-backend tolerance), and
    central finite differences of it (reference tests/helpers.py:58-79:
    f32-realised steps, h = 1e-3) match grpo_grad's gradient.  The reference
    pins its gradient against an f64-means loss at 1e-4; this loss rounds
    the means to f32 exactly as grpo_grad does, so the secants carry f32
    rounding: 1e-3 norm-wise."""
    from paper_2605_13276_b200 import grpo
    from paper_2605_13276_b200.policy import PolicyParams
    g = golden("grpo_gauss")
    for tag in ("s0_kl0", "s5_kl0", "s3_kl5"):
        if f"{tag}_loss" not in g.files:
            continue
        params, batches = _case(g, tag)
        cfg = grpo.GrpoConfig(group_size=4, clip_eps=0.2, adv_epsilon=1e-8, micro_batch=4,
                              kl_coeff=float(g[f"{tag}_kl"]))
        loss = grpo.grpo_loss(params, batches, cfg)
        assert loss == pytest.approx(float(g[f"{tag}_loss"]), abs=1e-6)
        _, grad, _ = grpo.grpo_grad(params, batches, cfg)
        names = ("w1", "b1", "w2", "b2", "log_std")
        flat = np.concatenate([getattr(params, k).ravel().astype(np.float64) for k in names])
        shapes = [getattr(params, k).shape for k in names]

        def unflat(v):
            out, i = {}, 0
            for k, shp in zip(names, shapes):
                n = int(np.prod(shp))
                out[k] = v[i:i + n].reshape(shp).astype(np.float32)
                i += n
            return PolicyParams(**out)

        fd = np.zeros(flat.size)
        h = 1e-3
        for idx in range(flat.size):
            up, dn = flat.copy(), flat.copy()
            up[idx] += h
            dn[idx] -= h
            pu, pd = unflat(up), unflat(dn)
            delta = float(np.float32(up[idx])) - float(np.float32(dn[idx]))
            fd[idx] = (grpo.grpo_loss(pu, batches, cfg) - grpo.grpo_loss(pd, batches, cfg)) / delta
        err = np.linalg.norm(fd - grad) / np.linalg.norm(grad)
        assert err < 1e-3, (tag, err)


@pytest.mark.parametrize("n_src,n,extra", [(2, 1 << 20, 64), (4, 1_000_003 // 4 * 4, 64),
                                           (3, 0, 64), (8, 4096, 0)])
def test_grad_sum_is_the_node_order_f64_sum(dev, n_src, n, extra):
    """dvla_grad_sum_f32 (the peer reduce-scatter's epilogue): out = f32 of
    the f64 sum in source order (reference reduce_serial, runtime.py:618-627),
    bit-exact; its sum of squares is bit-identical to dvla_grad_sumsq_f32 on
    the output; the side words past n are summed but stay out of the norm."""
    import ctypes as C

    import torch

    from paper_2605_13276_b200 import _lib
    n_all = n + extra
    g = torch.Generator(device=dev).manual_seed(n_src * 7 + n)
    srcs = [torch.randn(n_all, device=dev, generator=g) * (10.0 ** k) for k in range(n_src)]
    out = torch.empty(n_all, device=dev)
    ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(max(n, 1)), dtype=torch.uint8,
                     device=dev)
    ss, ss2 = (torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2))
    bad, bad2 = (torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(2))
    ptrs = (C.c_void_p * n_src)(*[t.data_ptr() for t in srcs])
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.dvla_grad_sum_f32(ptrs, n_src, n, n_all, 4.0, out.data_ptr(), ss.data_ptr(),
                                      bad.data_ptr(), ws.data_ptr(), st), "dvla_grad_sum_f32")
    want = np.zeros(n_all)
    for t in srcs:
        want += t.cpu().numpy().astype(np.float64)
    assert np.array_equal(out.cpu().numpy(), want.astype(np.float32))
    _lib.check(_lib.dvla_grad_sumsq_f32(out.data_ptr(), n, 4.0, ss2.data_ptr(), bad2.data_ptr(),
                                        ws.data_ptr(), st), "dvla_grad_sumsq_f32")
    assert float(ss) == float(ss2)
    ref = float(((want.astype(np.float32)[:n].astype(np.float64) / 4.0) ** 2).sum())
    assert float(ss) == pytest.approx(ref, rel=1e-12)
    assert int(bad) == 0
    if n:
        srcs[-1][n // 2] = float("inf")
        _lib.check(_lib.dvla_grad_sum_f32(ptrs, n_src, n, n_all, 1.0, out.data_ptr(),
                                          ss.data_ptr(), bad.data_ptr(), ws.data_ptr(), st),
                   "dvla_grad_sum_f32")
        assert int(bad) == 1


def _adam_tail_numpy(p, g32, m, v, t, lr, b1, b2, eps, div, f=None):
    """The reference update in numpy f64 (grpo.py:137-150, runtime.py:788
    ÷ nodes, grpo.py:297-301 scaling): every operation correctly rounded."""
    gi = g32.astype(np.float64)
    if div != 1.0:
        gi = gi / div
    if f is not None:
        gi = gi * f
    m2 = b1 * m + (1.0 - b1) * gi
    v2 = b2 * v + (1.0 - b2) * (gi * gi)
    mh = m2 / (1.0 - b1 ** t)
    vh = v2 / (1.0 - b2 ** t)
    p2 = (p.astype(np.float64) - (lr * mh) / (np.sqrt(vh) + eps)).astype(np.float32)
    return p2, m2, v2


@pytest.mark.parametrize("t,div", [(1, 1.0), (2, 3.0), (5, 4.0), (37, 7.0), (1000, 1.0),
                                   (30000, 3.0)])
def test_adam_tail_is_bitwise_on_wide_inputs(dev, t, div):
    """dvla_adam_tail_f32 (the learner's optimizer tail) against the
    reference arithmetic in numpy, bit for bit, on 4M elements spanning the
    f64 range the moments reach (zeros, -0, subnormal moments, 1e-300 ..
    1e+30) for several steps and node counts."""
    import torch

    from paper_2605_13276_b200 import _lib
    rng = np.random.default_rng(t * 10 + int(div))
    n = 1 << 22
    p = (rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 2, n)).astype(np.float32)
    g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-30, 3, n)).astype(np.float32)
    m = rng.standard_normal(n) * 10.0 ** rng.uniform(-300, 30, n)
    v = np.abs(rng.standard_normal(n)) * 10.0 ** rng.uniform(-300, 30, n)
    m[:64], v[:64] = 0.0, 0.0
    m[64:128] = -0.0
    m[128:192], v[128:192] = 1e-310, 3e-315           # subnormal f64
    g[192:256] = 0.0
    m[256:320] = np.nextafter(2.0, 0.0)               # all-ones significands
    v[256:320] = np.nextafter(1.0, 0.0)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    want_p, want_m, want_v = _adam_tail_numpy(p, g, m, v, t, lr, b1, b2, eps, div)
    tp, tg = torch.from_numpy(p).to(dev), torch.from_numpy(g).to(dev)
    tm, tv = torch.from_numpy(m).to(dev), torch.from_numpy(v).to(dev)
    w16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.dvla_adam_tail_f32(tp.data_ptr(), tg.data_ptr(), tm.data_ptr(),
                                       tv.data_ptr(), n, t, lr, b1, b2, eps, div, None, 0.0,
                                       None, w16.data_ptr(), bad.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream),
               "dvla_adam_tail_f32")
    got_m, got_v, got_p = tm.cpu().numpy(), tv.cpu().numpy(), tp.cpu().numpy()
    assert np.array_equal(got_m.view(np.int64), want_m.view(np.int64))
    assert np.array_equal(got_v.view(np.int64), want_v.view(np.int64))
    assert np.array_equal(got_p.view(np.int32), want_p.view(np.int32))
    assert torch.equal(w16.cpu(), torch.from_numpy(want_p).bfloat16())
