"""Weight plane over NVLINK-mode transports and the four-lane swimlane on a
single B200 (multi-GPU paths: tests/test_multigpu.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nvlink_broadcast_into_subscriber_regions(dev):
    import torch
    from paper_2605_13276_b200.core import snapshot_from_params
    from paper_2605_13276_b200.planes import ControlPlane, Plane, Transport, TransportMode
    from paper_2605_13276_b200.replicate import bytes_equal
    n = 3_000_000  # f32 params -> 12 MB regions
    t = Transport(TransportMode.NVLINK, Plane.CONTROL)
    plane = ControlPlane(t, chunk_bytes=1 << 20, ctas_per_hop=8)
    boxes = [plane.subscribe(f"r{i}", device=dev, nbytes=4 * n) for i in range(3)]
    for v in (1, 2, 3):
        p = torch.randn(n, device=dev) * v
        snap = snapshot_from_params(p, v)
        plane.broadcast(snap)
        torch.cuda.synchronize()
        plane.check()
        for b in boxes:
            got = b.take_newest()
            assert got.version == v and got.ready is not None and got.ready.query()
            assert got.params.data_ptr() == b.region(v).data_ptr()  # zero-copy view
            assert bytes_equal(got.params, p) == (0, -1)
    assert t.copy_counter == 9 and t.bytes_counter == 9 * 4 * n


def test_swimlane_runs_and_publishes_versions(dev):
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    cfg = SwimlaneConfig(n_groups=4, group_size=4, tokens=8, vocab=2048, action_bins=256,
                         hidden=128, epochs=5, seed=3)
    res = run_swimlane(cfg, device=dev)
    s = res.summary()
    assert res.counters["updates"] == 5
    assert s["staleness_max"] <= cfg.staleness_limit
    assert s["transitions_per_s"] > 0 and s["trajectories_per_s"] > 0
    assert all(np.isfinite(u["loss"]) for u in res.update_stats)
    assert [u["version"] for u in res.update_stats] == [1, 2, 3, 4, 5]


def test_swimlane_quarantines_poisoned_epoch(dev):
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    cfg = SwimlaneConfig(n_groups=4, group_size=4, tokens=8, vocab=2048, action_bins=256,
                         hidden=128, epochs=4, seed=5)
    res = run_swimlane(cfg, device=dev, poison_epochs={2})
    assert res.counters.get("quarantined_updates", 0) == 1
    assert res.counters["updates"] == 3


def test_nvlink_data_channel_moves_batches_to_the_consumer_gpu(dev):
    """Data-plane NVLINK channel: a GroupBatch put on the
    rollout GPU arrives on the learner GPU, bit-identical, with the bytes
    counted; on a 1-GPU box the batch stays (same device, zero copy)."""
    import numpy as np
    import torch
    from paper_2605_13276_b200.grpo import GroupBatch
    from paper_2605_13276_b200.planes import Channel, Plane, Transport, TransportMode
    src_dev = torch.device("cuda", 0)
    dst_dev = torch.device("cuda", 1 if torch.cuda.device_count() > 1 else 0)
    tr = Transport(TransportMode.NVLINK, Plane.DATA)
    ch = Channel(4, tr, name="traj", device=dst_dev)
    sent = []
    for gid in range(3):
        b = GroupBatch(group_id=gid, horizon=8, chunk=1,
                       obs=torch.randn(8, 1, 16, device=src_dev),
                       actions=torch.randn(8, 1, 7, device=src_dev),
                       behavior_log_prob=torch.randn(8, 1, device=src_dev),
                       rewards=torch.randint(0, 2, (8,), device=src_dev).float(),
                       behavior_version=gid,
                       tokens=torch.randint(0, 256, (8, 1, 56), device=src_dev, dtype=torch.int32))
        sent.append(b)
        ch.put(b)
    for b in sent:
        got = ch.take()
        assert got.group_id == b.group_id and got.behavior_version == b.behavior_version
        for f in ("obs", "actions", "behavior_log_prob", "rewards", "tokens"):
            t = getattr(got, f)
            assert t.device == dst_dev
            assert torch.equal(t.cpu(), getattr(b, f).cpu())
    per = sum(getattr(sent[0], f).numel() * getattr(sent[0], f).element_size()
              for f in ("obs", "actions", "behavior_log_prob", "rewards", "tokens"))
    assert tr.bytes_counter == (3 * per if dst_dev != src_dev else 0)
    assert np.isfinite(per)


def test_nccl_c_abi_single_process_allreduce(dev):
    """dvla_nccl_*: one process, every visible GPU, in-place sum all-reduce
    (f32 and f64) through the C-ABI (libnccl opened at run time)."""
    import ctypes as C
    import torch
    from paper_2605_13276_b200 import _lib
    n = torch.cuda.device_count()
    devs = (C.c_int * n)(*range(n))
    _lib.check(_lib.dvla_nccl_init(n, devs), "dvla_nccl_init")
    try:
        for dt, code in ((torch.float32, _lib.F32), (torch.float64, _lib.F64)):
            bufs = [torch.arange(1000, dtype=dt, device=f"cuda:{d}") * (d + 1) for d in range(n)]
            _lib.check(_lib.dvla_nccl_group_start(), "group_start")
            for d, b in enumerate(bufs):
                with torch.cuda.device(d):
                    _lib.check(_lib.dvla_nccl_allreduce_sum(
                        d, b.data_ptr(), b.numel(), code, torch.cuda.current_stream(d).cuda_stream),
                        "dvla_nccl_allreduce_sum")
            _lib.check(_lib.dvla_nccl_group_end(), "group_end")
            want = torch.arange(1000, dtype=dt) * (n * (n + 1) / 2)
            for d, b in enumerate(bufs):
                torch.cuda.synchronize(d)
                assert torch.equal(b.cpu(), want), (dt, d)
    finally:
        _lib.dvla_nccl_destroy()


def test_sampler_and_trainer_workers_against_the_oracle(dev):
    """SamplerWorker.run_epoch -> TrainerWorker.update (reference
    runtime.py:676-800): the update's loss equals the f64 oracle on the same
    logits; the head gradient is the f32 GEMM output dW = dl^T x (checked
    against an f64 product of the same operands at 1e-5, and its norm at
    1e-5); Adam's first step moves every parameter with a clear gradient by
    -lr * sign(grad) (m_hat / sqrt(v_hat) = sign(g) at step 1); the bf16
    working copy is the round-to-nearest of the new master weights."""
    import torch
    from oracle import grpo_oracle as O
    from paper_2605_13276_b200.grpo import GrpoAbort
    from paper_2605_13276_b200.pools import Pool, PoolKind
    from paper_2605_13276_b200.runtime import (GradReducer, SamplerWorker, SwimlaneConfig,
                                               TrainerWorker, token_positions)
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                         hidden=64, seed=11, lr=1e-3)
    V, H, G, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.tokens
    n_traj = cfg.n_groups * G
    model_pool = Pool(PoolKind.MODEL_COMPUTE, 64 << 20, device=dev)
    env_pools = [Pool(PoolKind.ENV_AUX, 32 << 20, device=dev) for _ in range(2)]
    s_sample, s_train = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    trainer = TrainerWorker(cfg, 0, model_pool, GradReducer(1, None), s_train, dev)
    sampler = SamplerWorker(cfg, 0, 1, env_pools, s_sample, dev)
    snap = trainer.snapshot()
    torch.cuda.synchronize()
    assert snap.version == 0
    assert torch.equal(snap.params.view(torch.int16),
                       trainer.policy.weight_bf16().reshape(-1).view(torch.int16))

    msgs, meta = sampler.run_epoch(0, snap)
    assert [m.group_id for m in msgs] == [0, 1]
    assert meta["behavior_version"] == 0 and meta["roll_wall"] > 0
    toks = torch.cat([m.actions.reshape(-1) for m in msgs])
    assert int(toks.min()) >= 0 and int(toks.max()) < V   # sampled over the full vocabulary
    feats = torch.cat([m.obs for m in msgs]).reshape(n_traj, H).clone()
    blp = torch.cat([m.behavior_log_prob.reshape(-1) for m in msgs]).clone()
    rw = torch.cat([m.rewards for m in msgs]).clone()
    W = trainer.policy.weight_bf16().clone()
    pos = token_positions(cfg, dev)
    ftok = (feats.view(n_traj, 1, H) + pos.view(1, T, H)).reshape(-1, H)   # bf16, as update()
    logits = ftok @ W.t()
    before = trainer.policy.master.clone()

    st = trainer.update(msgs)
    torch.cuda.synchronize()
    assert st["version"] == 1 and trainer.version == 1
    assert torch.equal(trainer.feats_tok, ftok) and torch.equal(trainer.logits, logits)
    x = logits.float().cpu().numpy().reshape(cfg.n_groups, G, 1, T, V)
    loss, dl, ost = O.grpo_token_grad(
        x, toks.cpu().numpy().reshape(cfg.n_groups, G, 1, T),
        blp.cpu().numpy().reshape(cfg.n_groups, G, 1), rw.cpu().numpy().reshape(cfg.n_groups, G),
        np.array([0, 1]))
    # on-policy batch (ratio ~ 1, zero-mean advantages): the loss is a
    # cancellation near 0, so compare it absolutely and the lp / ratio tightly
    np.testing.assert_allclose(st["loss"], loss, atol=1e-6)
    np.testing.assert_allclose(trainer.loss.lp_chunk.cpu().numpy().reshape(-1),
                               ost["lp_chunk"].reshape(-1), rtol=1e-9, atol=1e-5)
    np.testing.assert_allclose(st["mean_ratio"], ost["mean_ratio"], rtol=1e-6)
    assert st["n_chunks"] == n_traj
    # head gradient: f32 GEMM output of the bf16 operands (dl, features)
    assert trainer.grad2d.dtype == torch.float32
    g64 = trainer.dl.double().t() @ trainer.feats_tok.double()
    got = trainer.grad2d.double()
    assert float((got - g64).norm() / g64.norm()) <= 1e-5
    g = g64.reshape(-1).cpu().numpy()
    np.testing.assert_allclose(st["grad_norm"], np.sqrt((g * g).sum()), rtol=1e-5)
    # the bf16 d loss / d logits against the oracle's f64 gradient (bf16 tolerance)
    from oracle.check import assert_dlogits_close
    assert_dlogits_close(trainer.dl.float().cpu().numpy(), dl.reshape(-1, V), 1e-2)
    delta = (trainer.policy.master - before).cpu().double().numpy()
    clear = np.abs(g) > max(1e-2 * np.abs(g).max(), 1e-4)  # eps = 1e-8 negligible
    assert clear.sum() > 100
    np.testing.assert_allclose(delta[clear], -cfg.lr * np.sign(g[clear]), rtol=1e-3)
    assert torch.equal(trainer.policy.weight_bf16(),
                       trainer.policy.master.view(V, H).to(torch.bfloat16))

    # a poisoned batch: GrpoAbort, and the device skipped the step
    m0, v0 = trainer.policy.m.clone(), trainer.policy.v.clone()
    p0 = trainer.policy.master.clone()
    msgs2, _ = sampler.run_epoch(1, trainer.snapshot(), poison=True)
    with pytest.raises(GrpoAbort):
        trainer.update(msgs2)
    assert trainer.version == 1 and trainer.policy.step == 1
    assert torch.equal(trainer.policy.master, p0) and torch.equal(trainer.policy.m, m0) \
        and torch.equal(trainer.policy.v, v0)


def test_torch_arena_places_torch_allocations_in_env_aux(dev):
    """pools.TorchArena: tensors torch allocates inside
    `with arena:` live in the ENV_AUX pool's slab, placed by its first-fit
    arena; the bound pool refuses epoch_reset; the swimlane's temporaries go
    there (counters)."""
    import torch
    from paper_2605_13276_b200.pools import Pool, PoolKind, PoolUsageError, TorchArena
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    arena = TorchArena.shared(dev, 256 << 20)
    before = arena.pool.stats().alloc_count
    with arena:
        a = torch.randn(1 << 20, device=dev)
        b = torch.cat([a, a]) * 2
    c = torch.randn(1 << 20, device=dev)          # outside: torch's own segments
    assert arena.holds(a) and arena.holds(b) and not arena.holds(c)
    assert arena.pool.stats().alloc_count > before
    assert torch.equal(b[: 1 << 20], a * 2)
    with pytest.raises(PoolUsageError):
        arena.pool.epoch_reset()
    # another pool cannot take over the device's binding
    with pytest.raises(Exception):
        TorchArena(Pool(PoolKind.ENV_AUX, 1 << 20, device=dev))
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                         hidden=64, epochs=3, seed=21)
    res = run_swimlane(cfg, device=dev)
    assert res.counters["updates"] == 3
    assert res.counters["torch_arena"]["segments_allocated"] > 0


def test_torch_arena_close_returns_segments_and_unbinds(dev):
    """TorchArena.close(): torch's segments go back to the arena (live bytes
    0), the device is unbound and the pool may be epoch-reset again.  Runs
    in a fresh process (the device's binding is process-wide)."""
    import subprocess
    import sys
    code = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_2605_13276_b200.pools import Pool, PoolKind, TorchArena, PoolUsageError
dev = torch.device("cuda", 0)
arena = TorchArena(Pool(PoolKind.ENV_AUX, 64 << 20, device=dev))
with arena:
    x = torch.ones(1 << 18, device=dev)
assert arena.holds(x) and arena.pool.stats().live_bytes > 0
try:
    arena.pool.epoch_reset()
    raise SystemExit("epoch_reset allowed while bound")
except PoolUsageError:
    pass
del x
arena.close()
assert arena.pool.stats().live_bytes == 0, arena.pool.stats()
arena.pool.epoch_reset()
again = TorchArena(Pool(PoolKind.ENV_AUX, 16 << 20, device=dev))   # the device is free again
print("CLOSE_OK")
""" % (__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))),)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "CLOSE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[:3000]


def test_nvlink_broadcast_across_devices_one_process(dev):
    """ControlPlane NVLINK transport with subscribers on two GPUs of one
    process: hops on the second device run on the plane's own stream with
    their own timeout word; each mailbox's snapshot carries the event of the
    hop that wrote it."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs in one process")
    from paper_2605_13276_b200.core import snapshot_from_params
    from paper_2605_13276_b200.planes import ControlPlane, Plane, Transport, TransportMode
    from paper_2605_13276_b200.replicate import bytes_equal
    n = 2_000_000
    plane = ControlPlane(Transport(TransportMode.NVLINK, Plane.CONTROL), chunk_bytes=1 << 20,
                         ctas_per_hop=8)
    boxes = [plane.subscribe("a", device="cuda:0", nbytes=4 * n),
             plane.subscribe("b", device="cuda:1", nbytes=4 * n),
             plane.subscribe("c", device="cuda:1", nbytes=4 * n)]
    s = torch.cuda.Stream(device="cuda:0")
    for v in (1, 2, 3):
        p = torch.randn(n, device="cuda:0") + v
        plane.broadcast(snapshot_from_params(p, v), stream=s)
        for b in boxes:
            got = b.take_newest()
            got.ready.synchronize()
            assert got.version == v
            ref = p.to(got.params.device)
            assert bytes_equal(got.params, ref) == (0, -1), (b.name, v)
    plane.check()
