"""Host-side runtime logic on the CPU: the staleness gate (VersionBoard) and
the NCCL gradient reducer's semantics on a world_size-2 gloo group."""

import os
import threading

import numpy as np
import pytest

from paper_2605_13276_b200.core import ConfigError, ParamSnapshot
from paper_2605_13276_b200.runtime import GradReducer, Monitor, VersionBoard


def _board(limit=1):
    return VersionBoard(limit, Monitor(threading.Event()),
                        ParamSnapshot(version=0, params=np.zeros(4, np.float32)))


def test_gate_admits_up_to_the_staleness_limit():
    b = _board(limit=1)
    snap, stal = b.wait_gate()           # epoch 0 on v0
    assert stal == 0 and snap.version == 0
    b.produce(0, {})
    b.boundary()
    snap, stal = b.wait_gate()           # frontier 0 + 1 - 0 - 0 = 1 <= 1
    b.produce(1, {})
    b.boundary()
    # frontier 2 > limit: would block until the trainer publishes + we install
    t = threading.Thread(target=b.wait_gate)
    t.start()
    t.join(0.2)
    assert t.is_alive()
    b.publish()                          # v1, processed 1 -> frontier 1+2-1-0 = 2
    b.deposit(ParamSnapshot(version=1, params=np.ones(4, np.float32)))
    t.join(2.0)
    assert not t.is_alive() and b.installed == 1


def test_stale_deposits_are_ignored():
    b = _board()
    b.deposit(ParamSnapshot(version=2, params=np.zeros(4, np.float32)))
    b.wait_gate()
    assert b.installed == 2
    b.deposit(ParamSnapshot(version=1, params=np.zeros(4, np.float32)))
    assert b.regressions_ignored == 1


def test_pacing_blocks_mid_epoch_until_install():
    b = _board(limit=1)
    b.wait_gate()                        # sampler now mid-epoch on v0
    b.publish()                          # v1 may be published (installed 0 >= 1-1)
    done = threading.Event()

    def trainer():
        b.wait_pacing(2)                 # v2 needs installed >= 1 or a boundary
        done.set()

    t = threading.Thread(target=trainer)
    t.start()
    assert not done.wait(0.2)
    b.boundary()
    assert done.wait(2.0)


def _reduce_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.tensor([1.0 + rank, 1e-9 * (rank + 1), -3.0], dtype=torch.float64)
    out_fast = GradReducer(world).reduce(g.clone())
    out_exact = GradReducer(world, exact=True).reduce(g.clone())
    # ZeRO-1 transport choice: collective, peer memory when every rank is on
    # this host, NCCL when asked
    peer = (GradReducer(world).peer_scatter(), GradReducer(world, scatter="nccl").peer_scatter(),
            GradReducer(world, scatter="peer").peer_scatter())
    assert peer == (True, False, True), peer
    q.put((rank, out_fast.numpy().tolist(), out_exact.numpy().tolist()))
    dist.destroy_process_group()


def test_grad_reducer_mean_over_ranks_gloo():
    """Reference semantics (runtime.py:588-627): every node's gradient is
    quantised to f32, summed and divided by `nodes`; all ranks agree."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=60) for _ in range(2))
    for p in procs:
        p.join(30)
    f32 = np.float32
    want = [(float(f32(1.0)) + float(f32(2.0))) / 2,
            (float(f32(1e-9)) + float(f32(2e-9))) / 2, -3.0]
    for _, fast, exact in res:
        np.testing.assert_allclose(exact, want, rtol=1e-15)
        np.testing.assert_allclose(fast, want, rtol=1e-7)
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]


def test_single_node_reduce_is_identity():
    import torch
    g = torch.arange(4, dtype=torch.float64)
    assert GradReducer(1).reduce(g) is g


def test_barrier_free_handoff_audit():
    from paper_2605_13276_b200.runtime import RunResult, barrier_free_handoff_audit
    r = RunResult()
    r.wall = 2.0
    r.lane_busy = {"sampler": 1.5, "trainer": 2.5}
    r.reports = [{}, {}]
    b = barrier_free_handoff_audit(r)
    assert b.sampler_idle_fraction == 0.25 and b.trainer_idle_fraction == 0.0
    assert b.wall == 2.0 and not b.warmup_dominated
    r.reports = [{}]
    assert barrier_free_handoff_audit(r).warmup_dominated


def _token_case(seed, n_groups, G, T, V, H):
    rng = np.random.default_rng(seed)
    feats = rng.normal(0, 1, (n_groups * G * T, H))
    W = rng.normal(0, 0.3, (V, H))
    x = (feats @ W.T).astype(np.float32).reshape(n_groups, G, 1, T, V)
    tokens = rng.integers(0, V, (n_groups, G, 1, T)).astype(np.int32)
    from oracle import grpo_oracle as O
    _, _, st0 = O.grpo_token_grad(x, tokens, np.zeros((n_groups, G, 1), np.float32),
                                  np.ones((n_groups, G), np.float32), np.arange(n_groups),
                                  want_dlogits=False)
    blp = (st0["lp_chunk"] + rng.uniform(-0.3, 0.3, (n_groups, G, 1))).astype(np.float32)
    rewards = rng.uniform(0, 1, (n_groups, G)).astype(np.float32)
    return feats, W, x, tokens, blp, rewards


def _shard_grad(feats, x, tokens, blp, rewards, ids, poison=False):
    """One learner rank's gradient of the head: the token loss on its group
    shard (w = 1 / (n_traj_local * C)), dW = dl^T feats, as an f32 frame."""
    from oracle import grpo_oracle as O
    if poison:
        rewards = rewards.copy()
        rewards[0, 0] = np.nan
        try:
            O.grpo_token_grad(x, tokens, blp, rewards, ids)
        except O.OracleAbort:
            return None
    _, dl, _ = O.grpo_token_grad(x, tokens, blp, rewards, ids)
    V = x.shape[-1]
    return (dl.reshape(-1, V).T @ feats).reshape(-1)


def _update_worker(rank, world, port, q, poison_rank):
    """runtime.TrainerWorker.update's arithmetic with a CPU restatement of
    its device pieces: shard -> f32 gradient buffer + skip word -> bucketed
    GradReducer.reduce_async (gloo) -> / nodes -> clip -> Adam, skipped on
    every rank when any rank's batch aborted."""
    import torch
    import torch.distributed as dist
    from oracle import grpo_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_groups, G, T, V, H = 4, 4, 3, 16, 5
    feats, W, x, tokens, blp, rewards = _token_case(7, n_groups, G, T, V, H)
    k = n_groups // world
    sl = slice(rank * k, (rank + 1) * k)
    rows = slice(rank * k * G * T, (rank + 1) * k * G * T)
    g = _shard_grad(feats[rows], x[sl], tokens[sl], blp[sl], rewards[sl],
                    np.arange(n_groups)[sl], poison=(rank == poison_rank))
    n = V * H
    buf = torch.zeros(n + 1, dtype=torch.float32)
    if g is None:
        buf[n] = 1.0                     # dvla_loss_status: this rank aborted
    else:
        buf[:n] = torch.from_numpy(g.astype(np.float32))
    red = GradReducer(world)
    assert red.overlappable(buf)
    step = -(-V // 3)
    works = []
    for j in range(3):
        a, b = j * step, min(V, (j + 1) * step)
        works.append(red.reduce_async(buf[a * H:(b * H if b < V else n + 1)]))
    for w in works:
        w.wait()
    skipped = float(buf[n]) != 0.0
    params = W.reshape(-1).astype(np.float32)
    m = np.zeros(n)
    v = np.zeros(n)
    norm = None
    if not skipped:
        gm = buf[:n].double().numpy() / world
        norm, gm = O.clip_grad_norm(gm, 0.05)
        params, m, v, _ = O.adam_step(params, gm, m, v, 0, 1e-3, 0.9, 0.999, 1e-8)
    q.put((rank, skipped, norm, params.tobytes()))
    dist.destroy_process_group()


def _run_update_workers(poison_rank):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_update_worker, args=(r, 2, port, q, poison_rank))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(30)
    return res


def test_sharded_update_arithmetic_gloo():
    """World size 2 (reference runtime.py:775-796): each rank's shard
    gradient, reduced in f32 buckets, divided by the node count, clipped and
    stepped, equals the single-process arithmetic on the same shards, and
    both ranks hold bitwise-identical parameters afterwards."""
    from oracle import grpo_oracle as O
    res = _run_update_workers(poison_rank=-1)
    (_, sk0, n0, p0), (_, sk1, n1, p1) = res
    assert not sk0 and not sk1 and p0 == p1 and n0 == n1
    n_groups, G, T, V, H = 4, 4, 3, 16, 5
    feats, W, x, tokens, blp, rewards = _token_case(7, n_groups, G, T, V, H)
    gs = [_shard_grad(feats[r * 2 * G * T:(r + 1) * 2 * G * T], x[2 * r:2 * r + 2],
                      tokens[2 * r:2 * r + 2], blp[2 * r:2 * r + 2], rewards[2 * r:2 * r + 2],
                      np.arange(2 * r, 2 * r + 2)) for r in range(2)]
    # the reference's mean of f32 frames (runtime.py:590-627), f64 sum
    gm = (gs[0].astype(np.float32).astype(np.float64) +
          gs[1].astype(np.float32).astype(np.float64)) / 2
    norm, gm = O.clip_grad_norm(gm, 0.05)
    want, _, _, _ = O.adam_step(W.reshape(-1).astype(np.float32), gm, np.zeros(V * H),
                                np.zeros(V * H), 0, 1e-3, 0.9, 0.999, 1e-8)
    got = np.frombuffer(p0, dtype=np.float32)
    np.testing.assert_allclose(n0, norm, rtol=1e-6)
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
    # the mean of the equal-size shards' gradients is the full batch's
    _, dl, _ = O.grpo_token_grad(x, tokens, blp, rewards, np.arange(n_groups))
    full = (dl.reshape(-1, V).T @ feats).reshape(-1)
    np.testing.assert_allclose((gs[0] + gs[1]) / 2, full, rtol=1e-9, atol=1e-12)


def test_one_rank_abort_skips_the_update_on_every_rank_gloo():
    res = _run_update_workers(poison_rank=1)
    (_, sk0, _, p0), (_, sk1, _, p1) = res
    assert sk0 and sk1 and p0 == p1


def test_disagg_key_board_polls_without_blocking_other_lanes():
    """disagg._Keys: waits poll the store with the non-blocking check(), so
    a lane waiting on a key never holds the store client against another
    lane's set (the deadlock a blocking get caused); timeouts and a peer
    lane's error surface instead of hanging."""
    import threading
    import time as _t

    import torch.distributed as dist
    from paper_2605_13276_b200.disagg import _Keys
    store = dist.HashStore()
    errors = []
    kb = _Keys(store, "ns/", 2.0, errors)
    got = {}

    def waiter():
        got["v"] = kb.get(kb.key("pub", 3), "v3")

    th = threading.Thread(target=waiter)
    th.start()
    _t.sleep(0.05)
    kb.set(kb.key("rel", 2, 0), "1")          # another lane's set goes through
    kb.set(kb.key("pub", 3), "end")
    th.join(2.0)
    assert got["v"] == b"end"
    kb.wait([kb.key("rel", 2, 0)])
    t0 = _t.perf_counter()
    with pytest.raises(TimeoutError):
        _Keys(store, "ns/", 0.2, errors).wait([kb.key("never")], "never")
    assert _t.perf_counter() - t0 < 1.0
    errors.append(RuntimeError("peer lane failed"))
    with pytest.raises(RuntimeError, match="peer lane failed"):
        kb.wait([kb.key("never")])


def test_grad_reducer_reference_signatures():
    """GradReducer keeps the reference's call forms: reduce(node, round,
    grad, clock) (a no-op on one node) and reduce_serial(round, grads) with
    the reference arithmetic (f32 frames, f64 sum in node order, / nodes)."""
    import torch
    g = np.array([1.0 / 3, 2.0, -1e-9])
    r = GradReducer(1)
    assert r.reduce(0, 5, g, None) is g and r.reduce(g) is g
    r3 = GradReducer(3)
    gs = [g * (k + 1) for k in range(3)]
    want = sum(x.astype(np.float32).astype(np.float64) for x in gs) / 3
    np.testing.assert_array_equal(r3.reduce_serial(0, gs), want)
    got_t = r3.reduce_serial(0, [torch.from_numpy(x) for x in gs])
    np.testing.assert_array_equal(got_t.numpy(), want)
    with pytest.raises(TypeError):
        r.reduce(1, 2)
    with pytest.raises(ConfigError, match="reduce-scatter transport"):
        GradReducer(2, scatter="ring")
    assert not GradReducer(1).peer_scatter()


def test_retire_waits_for_a_newer_install_and_blocks_stale_deposits():
    """VersionBoard.retire (the published-weight ring, run_swimlane): the
    publisher may reuse version u's slot only once the sampler installed
    something newer; u (and anything older) is dropped from the pending
    deliveries and later deposits of it are ignored."""
    b = _board(limit=1)
    b.wait_gate()                                    # sampler installed v0 (mid-epoch)
    done = threading.Event()

    def publisher():
        b.retire(0)                                  # slot of v0 about to be reused
        done.set()

    t = threading.Thread(target=publisher)
    t.start()
    assert not done.wait(0.2)                        # v0 is installed: must wait
    b.publish()
    b.deposit(ParamSnapshot(version=1, params=np.ones(4, np.float32)))
    b.produce(0, {})
    b.boundary()
    b.wait_gate()                                    # installs v1
    assert done.wait(2.0) and b.installed == 1
    b.deposit(ParamSnapshot(version=0, params=np.zeros(4, np.float32)))
    assert b.regressions_ignored == 1
    # pending deliveries at or below the retired version are dropped
    b2 = _board(limit=2)
    b2.deposit(ParamSnapshot(version=1, params=np.zeros(4, np.float32)))
    b2.deposit(ParamSnapshot(version=2, params=np.zeros(4, np.float32)))
    b2.installed = 3                                 # (as if v3 were installed)
    b2.retire(2)
    assert 1 not in b2.delivered and 2 not in b2.delivered and b2.retired_max == 2
    # a finished sampler never blocks the publisher
    b3 = _board(limit=1)
    b3.mark_sampler_done()
    b3.retire(0)


def test_zero1_gemm_plans_cover_every_block_once_own_last():
    """TrainerWorker._grad_segments: the GEMM row ranges tile [0, N Vs)
    exactly once; every peer block is pushed exactly once, after the GEMM
    that completes it; the last GEMM computes only own rows (it hides the
    earlier pushes), for every plan and N = 2..8."""
    from types import SimpleNamespace

    from paper_2605_13276_b200.runtime import TrainerWorker
    Vs = 1000
    for plan in ("halves", "halves1", "runs"):
        for N in range(2, 9):
            for r in range(N):
                me = SimpleNamespace(reducer=SimpleNamespace(nodes=N), reducer_rank=r,
                                     grad_plan=plan, policy=SimpleNamespace(Vs=Vs))
                segs = TrainerWorker._grad_segments(me)
                rows = sorted((a, b) for a, b, _ in segs)
                assert rows[0][0] == 0 and rows[-1][1] == N * Vs, (plan, N, r, segs)
                assert all(x[1] == y[0] for x, y in zip(rows, rows[1:])), (plan, N, r, segs)
                pushed, done_rows = [], set()
                for a, b, blocks in segs:
                    done_rows.update(range(a // 10, b // 10))   # 10-row granules
                    for j in blocks:
                        assert j != r
                        assert set(range(j * Vs // 10, (j + 1) * Vs // 10)) <= done_rows
                        pushed.append(j)
                assert sorted(pushed) == [j for j in range(N) if j != r], (plan, N, r, segs)
                a, b, blocks = segs[-1]
                assert a < (r + 1) * Vs and b > r * Vs, (plan, N, r, segs)   # own rows last
                h = N // 2
                split = plan == "halves" and N > 2 and r in (0, h - 1, h, N - 1) and (
                    (N - h if r >= h else h) > 1)
                if plan == "runs" or N == 2 or split:
                    # the last GEMM is own rows only: every push is hidden
                    assert r * Vs <= a and b <= (r + 1) * Vs and not blocks, (plan, N, r, segs)
                if plan != "runs" and N > 2:
                    assert len(segs) in (2, 3)
