"""Host-side runtime logic on the CPU: the staleness gate (VersionBoard) and
the NCCL gradient reducer's semantics on a world_size-2 gloo group."""

import os
import threading

import numpy as np
import pytest

from paper_2605_13276_b200.core import ParamSnapshot
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
