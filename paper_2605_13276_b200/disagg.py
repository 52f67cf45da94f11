"""Disaggregated swimlane (BASELINE config 3 layout): learner GPUs and
rollout GPUs, weights replicated over NVLink every iteration.

Reference: the disaggregated placement plans (placement.py:119-177) put the
learner and the rollout workers on different slot groups; the asynchronous
runtime's lanes (runtime.py:1157-1318) then move trajectories to the
trainer over the data plane and each published snapshot to every rollout
worker over the control plane (dist_lane -> ControlPlane.broadcast,
runtime.py:1259-1276; recv_lane -> WeightMailbox -> VersionBoard deposit /
install at the epoch boundary, runtime.py:1195-1214).  B200 layout, one
process per GPU:

  * learner ranks (default {0, 1} from 4 GPUs, {0} below): trainer lane +
    weight-distribution lane.  TrainerWorker.update on the groups of the
    rollout ranks assigned to it (group-sharded; NCCL reduce-scatter /
    all-gather over the learner group, ZeRO-1), then the new bf16 weights
    are snapshotted on the trainer stream and the distribution stream
    pushes them through a SplitReplicator: learner i sources part i of the
    region along its own chain through every rollout rank (TMA-staged peer
    stores, csrc/replicate.cu), straight into the receivers' replica ring
    in their MODEL_COMPUTE pools.  The next update overlaps the push.
  * rollout ranks: sampler lane + weight-receive lane.  The sampler runs
    epochs on the installed replica in place (zero copy) and ships each
    epoch's trajectories to its learner through a PeerChannel (NVLink peer
    copies into the learner's slot ring, device flags); the receive lane
    runs this rank's hop of every version's chain on its own stream and
    deposits the replica view; the sampler installs the newest deposit at
    its epoch boundary.

Host coordination uses the job's c10d store (small keys; no payload):
  pub/{v}     learner 0: version v's chain heads are launched (or "end")
  proc/{e}    learner 0: epoch e processed; value = version after it
  rel/{r}/{u} rollout rank r no longer reads version u (ring slot reusable)
  sum/{v}     learner 0: checksum of version v's bytes (verify=True)
Staleness gate (the reference's two-ended gate restated for disjoint
processes): epoch e starts on a version >= the one published after epoch
e - limit - 1 was processed.  The replica ring has limit + 2 slots; the
learner pushes version v only once every rollout rank released v - ring
(a rank releases everything older than what it installs at a boundary),
so a slot is never overwritten while a sampler reads it.
"""

from __future__ import annotations

import logging
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .core import ConfigError, ParamSnapshot
from .grpo import GroupBatch, GrpoAbort

log = logging.getLogger("dvla_b200.disagg")


_CALLS = [0]


def default_learners(world: int) -> list:
    """Learner ranks: two learners (the C3 layout) when the rest split
    evenly between them, else one."""
    if world >= 4 and (world - 2) % 2 == 0:
        return [0, 1]
    return [0]


@dataclass
class DisaggResult:
    role: str
    rank: int
    updates: int = 0
    quarantined: int = 0
    epochs: int = 0
    wall: float = 0.0
    trajectories_per_s: float = 0.0
    replication: list = field(default_factory=list)     # learner 0: per-version dicts
    checksum_mismatches: int = 0
    versions_received: int = 0
    installed: list = field(default_factory=list)      # rollout: version per epoch
    update_stats: list = field(default_factory=list)
    overlap: dict = field(default_factory=dict)
    policy: object = None
    replica_of: object = None      # rollout: fn(version) -> replica view (tests)
    lane_s: dict = field(default_factory=dict)   # host seconds per lane phase
    recv_ms: list = field(default_factory=list)  # rollout: per-version hop time (CUDA events)
    recv_ms_median_max: float | None = None      # max over rollout ranks of their medians
    timeline: list = field(default_factory=list)  # (event, epoch/version, host monotonic s)
    mismatched: list = field(default_factory=list)  # rollout: (version, got, want) checksums

    def summary(self) -> dict:
        reps = [r["ms"] for r in self.replication]
        gbs = [r["gbs"] for r in self.replication]
        return {"role": self.role, "updates": self.updates, "quarantined": self.quarantined,
                "trajectories_per_s": self.trajectories_per_s, "wall": self.wall,
                "replication_ms_median": float(np.median(reps)) if reps else None,
                "replication_gbs_median": float(np.median(gbs)) if gbs else None,
                "checksum_mismatches": self.checksum_mismatches, "overlap": self.overlap,
                "receiver_ms_median_max": self.recv_ms_median_max, "lane_s": self.lane_s}


def _checksum_async(t):
    """dvla_checksum64 of the region on the current stream (one read; order-
    independent, so both ends compute the same value)."""
    import torch

    from .replicate import checksum64_async
    return checksum64_async(t, torch.cuda.current_stream(t.device))


class _Keys:
    """The job's c10d store as a small key/value board shared by the lanes of
    every process.  The store client serialises its operations, so a
    blocking get in one lane would stall every other lane's set: waits poll
    with the non-blocking check() instead."""

    def __init__(self, store, ns: str, timeout_s: float, errors: list):
        self.store, self.ns, self.timeout_s, self.errors = store, ns, timeout_s, errors

    def key(self, *parts) -> str:
        return self.ns + "/".join(str(p) for p in parts)

    def set(self, k: str, value: str):
        self.store.set(k, value)

    def wait(self, keys, what: str = ""):
        deadline = time.monotonic() + self.timeout_s
        pause = 2e-4
        while not self.store.check(list(keys)):
            if self.errors:
                raise self.errors[0]
            if time.monotonic() > deadline:
                raise TimeoutError(f"disaggregated swimlane: no {what or keys} after "
                                   f"{self.timeout_s:.0f} s")
            time.sleep(pause)
            pause = min(pause * 1.5, 5e-4)

    def get(self, k: str, what: str = "") -> bytes:
        self.wait([k], what)
        return self.store.get(k)


def _fmt(c, stream) -> str:
    """The checksum as text, once `stream` (the one that computed it) got
    there.  The wait is an event synchronisation, which releases the GIL: a
    blocking .cpu() holds it for the whole wait and stalls the other lanes'
    Python (measured: the trainer lane's enqueue stretched by the ~10 ms the
    push took)."""
    import torch
    ev = torch.cuda.Event()
    ev.record(stream)
    ev.synchronize()
    with torch.cuda.stream(stream):
        return ",".join(str(int(x)) for x in c.cpu().tolist())


def run_disaggregated(cfg, learners=None, verify: bool = True,
                      poison_epochs=frozenset(), timeout_s: float = 120.0,
                      body_bytes: int = 0, engine: str = "ce_head") -> DisaggResult:
    """Collective: every rank of the job calls it (torch.distributed with
    the NCCL backend, one GPU per process).  Returns this rank's result.

    body_bytes: weights of the rest of the VLA (vision encoder + LLM body,
    out of scope as compute) carried with every published
    version as a constant blob behind the action head -- the weight-sync
    volume of BASELINE config 3 (pi0-3B: ~6.6 GB bf16) -- so replication
    moves the bytes the real system moves every iteration.

    engine: "ce_head" (default) -- the learners push with their copy
    engines (stream memory operations carry the per-chunk flags), so the
    replication holds none of the SMs the learner's GEMMs need, and the
    rollout ranks forward with the TMA chain kernel (their GPUs have idle
    SM time between sampling epochs); "sm" runs the TMA kernel on every hop
    (measured at 4 GPUs with 6.6 GB versions: ~10 % fewer trajectories/s --
    the heads' kernel takes SMs from the learner's GEMMs); "ce" uses copy
    engines on every hop (forwarding with per-chunk stream waits is slower:
    15.3 ms per version vs 9.9 for "ce_head", tools/split_sweep.py)."""
    import datetime

    import torch
    import torch.distributed as dist

    from .planes import PeerChannel
    from .pools import Pool, PoolKind
    from .replicate import SplitReplicator
    from .runtime import Monitor

    cfg.validate()
    if not dist.is_initialized():
        raise ConfigError("the disaggregated layout needs torch.distributed (one process per GPU)")
    rank, world = dist.get_rank(), dist.get_world_size()
    L = list(learners) if learners is not None else default_learners(world)
    Rr = [r for r in range(world) if r not in L]
    if not L or not Rr:
        raise ConfigError("need at least one learner and one rollout rank")
    if len(Rr) % len(L):
        raise ConfigError(f"{len(Rr)} rollout ranks do not split evenly over {len(L)} learners")
    dev = torch.device("cuda", torch.cuda.current_device())
    V, H, G, C, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.chunks, cfg.tokens
    n = V * H
    parts = len(L)                              # one chain (region part) per learner
    S = -(-(n * 2 + int(body_bytes)) // (256 * parts)) * (256 * parts)   # head + body blob
    n_traj = cfg.n_groups * G
    ring = cfg.staleness_limit + 2
    assign = {r: L[i % len(L)] for i, r in enumerate(Rr)}     # rollout rank -> learner
    k_per_learner = len(Rr) // len(L)
    errors: list = []
    raw = dist.distributed_c10d._get_default_store()
    raw.set_timeout(datetime.timedelta(seconds=timeout_s))
    _CALLS[0] += 1     # collective: every rank counts the same calls -> a fresh key space
    store = _Keys(raw, f"dvla/disagg/{_CALLS[0]}/", timeout_s, errors)
    key = store.key

    # ---- collective construction (same order on every rank)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True
    lgroup = dist.new_group(L, pg_options=opts)
    role = "learner" if rank in L else "rollout"
    model_pool = None
    if role == "learner":
        model_pool = Pool(PoolKind.MODEL_COMPUTE, n * 26 + 2 * S + (64 << 20), device=dev)
    else:
        model_pool = Pool(PoolKind.MODEL_COMPUTE, ring * S + (64 << 20), device=dev)
    # one PeerChannel per rollout rank -> its learner (one epoch per message)
    msg_bytes = n_traj * C * (H * 2 + 4 + T * 4) + n_traj * 4 + 4 * 1024 + 512
    chans = {r: PeerChannel(r, assign[r], msg_bytes, slots=cfg.queue_capacity + 1)
             for r in Rr}
    # learner i sources part i along its own chain through every rollout rank
    chains = [[L[0]] + Rr] if len(L) == 1 else \
        [[L[i]] + (Rr if i % 2 == 0 else Rr[::-1]) for i in range(len(L))]
    rep = SplitReplicator(S, chains, n_buffers=ring, ctas_per_hop=64,
                          pool=model_pool if role == "rollout" else None, engine=engine)
    res = DisaggResult(role=role, rank=rank)
    abort = threading.Event()
    monitor = Monitor(abort)
    try:
        if role == "learner":
            _learner(cfg, rank, L, Rr, assign, k_per_learner, lgroup, model_pool, chans, rep,
                     store, key, ring, S, verify, res, errors, monitor, dev)
        else:
            _rollout(cfg, rank, Rr, assign, chans, rep, store, key, ring, S, verify,
                     poison_epochs, res, errors, monitor, dev)
        torch.cuda.synchronize()
        dist.barrier()
        flag = torch.tensor([float(res.checksum_mismatches)], device=dev)
        dist.all_reduce(flag)
        res.checksum_mismatches = int(flag.item())
        # receiver-side replication time: from the hop launch (the chain heads
        # are already running) until every chunk of both parts has landed
        rt = torch.tensor([float(np.median(res.recv_ms[1:] or res.recv_ms or [0.0]))], device=dev)
        dist.all_reduce(rt, op=dist.ReduceOp.MAX)
        res.recv_ms_median_max = float(rt.item())
    finally:
        rep.close()
        for ch in chans.values():
            ch.close()
    if errors:
        raise errors[0]
    return res


def _split_epoch(msg, n_groups: int, G: int):
    """One epoch message (a whole rollout rank's epoch) -> n_groups
    GroupBatch views on the learner GPU."""
    out = []
    for gi in range(n_groups):
        sl = slice(gi * G, (gi + 1) * G)
        toks = msg.actions[sl]
        out.append(GroupBatch(group_id=msg.group_id + gi, horizon=msg.horizon, chunk=msg.chunk,
                              obs=msg.obs[sl], actions=toks,
                              behavior_log_prob=msg.behavior_log_prob[sl],
                              rewards=msg.rewards[sl], behavior_version=msg.behavior_version,
                              tokens=toks))
    return out


def _learner(cfg, rank, L, Rr, assign, k, lgroup, model_pool, chans, rep, store, key, ring, S,
             verify, res, errors, monitor, dev):
    import torch

    from .replicate import device_snapshot
    from .runtime import GradReducer, TrainerWorker
    V, H = cfg.vocab, cfg.hidden
    lead = rank == L[0]
    mine = [r for r in Rr if assign[r] == rank]
    s_train = torch.cuda.Stream(device=dev, priority=-1)
    s_dist = torch.cuda.Stream(device=dev)
    reducer = GradReducer(len(L), lgroup)
    trainer = TrainerWorker(cfg, L.index(rank), model_pool, reducer, s_train, dev,
                            n_groups=k * cfg.n_groups)
    res.policy = trainer.policy
    hb = V * H * 2
    pub = [model_pool.view(model_pool.alloc(S, align=256)) for _ in range(2)]
    if S > hb:   # the body blob: the same constant bytes on every learner, set once
        g = torch.Generator(device=dev).manual_seed(cfg.seed + 3)
        body = torch.randint(0, 256, (S - hb,), dtype=torch.uint8, device=dev, generator=g)
        for p in pub:
            p[hb:].copy_(body)
        del body
    # the body blob never changes: its share of every version's checksum is
    # taken once (sub-range checksums add up), so each version only re-reads
    # the head it rewrote
    from .replicate import checksum64_async
    body_sum = (checksum64_async(pub[0][hb:], first_word=hb // 8) if S > hb
                else torch.zeros(2, dtype=torch.int64, device=dev))
    # the initialisation above ran on this thread's default stream, which the
    # (non-blocking) trainer / weight-dist streams do not order against
    torch.cuda.synchronize(dev)
    # pub_done[i]: event after which the chain heads (and the checksum) no
    # longer read pub[i]; `pushed` = the newest version whose push has been
    # enqueued (the trainer reuses pub[v % 2] only after v - 2 was enqueued)
    pub_done = [None, None]
    pushed = [-1]
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(s_train)
    dist_q: list = []
    cv = threading.Condition()
    intervals = {"update": [], "repl": []}

    def push(v, snap):
        """Enqueue version v's chain heads on the distribution stream (and
        its checksum); learner 0 then signals the receivers."""
        b = v % 2
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        s_dist.wait_event(snap.ready)
        e0.record(s_dist)
        res.timeline.append(("push", v, time.perf_counter()))
        rep.broadcast(pub[b], v, stream=s_dist)
        e1.record(s_dist)
        if lead:   # receivers launch their hops now: the chain pipelines through them
            store.set(key("pub", v), "1")
        csum = None
        if verify and lead:
            with torch.cuda.stream(s_dist):
                csum = _checksum_async(pub[b][:hb]) + body_sum   # wraps mod 2^64
        done = torch.cuda.Event()
        done.record(s_dist)
        with cv:
            pub_done[b] = done
            pushed[0] = v
            cv.notify_all()
        if lead:
            if csum is not None:
                store.set(key("sum", v), _fmt(csum, s_dist))
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            res.replication.append({"version": v, "ms": ms, "gbs": S / (ms / 1e3) / 1e9,
                                    "t0_ms": t0.elapsed_time(e0), "t1_ms": t0.elapsed_time(e1)})

    # version 0 (the initial weights) goes out before the first epoch
    snap0 = device_snapshot(trainer.policy.weight_bf16().reshape(-1), 0, out=pub[0][:hb],
                            stream=s_train, verified=True)
    push(0, snap0)

    def dist_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            while True:
                with cv:
                    while not dist_q:
                        cv.wait(0.05)
                    item = dist_q.pop(0)
                if item is None:
                    break
                push(*item)
            rep.check()
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            monitor.fail(f"dist: {e!r}", "WeightDist", -1)

    th = threading.Thread(target=dist_lane, name="dist", daemon=True)
    th.start()
    t_pub = []
    lane = res.lane_s = {"take": 0.0, "update": 0.0, "release_wait": 0.0}
    try:
        for e in range(cfg.epochs):
            batches = []
            for r in mine:
                tt = time.perf_counter()
                msg = chans[r].take(stream=s_train)
                lane["take"] += time.perf_counter() - tt
                res.timeline.append(("took", e, time.perf_counter()))
                batches.extend(_split_epoch(msg, cfg.n_groups, cfg.group_size))
            ev_u = {kk: torch.cuda.Event(enable_timing=True)
                    for kk in ("start", "loss0", "loss1", "grad1", "reduce1", "end")}
            trainer.timing = ev_u
            try:
                tt = time.perf_counter()
                st = trainer.update(batches)
                lane["update"] += time.perf_counter() - tt
                res.timeline.append(("updated", e, time.perf_counter()))
            except GrpoAbort as ex:
                log.warning("quarantined update: %s", ex)
                res.quarantined += 1
                if lead:
                    store.set(key("proc", e), str(trainer.version))
                continue
            intervals["update"].append((t0.elapsed_time(ev_u["start"]),
                                        t0.elapsed_time(ev_u["end"])))
            names = ("start", "loss0", "loss1", "grad1", "reduce1", "end")
            res.lane_s.setdefault("update_phases_ms", []).append(
                {**{n1: round(ev_u[n0].elapsed_time(ev_u[n1]), 3)
                    for n0, n1 in zip(names, names[1:])},
                 "host_enqueue_ms": round(1e3 * ev_u["host_enqueue_s"], 3),
                 "host_wait_ms": round(1e3 * ev_u["host_wait_s"], 3)})
            v = trainer.version
            res.update_stats.append({"version": v, **{kk: st[kk] for kk in (
                "loss", "mean_ratio", "clip_fraction", "n_chunks", "grad_norm")}})
            # the ring slot of v on every rollout rank must be free
            if v - ring >= 0:
                tt = time.perf_counter()
                store.wait([key("rel", r, v - ring) for r in Rr], f"release of v{v - ring}")
                lane["release_wait"] += time.perf_counter() - tt
            b = v % 2
            with cv:                                 # v - 2's push enqueued (it reads pub[b])
                while pushed[0] < v - 2 and not errors:
                    cv.wait(0.05)
            if errors:
                raise errors[0]
            if pub_done[b] is not None:
                s_train.wait_event(pub_done[b])
            snap = device_snapshot(trainer.policy.weight_bf16().reshape(-1), v, out=pub[b][:hb],
                                   stream=s_train, verified=True)
            t_pub.append(time.perf_counter())
            res.timeline.append(("snapshot", v, t_pub[-1]))
            with cv:
                dist_q.append((v, snap))
                cv.notify_all()
            if lead:
                store.set(key("proc", e), str(v))
            res.updates += 1
    finally:
        trainer.timing = None
        with cv:
            dist_q.append(None)
            cv.notify_all()
        th.join()
        if lead:
            store.set(key("pub", trainer.version + 1), "end")
        trainer.close()
    res.epochs = cfg.epochs
    n_traj_all = len(Rr) * cfg.n_groups * cfg.group_size
    if len(t_pub) > 1:
        res.wall = t_pub[-1] - t_pub[0]
        res.trajectories_per_s = (len(t_pub) - 1) * n_traj_all / max(res.wall, 1e-12)
    intervals["repl"] = [(r["t0_ms"], r["t1_ms"]) for r in res.replication]
    if lead and intervals["repl"]:
        ov = 0.0
        for a0, a1 in intervals["repl"]:
            for b0, b1 in intervals["update"]:
                ov += max(0.0, min(a1, b1) - max(a0, b0))
        tot = sum(a1 - a0 for a0, a1 in intervals["repl"])
        res.overlap = {"replication_ms_total": tot, "overlapped_with_updates_ms": ov,
                       "fraction": ov / max(tot, 1e-12)}
    _ = (V, H)


def _rollout(cfg, rank, Rr, assign, chans, rep, store, key, ring, S, verify, poison_epochs,
             res, errors, monitor, dev):
    import torch

    from .pools import Pool, PoolKind
    from .runtime import SamplerWorker
    V, H, G, C, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.chunks, cfg.tokens
    n_traj = cfg.n_groups * G
    R = n_traj * C * T
    ri = Rr.index(rank)
    env_bytes = R * (V * 2 + H * 2 + 64) + n_traj * C * (H * 2 + 224 * 224 * 3 // 64 * 5) + \
        (16 << 20)
    env_pools = [Pool(PoolKind.ENV_AUX, env_bytes, device=dev)
                 for _ in range(cfg.staleness_limit + 2)]
    s_sample = torch.cuda.Stream(device=dev)
    s_recv = torch.cuda.Stream(device=dev)
    sampler = SamplerWorker(cfg, ri, len(Rr), env_pools, s_sample, dev)
    res.replica_of = lambda v: rep.replica(v)
    cv = threading.Condition()
    deposited: dict = {}
    hops: list = []
    state = {"done": False, "released": -1, "installed": -1}

    def release_below(v):
        # everything older than v may be overwritten by its publisher
        for u in range(state["released"] + 1, v):
            store.set(key("rel", rank, u), "1")
        state["released"] = max(state["released"], v - 1)

    def recv_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            v = 0
            while True:
                val = store.get(key("pub", v), f"publication of v{v}")
                if val == b"end":
                    break
                h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                h0.record(s_recv)
                rep.broadcast(None, v, stream=s_recv)      # this rank's hops of the chains
                h1.record(s_recv)
                hops.append((h0, h1))
                region = rep.replica(v)
                # deposit at once: the sampler's stream waits on the hop's
                # event when it installs the version (device-ordered), so the
                # host never waits for the bytes before the gate can see them
                ev = torch.cuda.Event()
                ev.record(s_recv)
                snap = ParamSnapshot(version=v, params=region[:V * H * 2].view(torch.bfloat16),
                                     ready=ev)
                with cv:
                    deposited[v] = snap
                    res.versions_received += 1
                    res.timeline.append(("received", v, time.perf_counter()))
                    if state["done"]:
                        release_below(v)
                    cv.notify_all()
                if verify:   # the replica against the learner's checksum, off the gate's path
                    with torch.cuda.stream(s_recv):
                        csum = _checksum_async(region)
                    got = _fmt(csum, s_recv)
                    want = store.get(key("sum", v), "checksum").decode()
                    if got != want:
                        res.checksum_mismatches += 1
                        res.mismatched.append((v, got, want))
                    res.timeline.append(("verified", v, time.perf_counter()))
                v += 1
            rep.check()
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            monitor.fail(f"recv: {e!r}", "WeightRecv", -1)
            with cv:
                cv.notify_all()

    th = threading.Thread(target=recv_lane, name="recv", daemon=True)
    th.start()
    ch = chans[rank]
    lane = res.lane_s = {"gate": 0.0, "epoch": 0.0}
    try:
        snap = None
        for e in range(cfg.epochs):
            need = e - cfg.staleness_limit - 1
            tt = time.perf_counter()
            vneed = int(store.get(key("proc", need), f"epoch {need} processed")) \
                if need >= 0 else 0
            with cv:
                # the gate: a version >= vneed installed or deposited
                while max(max(deposited, default=-1), state["installed"]) < vneed:
                    if errors:
                        raise errors[0]
                    cv.wait(0.05)
                if deposited and max(deposited) > state["installed"]:   # install the newest
                    newest = max(deposited)
                    snap = deposited[newest]
                    for u in [u for u in deposited if u <= newest]:
                        del deposited[u]
                    state["installed"] = newest
                    release_below(newest)
            res.installed.append(snap.version)
            lane["gate"] += time.perf_counter() - tt
            res.timeline.append(("gate_passed", e, time.perf_counter()))
            tt = time.perf_counter()
            msgs, meta = sampler.run_epoch(e, snap, poison=e in poison_epochs,
                                           group_base=(e * len(Rr) + ri) * cfg.n_groups)
            full = meta["epoch_batch"]       # the whole epoch: one message
            ch.put(full, stream=s_sample)
            lane["epoch"] += time.perf_counter() - tt
            res.timeline.append(("epoch_put", e, time.perf_counter()))
        res.epochs = cfg.epochs
        s_sample.synchronize()
    finally:
        with cv:
            state["done"] = True
        with cv:
            newest = max(deposited) if deposited else state["installed"] + 1
            release_below(max(newest, state["installed"] + 1))
        th.join()
        s_recv.synchronize()
        res.recv_ms = [a.elapsed_time(b) for a, b in hops]
