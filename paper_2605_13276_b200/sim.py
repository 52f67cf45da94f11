"""Swimlane cost model: a discrete-event simulation of the sampler / trainer
pipeline with its side channels, recalibrated with measured B200 numbers
(SURVEY §8 f4).

The event rules are the reference's (dvla/sim.py:150-374), restated over an
explicit cost tuple instead of a RunConfig:
  * the sampler may start an epoch only when
    ``version + unprocessed - installed <= staleness_limit`` (the two-ended
    gate, sim.py:232-234); the trainer may publish V+1 only when no sampler
    is mid-epoch with ``installed < V+1-limit`` (sim.py:236-240);
  * a finished epoch waits for queue space (``queue_capacity`` batches) and
    becomes takeable ``transfer_s`` later (sim.py:285-293);
  * published weights land ``broadcast_s`` after the publish, latest-wins,
    and are installed only at an epoch boundary (sim.py:242-264, 270-278);
  * with several nodes every trainer reaches the pacing barrier and the
    update is published ``reduce_s`` after the last one (sim.py:305-314);
  * tasks sharing a slot group progress at rate 1/k (linear contention,
    sim.py:328-334) — by default, as in the reference, one group per role
    across all nodes; ``per_node_slots=True`` gives every node its own
    (B200 topology replication: one GPU per closed loop).
Sync mode is roll + transfer + actor + broadcast + reduce per epoch
(sim.py:150-169).  Results match the reference on its own cost inputs
(tests/golden/sim_cases.json, tests/test_sim.py).

``b200_costs`` fills the cost tuple from measured B200 rates (bench.py /
MEASURED_PEAKS.json numbers: cuBLAS bf16 TFLOP/s for the head GEMMs, HBM
GB/s for the sampling, fused-loss and Adam kernels, NVLink GB/s for weight
replication, NCCL bus bandwidth for the gradient mean) and ``fit_check``
compares a prediction with a live ``run_swimlane`` summary (sim.py:416-439).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .core import ConfigError

_EPS = 1e-12


@dataclass(frozen=True)
class LaneCosts:
    """Per-epoch costs (seconds) of one node's lanes, run alone."""

    rollout_s: float            # sampler: one epoch of rollout incl. inference
    actor_s: float              # trainer: one update on one epoch
    transfer_s: float = 0.0     # sampler -> trainer batch handoff
    broadcast_s: float = 0.0    # trainer -> sampler weight delivery
    reduce_s: float = 0.0       # cross-node gradient mean
    shared_slots: bool = False  # sampler and trainer contend for the same slots
    transitions_per_epoch: int = 1

    def validate(self):
        for k in ("rollout_s", "actor_s", "transfer_s", "broadcast_s", "reduce_s"):
            v = getattr(self, k)
            if not (v >= 0.0):
                raise ConfigError(f"{k} must be >= 0, got {v}")
        if self.rollout_s <= 0.0 or self.actor_s <= 0.0:
            raise ConfigError("rollout_s and actor_s must be > 0")


@dataclass
class SimResult:
    mode: str
    throughput: float           # transitions/s after warm-up
    step_time: float
    rollout_time: float
    actor_time: float
    transfer_time: float
    broadcast_time: float
    bottleneck: str
    occupancy: dict
    staleness_max: int
    total_transitions: int
    wall: float
    epochs: list = field(default_factory=list)


def _bottleneck(roll, act, xfer):
    top = max(roll, act, xfer)
    return "Rollout" if top == roll else ("Actor" if top == act else "Transfer")


def _summarise(mode, rows, wall, busy, staleness_max, warmup):
    post = rows[warmup:] if len(rows) > warmup else rows
    mean = {k: sum(r[k] for r in post) / len(post)
            for k in ("step_time", "rollout_time", "actor_time", "transfer_time",
                      "broadcast_time")}
    trans = sum(r["transitions"] for r in post)
    t0 = rows[warmup - 1]["end"] if warmup and len(rows) > warmup else 0.0
    return SimResult(
        mode=mode, throughput=trans / max(post[-1]["end"] - t0, _EPS),
        step_time=mean["step_time"], rollout_time=mean["rollout_time"],
        actor_time=mean["actor_time"], transfer_time=mean["transfer_time"],
        broadcast_time=mean["broadcast_time"],
        bottleneck=_bottleneck(mean["rollout_time"], mean["actor_time"], mean["transfer_time"]),
        occupancy={k: v / max(wall, _EPS) for k, v in busy.items()},
        staleness_max=staleness_max, total_transitions=trans, wall=wall, epochs=rows)


def _row(epoch, roll, act, xfer, bcast, step, trans, end):
    return {"epoch": epoch, "rollout_time": roll, "actor_time": act, "transfer_time": xfer,
            "broadcast_time": bcast, "step_time": step, "transitions": trans, "end": end}


def simulate_sync(c: LaneCosts, epochs: int, warmup_epochs: int = 1) -> SimResult:
    c.validate()
    step = c.rollout_s + c.transfer_s + c.actor_s + (c.broadcast_s + c.reduce_s)
    rows, t = [], 0.0
    for e in range(epochs):
        t += step
        rows.append(_row(e, c.rollout_s, c.actor_s, c.transfer_s, c.broadcast_s + c.reduce_s,
                         step, c.transitions_per_epoch, t))
    busy = {"sampler": c.rollout_s * epochs, "trainer": c.actor_s * epochs}
    return _summarise("sync", rows, t, busy, 0, warmup_epochs)


class _Lanes:
    """One node's sampler and trainer lane state."""

    def __init__(self, idx):
        self.idx = idx
        self.sampler = "boundary"     # boundary -> rolling -> enqueue -> boundary | done
        self.epoch = 0                # epochs the sampler has handed off
        self.installed = 0            # weight version the sampler runs with
        self.mailbox = None           # (version, arrival) latest-wins
        self.finished = None          # (epoch, rollout wall) waiting for queue space
        self.queue = []               # [(epoch, version, available_at, rollout wall)]
        self.trainer = "take"         # take -> training -> pacing -> take | done
        self.last_roll = 0.0
        self.last_train = 0.0
        self.busy_s = 0.0
        self.busy_t = 0.0

    def in_flight(self):
        """Epochs produced whose update is not yet published."""
        return (len(self.queue) + (self.finished is not None)
                + (self.trainer in ("training", "pacing")))


class _Async:
    def __init__(self, c: LaneCosts, nodes, epochs, limit, qcap, per_node_slots):
        self.c, self.epochs, self.limit, self.qcap = c, epochs, limit, qcap
        self.per_node = per_node_slots
        self.nodes = [_Lanes(i) for i in range(nodes)]
        self.t = 0.0
        self.version = 0
        self.version_at = 0.0
        self.staleness_max = 0
        self.tasks = []               # [kind, node, remaining work, slot group, start]
        self.timers = []              # future instants something becomes ready
        self.arrived = {}             # node -> time it reached the pacing barrier
        self.publish_due = None
        self.rows = []

    def group(self, kind, node):
        g = "shared" if self.c.shared_slots else kind
        return (g, node.idx) if self.per_node else g

    def load(self, group):
        return sum(1 for task in self.tasks if task[3] == group)

    def start(self, kind, node, work):
        self.tasks.append([kind, node, work, self.group(kind, node), self.t])

    def publish(self):
        self.version += 1
        v, t = self.version, self.t
        for nd in self.nodes:
            if nd.sampler == "rolling":
                self.staleness_max = max(self.staleness_max, v - nd.installed)
            at = t + self.c.broadcast_s
            if nd.mailbox is None or v > nd.mailbox[0]:
                nd.mailbox = (v, at)
            if at > t:
                self.timers.append(at)
        n0 = self.nodes[0]
        self.rows.append(_row(v - 1, n0.last_roll, n0.last_train, self.c.transfer_s,
                              self.c.broadcast_s, t - self.version_at if v > 1 else t,
                              self.c.transitions_per_epoch, t))
        self.version_at = t
        for nd in self.nodes:
            nd.trainer = "done" if v >= self.epochs else "take"

    def may_publish(self, nxt):
        return all(not (nd.sampler == "rolling" and nd.installed < nxt - self.limit)
                   for nd in self.nodes)

    def settle(self):
        """Apply every state change possible at the current instant."""
        t, c = self.t, self.c
        changed = True
        while changed:
            changed = False
            for nd in self.nodes:
                if nd.sampler == "boundary":
                    if nd.mailbox is not None:
                        if nd.mailbox[1] <= t + _EPS:
                            nd.installed = max(nd.installed, nd.mailbox[0])
                            nd.mailbox = None
                            changed = True
                        else:
                            self.timers.append(nd.mailbox[1])
                    if nd.epoch >= self.epochs:
                        nd.sampler = "done"
                        changed = True
                    elif self.version + nd.in_flight() - nd.installed <= self.limit:
                        self.staleness_max = max(self.staleness_max,
                                                 self.version - nd.installed)
                        nd.sampler = "rolling"
                        self.start("roll", nd, c.rollout_s)
                        changed = True
                if nd.sampler == "enqueue" and len(nd.queue) < self.qcap:
                    ep, wall = nd.finished
                    nd.finished = None
                    nd.queue.append((ep, nd.installed, t + c.transfer_s, wall))
                    if c.transfer_s > 0:
                        self.timers.append(t + c.transfer_s)
                    nd.epoch += 1
                    nd.sampler = "boundary"
                    changed = True
                if nd.trainer == "take" and nd.queue:
                    if nd.queue[0][2] <= t + _EPS:
                        nd.last_roll = nd.queue.pop(0)[3]
                        nd.trainer = "training"
                        self.start("train", nd, c.actor_s)
                        changed = True
                    else:
                        self.timers.append(nd.queue[0][2])
                if (nd.trainer == "pacing" and nd.idx not in self.arrived
                        and self.may_publish(self.version + 1)):
                    self.arrived[nd.idx] = t
                    changed = True
            if len(self.arrived) == len(self.nodes) and self.publish_due is None:
                at = max(self.arrived.values()) + c.reduce_s
                self.arrived = {}
                if at <= t + _EPS:
                    self.publish()
                else:
                    self.publish_due = at
                    self.timers.append(at)
                changed = True

    def advance(self):
        """Move time to the next task completion or timer."""
        t = self.t
        nxt = [t + task[2] * self.load(task[3]) for task in self.tasks]
        nxt += [w for w in self.timers if w > t + _EPS]
        if not nxt:
            raise RuntimeError(f"simulation blocked at version {self.version}")
        t1 = min(nxt)
        dt = max(t1 - t, 0.0)
        rates = [1.0 / self.load(task[3]) for task in self.tasks]
        for task, r in zip(self.tasks, rates):
            task[2] -= dt * r
        self.t = t1
        self.timers = [w for w in self.timers if w > t1 + _EPS]
        for task in [x for x in self.tasks if x[2] <= 1e-9]:
            self.tasks.remove(task)
            kind, nd, _, _, t0 = task
            wall = t1 - t0
            if kind == "roll":
                nd.busy_s += wall
                nd.finished = (nd.epoch, wall)
                nd.sampler = "enqueue"
            else:
                nd.busy_t += wall
                nd.last_train = wall
                nd.trainer = "pacing"
        if self.publish_due is not None and self.publish_due <= t1 + _EPS:
            self.publish_due = None
            self.publish()

    def run(self):
        self.settle()
        steps = 0
        while any(nd.trainer != "done" for nd in self.nodes):
            steps += 1
            if steps > 500000:
                raise RuntimeError("simulation failed to converge")
            self.advance()
            self.settle()
        n = len(self.nodes)
        busy = {"sampler": sum(nd.busy_s for nd in self.nodes) / n,
                "trainer": sum(nd.busy_t for nd in self.nodes) / n}
        return self.rows, self.t, busy


def simulate_async(c: LaneCosts, epochs: int, staleness_limit: int = 1,
                   queue_capacity: int = 2, nodes: int = 1, warmup_epochs: int = 1,
                   per_node_slots: bool = False) -> SimResult:
    c.validate()
    if staleness_limit < 0 or queue_capacity < 1 or nodes < 1 or epochs < 1:
        raise ConfigError("need staleness_limit >= 0, queue_capacity >= 1, nodes >= 1, "
                          "epochs >= 1")
    sim = _Async(c, nodes, epochs, staleness_limit, queue_capacity, per_node_slots)
    rows, wall, busy = sim.run()
    return _summarise("async", rows, wall, busy, sim.staleness_max, warmup_epochs)


def simulate(c: LaneCosts, mode: str = "async", **kw) -> SimResult:
    if mode == "sync":
        return simulate_sync(c, kw["epochs"], kw.get("warmup_epochs", 1))
    if mode != "async":
        raise ConfigError(f"mode must be 'sync' or 'async', got {mode!r}")
    return simulate_async(c, **kw)


# ------------------------------------------------------- B200 calibration

@dataclass(frozen=True)
class B200Rates:
    """Measured B200 rates (defaults: round-1 bench.py / MEASURED_PEAKS.json)."""

    gemm_tflops: float = 1692.6        # cuBLAS bf16 (MEASURED_PEAKS bf16_tflops)
    hbm_gbs: float = 6434.2            # device copy peak (MEASURED_PEAKS)
    loss_frac: float = 0.785           # fused loss kernel, fraction of hbm_gbs (bench)
    sample_frac: float = 0.97          # rollout sampling kernel (bench)
    adam_frac: float = 0.955           # Adam (bench)
    nvlink_gbs: float = 705.0          # chain replication per receiver (bench / C5 sweep)
    allreduce_busbw_gbs: float = 634.0  # NCCL, 1 GiB, 4 GPUs (bench)
    launch_overhead_s: float = 0.5e-3  # host lane bookkeeping per epoch (fit)


def b200_costs(n_groups: int = 64, group_size: int = 8, chunks: int = 1, tokens: int = 56,
               vocab: int = 32064, hidden: int = 4096, replicas: int = 0, nodes: int = 1,
               rates: B200Rates = B200Rates(), shared_gpu: bool = True,
               peer_exchange: bool = True, gather_chunks: int = 4) -> LaneCosts:
    """Lane costs of the token-head swimlane (runtime.run_swimlane) on B200.

    Sampler: logits GEMM [R, H] x [H, V] + one-pass sampling over the logits.
    Trainer (TrainerWorker.update, round 2): logits GEMM + fused loss
    fwd/bwd (2 R V bf16 bytes) + the head-gradient GEMM (f32 output, 4 n
    bytes written) + the [R, H] feature expansion + grad norm (4 n / N read)
    + the optimizer tail on this learner's 1/N of the parameters (46 B each:
    f32 gradient, f64 moments, f32 master, bf16 copy) + the snapshot copy of
    the bf16 weights.  With ``nodes`` = N > 1 learners the gradient is
    reduce-scattered (f32) and the bf16 blocks all-gathered (ZeRO-1):
    with ``peer_exchange`` (exchange.PeerGradExchange, the default) both are
    copy-engine pushes under the gradient GEMM / optimizer tail, so only the
    own half's peer blocks (pushed after the last GEMM), the last optimizer
    chunk's pushes and the node-order sum (N + 1 blocks read / written)
    remain exposed; with NCCL, (N - 1) / N (4 + 2) n bytes per GPU and
    direction at the measured bus bandwidth.  Weight replication to
    ``replicas`` other GPUs over the chain."""
    R = n_groups * group_size * chunks * tokens
    n = vocab * hidden
    N = max(int(nodes), 1)
    gemm = 2.0 * R * hidden * vocab / (rates.gemm_tflops * 1e12)
    hbm = rates.hbm_gbs * 1e9
    roll = gemm + R * vocab * 2 / (hbm * rates.sample_frac) + rates.launch_overhead_s
    loss = 2 * R * vocab * 2 / (hbm * rates.loss_frac)
    tail = 46.0 * n / N / (hbm * rates.adam_frac)
    snap = 2 * n * 2 / hbm
    passes = (4.0 * n + 4.0 * n / N + 2 * R * hidden * 2) / hbm
    act = 2 * gemm + loss + tail + snap + passes + rates.launch_overhead_s
    bcast = (n * 2 / (rates.nvlink_gbs * 1e9)) if replicas else 0.0
    if N == 1:
        reduce = 0.0
    elif peer_exchange:
        own_half = N // 2 if N > 2 else 1
        pushes = (own_half - 1) * 4.0 * n / N + (N - 1) * 2.0 * n / N / max(gather_chunks, 1)
        reduce = pushes / (rates.nvlink_gbs * 1e9) + (N + 1) * 4.0 * n / N / hbm
    else:
        reduce = (N - 1) / N * n * (4 + 2) / (rates.allreduce_busbw_gbs * 1e9)
    return LaneCosts(rollout_s=roll, actor_s=act, broadcast_s=bcast, reduce_s=reduce,
                     shared_slots=shared_gpu, transitions_per_epoch=R)


def fit_check(sim: SimResult, live: dict, threshold: float = 0.10) -> dict:
    """Relative deviation of a live aggregate from a prediction (reference
    sim.py:416-439).  ``live`` needs mode, throughput, rollout_time and
    actor_time; a different mode is an error, not a deviation."""
    if live.get("mode") != sim.mode:
        raise ConfigError("fit_check: live run and simulation modes differ")

    def dev(a, b):
        return abs(a - b) / max(abs(b), _EPS)

    rep = {"throughput_dev": dev(live["throughput"], sim.throughput),
           "rollout_dev": dev(live["rollout_time"], sim.rollout_time),
           "actor_dev": dev(live["actor_time"], sim.actor_time),
           "threshold": threshold}
    rep["pass"] = all(rep[k] <= threshold for k in ("throughput_dev", "rollout_dev", "actor_dev"))
    return rep
