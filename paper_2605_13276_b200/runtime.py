"""The four-lane swimlane on B200: sampler, weight-receive, trainer and
weight-distribution lanes as host threads, each driving its own CUDA stream.

Mirrors the coordination of reference pkg/src/dvla/runtime.py (LaneId :53-57,
RunAbort :65-79, Monitor :120-156, VersionBoard busy-mode gate :211-564,
GradReducer :569-637, SamplerWorker :655-729, TrainerWorker :732-800,
_run_async lanes :1157-1318) with the data plane kept on the device:

  * rollouts are produced on the SAMPLER stream and handed to the trainer as
    device-resident GroupBatch objects through a bounded Channel (zero copy);
  * the TRAINER stream runs the fused token loss (csrc/token_loss.cu), the
    head-gradient GEMM (cuBLAS), the NCCL gradient all-reduce (multi-GPU) and
    Adam (csrc/optim.cu);
  * the WEIGHT_DIST stream snapshots the parameters into a double-buffered
    MODEL_COMPUTE region (fused copy + isfinite) and broadcasts it;
  * the WEIGHT_RECV lane installs the newest snapshot at epoch boundaries
    (latest-wins mailbox + staleness gate), a pointer swap -- no copy.
Cross-stream ordering uses CUDA events; cross-lane ordering uses the same
three host primitives as the reference (bounded channel, latest-wins
mailbox, two-ended staleness gate).

The policy is an action-token head: logits = features @ W^T with W the
[V, H] head matrix (OpenVLA-style: the last 256 of V ids are action bins);
features are a fixed random projection of synthetic LIBERO-shaped
observations (224x224x3 uint8 + 8-d proprio summarised to H dims).  The VLA
body is out of scope; the hot path is everything after it.
"""

from __future__ import annotations

import contextlib
import logging
import math
import os
import threading
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .core import ConfigError, ParamSnapshot
from .grpo import GroupBatch, GrpoAbort, GrpoConfig, TokenLoss

log = logging.getLogger("dvla_b200.runtime")


class LaneId(Enum):
    SAMPLER = "Sampler"
    WEIGHT_RECV = "WeightRecv"
    TRAINER = "Trainer"
    WEIGHT_DIST = "WeightDist"


class RunAbort(RuntimeError):
    """Run-level failure: watchdog timeout or a poisoned update."""

    def __init__(self, reason: str, lane: str = "", epoch: int = -1,
                 lane_states: dict | None = None):
        self.reason = reason
        self.lane = lane
        self.epoch = epoch
        self.lane_states = lane_states or {}
        super().__init__(f"{reason} (lane={lane or 'n/a'}, epoch={epoch}); "
                         f"lanes: {self.lane_states}")


class Monitor:
    """Lane heartbeat registry; the watchdog aborts silent runs."""

    def __init__(self, abort: threading.Event):
        self.abort = abort
        self._lock = threading.Lock()
        self._lanes: dict = {}
        self.abort_reason: str | None = None
        self.abort_lane = ""
        self.abort_epoch = -1

    def beat(self, lane: str, state: str | None = None):
        with self._lock:
            prev = self._lanes.get(lane)
            self._lanes[lane] = (time.perf_counter(),
                                 state if state is not None else (prev[1] if prev else "run"))

    def fail(self, reason: str, lane: str, epoch: int):
        with self._lock:
            if self.abort_reason is None:
                self.abort_reason, self.abort_lane, self.abort_epoch = reason, lane, epoch
        self.abort.set()

    def dump(self) -> dict:
        with self._lock:
            now = time.perf_counter()
            return {ln: f"{st} (last beat {now - ts:.2f}s ago)"
                    for ln, (ts, st) in self._lanes.items()}

    def stale_lanes(self, timeout: float) -> list:
        with self._lock:
            now = time.perf_counter()
            return [ln for ln, (ts, st) in self._lanes.items()
                    if st != "done" and now - ts > timeout]


class VersionBoard:
    """Two-ended staleness gate (reference runtime.py:211-564, busy mode).
    The reference's methods also take the lane clock / virtual timestamps
    (its virtual-time mode); they are accepted and ignored here (busy mode,
    real time only).

    Sampler end: an epoch may start iff version + produced - processed -
    installed <= limit (wait_gate).  Trainer end: version V+1 may be
    published iff the sampler is between epochs or has installed at least
    V+1-limit (wait_pacing).  Deliveries older than the installed version
    are ignored and counted (deposit)."""

    def __init__(self, limit: int, monitor: Monitor, snap0: ParamSnapshot):
        self.limit = limit
        self.monitor = monitor
        self._c = threading.Condition()
        self.version = 0
        self.produced = 0
        self.processed = 0
        self.installed = 0
        self.snap = snap0
        self.at_boundary = True
        self.sampler_done = False
        self.staleness_max = 0
        self.regressions_ignored = 0
        self.delivered: dict = {}
        self.epoch_meta: dict = {}
        self.retired_max = -1   # versions <= this one's buffer has been reused

    def deposit(self, snap: ParamSnapshot, *_virtual_time):
        with self._c:
            if snap.version <= self.installed or snap.version in self.delivered or \
                    snap.version <= self.retired_max:
                self.regressions_ignored += 1
                log.warning("ignoring stale weight snapshot v%d (installed v%d)", snap.version,
                            self.installed)
                return
            self.delivered[snap.version] = snap
            self._c.notify_all()

    def boundary(self, *_clock):
        with self._c:
            self.at_boundary = True
            self._c.notify_all()

    def produce(self, epoch: int, meta: dict):
        with self._c:
            self.epoch_meta[epoch] = meta
            self.produced += 1
            self._c.notify_all()

    def take_meta(self, epoch: int) -> dict:
        with self._c:
            return self.epoch_meta.pop(epoch)

    def mark_sampler_done(self, *_clock):
        with self._c:
            self.sampler_done = True
            self.at_boundary = True
            self._c.notify_all()

    def wait_gate(self, *_clock):
        """Block until the gate admits the next epoch; installs the newest
        delivered snapshot first (epoch-boundary install).  Returns
        (snapshot, staleness)."""
        with self._c:
            while True:
                if self.monitor.abort.is_set():
                    from .planes import RunAborted
                    raise RunAborted("abort in gate wait")
                newest = max(self.delivered, default=0)
                if newest > self.installed:
                    self.installed = newest
                    self.snap = self.delivered[newest]
                    for v in [k for k in self.delivered if k <= newest]:
                        del self.delivered[v]
                    self._c.notify_all()
                if self.version + self.produced - self.processed - self.installed <= self.limit:
                    stal = self.version - self.installed
                    self.staleness_max = max(self.staleness_max, stal)
                    self.at_boundary = False
                    return self.snap, stal
                self.monitor.beat(LaneId.SAMPLER.value, "gate-wait")
                self._c.wait(0.05)

    def wait_pacing(self, next_version: int, *_clock):
        with self._c:
            while True:
                if self.monitor.abort.is_set():
                    from .planes import RunAborted
                    raise RunAborted("abort in pacing wait")
                if self.sampler_done or self.at_boundary or \
                        self.installed >= next_version - self.limit:
                    return
                self.monitor.beat(LaneId.TRAINER.value, "pacing-wait")
                self._c.wait(0.05)

    def publish(self, *_clock) -> int:
        with self._c:
            self.version += 1
            self.processed += 1
            if not self.at_boundary:
                self.staleness_max = max(self.staleness_max, self.version - self.installed)
            self._c.notify_all()
            return self.version

    def quarantine(self, *_clock):
        with self._c:
            self.processed += 1
            self._c.notify_all()

    def retire(self, version: int):
        """The publisher is about to reuse the buffer of `version` (a ring of
        published-weight regions): wait until the sampler no longer reads
        it or anything older (a newer version is installed -- the gate
        installs the newest delivered one at every epoch boundary, and the
        versions between it and the one about to be published already are
        published), then drop it and everything
        older from the pending deliveries so it can never be installed."""
        if version < 0:
            return
        with self._c:
            while self.installed <= version and not self.sampler_done:
                if self.monitor.abort.is_set():
                    from .planes import RunAborted
                    raise RunAborted("abort in retire wait")
                self.monitor.beat(LaneId.TRAINER.value, "retire-wait")
                self._c.wait(0.05)
            self.retired_max = max(self.retired_max, version)
            for v in [k for k in self.delivered if k <= version]:
                del self.delivered[v]


class GradReducer:
    """Cross-node gradient mean (reference runtime.py:569-637).

    The reference ships every node's gradient as an f32 frame, sums the
    decoded frames in f64 in node order and divides by `nodes`.  Here the
    gradient is quantised to f32 exactly as the frame would be, then
    all-reduced:
      * `exact=True`: NCCL sum of the f32 values in f64 (the reference's
        arithmetic up to summation order);
      * backend "nvls": the switch-reduced all-reduce over NVSwitch multicast
        memory (`replicate.McAllReduce`, f32 sums in the switch, 1/nodes
        applied in the same pass; 685 vs 635 GB/s busbw for NCCL's ring at
        1 GiB on 4 B200);
      * backend "nccl": NCCL f32 all-reduce.
    The default is NCCL (the north star's gradient path); "auto" picks nvls
    from 4 nodes up when the box has NVSwitch multicast and the sum need not
    be exact: per GPU and link direction it moves
    (N + 1) / N of the buffer against the ring's 2 (N - 1) / N, so at 2
    nodes the ring wins (569 vs 400 GB/s busbw measured).  Single-node runs
    are a no-op, as in the reference."""

    def __init__(self, nodes: int, group=None, exact: bool = False, backend: str = "nccl",
                 scatter: str = "auto"):
        if backend not in ("auto", "nccl", "nvls"):
            raise ConfigError(f"unknown gradient reduction backend {backend!r}")
        if exact and backend == "nvls":
            raise ConfigError("exact=True needs the NCCL f64 path")
        if scatter not in ("auto", "peer", "nccl"):
            raise ConfigError(f"unknown reduce-scatter transport {scatter!r}")
        self.nodes = nodes
        self.group = group
        self.exact = exact
        self.backend = backend
        # TrainerWorker's ZeRO-1 reduce-scatter: "peer" = copy-engine pushes
        # over NVLink overlapped with the gradient GEMM + a node-order f64 sum
        # (exchange.PeerGradExchange); "nccl" = NCCL reduce_scatter after the
        # GEMM; "auto" = peer when every rank is on this host's GPUs
        self.scatter = scatter
        self._ar = None

    def peer_scatter(self) -> bool:
        """Collective: True when the ZeRO-1 reduce-scatter runs over peer
        memory (scatter "peer", or "auto" with every rank on one host)."""
        if self.scatter == "nccl" or self.nodes == 1:
            return False
        if self.scatter == "peer":
            return True
        import socket

        from .replicate import _gather_by_rank
        hosts = set(_gather_by_rank(socket.gethostname(), self.group).values())
        self.scatter = "peer" if len(hosts) == 1 else "nccl"
        return self.scatter == "peer"

    def _use_nvls(self, grad) -> bool:
        if self.exact or self.backend == "nccl" or self.nodes == 1 or not grad.is_cuda:
            return False
        if self.backend == "nvls":
            return True
        if self.nodes < 4:
            self.backend = "nccl"
            return False
        from .replicate import multicast_supported
        import torch
        import torch.distributed as dist
        ok = torch.tensor([1.0 if multicast_supported() else 0.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        self.backend = "nvls" if ok.item() == 1.0 else "nccl"
        return self.backend == "nvls"

    def reduce(self, *args):
        """The mean of this rank's gradient over the nodes.  Called as
        reduce(grad), or with the reference's signature reduce(node, round,
        grad, clock) (runtime.py:596-627: there every node is a thread of one
        process; here every node is a process, so node / round / clock carry
        no information)."""
        if len(args) == 1:
            grad = args[0]
        elif len(args) in (3, 4):
            grad = args[2]
        else:
            raise TypeError("reduce(grad) or reduce(node, round, grad, clock)")
        return self._reduce(grad)

    def reduce_serial(self, rnd: int, grads: list):
        """Sync-mode path (reference runtime.py:629-637): every node's
        gradient on hand in one place; each is quantised to the f32 frame,
        summed in f64 in node order and divided by the node count -- the
        reference's arithmetic.  numpy in -> numpy out; tensors stay on the
        first gradient's device."""
        del rnd
        if self.nodes == 1 or len(grads) == 1:
            return grads[0]
        if isinstance(grads[0], np.ndarray):
            total = np.zeros(grads[0].shape[0], dtype=np.float64)
            for g in grads:
                total += np.asarray(g).astype(np.float32).astype(np.float64)
            return total / len(grads)
        import torch
        dev = grads[0].device
        total = torch.zeros(grads[0].numel(), dtype=torch.float64, device=dev)
        for g in grads:
            total += g.reshape(-1).to(dev).to(torch.float32).to(torch.float64)
        return total / len(grads)

    def _reduce(self, grad):
        import torch
        import torch.distributed as dist
        if self.nodes == 1:
            return grad
        if self._use_nvls(grad):
            from .replicate import McAllReduce
            n = grad.numel()
            if self._ar is None or self._ar.n < n:
                if self._ar is not None:
                    self._ar.close()
                from ._lib import NativeError
                try:
                    self._ar = McAllReduce((n + 3) // 4 * 4, group=self.group)
                except NativeError:  # raised on every rank alike: fall back together
                    self._ar = None
                    self.backend = "nccl"
                    return self._reduce(grad)
                self._ar.buf.zero_()
            self._ar.buf[:n].copy_(grad.reshape(-1))  # f32 quantisation (the frame)
            self._ar.allreduce(scale=1.0 / self.nodes)
            out = self._ar.buf[:n].to(grad.dtype).reshape(grad.shape)
            return out
        q = grad.to(torch.float32)
        if self.exact:
            q = q.to(torch.float64)
        dist.all_reduce(q, op=dist.ReduceOp.SUM, group=self.group)
        return q.to(grad.dtype) / self.nodes if q.dtype != grad.dtype else q / self.nodes

    def overlappable(self, grad) -> bool:
        """True when reduce_async can take the gradient bucket by bucket
        (NCCL f32 sum; the caller divides by `nodes`)."""
        return self.nodes > 1 and not self.exact and not self._use_nvls(grad)

    def reduce_async(self, bucket):
        """In-place NCCL sum of one f32 gradient bucket, asynchronous: NCCL's
        stream waits for the current stream at this call, so the next
        bucket's GEMM overlaps this bucket's all-reduce; wait() on the
        returned work makes the current stream wait for the sum.  The mean's
        division by `nodes` is the caller's (fused into the optimizer tail)."""
        import torch.distributed as dist
        return dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=self.group, async_op=True)

    def close(self):
        if self._ar is not None:
            self._ar.close()
            self._ar = None


# --------------------------------------------------------------- workers
@dataclass
class SwimlaneConfig:
    """Shapes of the token-head swimlane (defaults: small enough to run in
    seconds; BASELINE config 4 uses V=32064, T=56, 64 groups/GPU)."""

    n_groups: int = 8            # groups per epoch per GPU
    group_size: int = 8
    chunks: int = 1
    tokens: int = 56             # action tokens per chunk (8 steps x 7 DoF)
    vocab: int = 32064
    action_bins: int = 256       # OpenVLA: the last 256 token ids
    hidden: int = 1024
    epochs: int = 6
    staleness_limit: int = 1
    queue_capacity: int = 2      # epochs of groups buffered in the channel
    lr: float = 1e-4
    seed: int = 0
    watchdog_s: float = 60.0
    max_grad_norm: float | None = None
    # torch's own temporaries (concatenations, sampling outputs) in an
    # ENV_AUX pool through a MemPool (pools.TorchArena); 0 = torch's allocator
    torch_pool_bytes: int = 256 << 20

    def validate(self):
        if self.group_size < 2:
            raise ConfigError("group_size must be >= 2")
        if self.action_bins > self.vocab:
            raise ConfigError("action_bins must be <= vocab")
        if self.staleness_limit < 0:
            raise ConfigError("staleness_limit must be >= 0")


def token_positions(cfg: "SwimlaneConfig", device):
    """Per-position embeddings [T, H] (bf16, fixed random, seed cfg.seed + 2):
    the feature of action token t of a chunk is the chunk's observation
    feature + positions[t], so the T rows of a chunk have distinct logits
    (an autoregressive VLA decodes each action token from its own hidden
    state).  The sampler and the trainer build the same table."""
    import torch
    g = torch.Generator(device=device).manual_seed(cfg.seed + 2)
    return (torch.randn(cfg.tokens, cfg.hidden, device=device, generator=g) * 0.05).to(
        torch.bfloat16)


def expand_token_features(feats, pos, out):
    """out[(c, t)] = feats[c] + pos[t] (bf16; one broadcast kernel):
    feats [n_chunks, H], pos [T, H], out [n_chunks * T, H]."""
    import torch
    nc, H = feats.shape[0], feats.shape[-1]
    T = pos.shape[0]
    torch.add(feats.reshape(nc, 1, H), pos.reshape(1, T, H), out=out.view(nc, T, H))
    return out


class TokenPolicy:
    """Action-token head W [V, H]: f32 master weights, f64 Adam moments and
    the bf16 working copy (what the forward GEMM reads; the optimizer tail
    rewrites it as it steps the master weights) in a MODEL_COMPUTE pool.

    shard=(rank, N): ZeRO-1 layout for N learner GPUs -- the head's rows are
    cut into N blocks of Vs = ceil(V / N) rows; this rank keeps the master
    weights and moments of block `rank` only (the rows past V are zero
    padding), the bf16 working copy of all blocks (all-gathered after each
    step, so every rank holds the same bytes)."""

    def __init__(self, cfg: SwimlaneConfig, pool, device, shard=None):
        import torch
        V, H = cfg.vocab, cfg.hidden
        r, N = shard if shard is not None else (0, 1)
        Vs = -(-V // N)
        nloc = Vs * H
        g = torch.Generator(device=device).manual_seed(cfg.seed)
        self.hm = pool.alloc(nloc * 4, align=256)
        self.hmm = pool.alloc(nloc * 8, align=256)
        self.hmv = pool.alloc(nloc * 8, align=256)
        self.hw = pool.alloc(N * nloc * 2, align=256)
        full = torch.zeros(N * nloc, dtype=torch.float32, device=device)
        full[:V * H] = torch.randn(V * H, device=device, generator=g) * (H ** -0.5)
        self.master = pool.view(self.hm, torch.float32)[:nloc]
        self.master.copy_(full[r * nloc:(r + 1) * nloc])
        self.m = pool.view(self.hmm, torch.float64)[:nloc]
        self.v = pool.view(self.hmv, torch.float64)[:nloc]
        self.m.zero_()
        self.v.zero_()
        self.w16pad = pool.view(self.hw, torch.bfloat16)[:N * nloc]
        self.w16pad.copy_(full)
        self.w16 = self.w16pad[:V * H].view(V, H)
        self.w16_own = self.w16pad[r * nloc:(r + 1) * nloc]
        del full
        self.step = 0
        self.V, self.H, self.Vs, self.rank, self.N = V, H, Vs, r, N

    def weight_bf16(self):
        """The bf16 head (round-to-nearest of the master weights), kept
        current by the optimizer tail: no copy."""
        return self.w16


class SamplerWorker:
    """One per GPU: owns the epoch-recycled ENV_AUX pools, the observation
    projection and the SAMPLER stream (reference runtime.py:655-729).
    run_epoch produces one epoch of device-resident GroupBatch messages with
    the installed weights read in place."""

    def __init__(self, cfg: SwimlaneConfig, node: int, nodes: int, env_pools, stream, device,
                 torch_arena=None):
        import torch
        self.torch_arena = torch_arena
        self.cfg, self.node, self.nodes = cfg, node, nodes
        self.env_pools, self.stream, self.device = env_pools, stream, device
        H = cfg.hidden
        self.proj = torch.randn(224 * 224 * 3 // 64 + 8, H, device=device,
                                generator=torch.Generator(device=device).manual_seed(
                                    cfg.seed + 1)) * 0.05
        self.pos = token_positions(cfg, device)
        self.rng = torch.Generator(device=device).manual_seed(cfg.seed * 7919 + node)
        torch.cuda.synchronize(device)   # tables built on the default stream

    def run_epoch(self, epoch: int, snap: ParamSnapshot, poison: bool = False,
                  group_base: int | None = None):
        """One epoch of rollouts; returns (messages, meta) like the reference.
        group_base: first group id (default: the reference's
        (epoch * nodes + node) * groups_per_epoch)."""
        import torch

        from .rollout import sample_action_tokens
        cfg, dev = self.cfg, self.device
        V, H, G, C, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.chunks, cfg.tokens
        n_traj = cfg.n_groups * G
        R = n_traj * C * T
        t0 = time.perf_counter()
        pool = self.env_pools[epoch % len(self.env_pools)]
        pool.epoch_reset()  # its previous epoch was consumed (staleness gate)

        def stage(shape, dtype):
            n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
            return pool.view(pool.alloc(n, align=256), dtype).view(*shape)

        with (self.torch_arena or contextlib.nullcontext()), torch.cuda.stream(self.stream):
            if getattr(snap, "ready", None) is not None:
                self.stream.wait_event(snap.ready)  # the snapshot's bytes landed
            W = snap.params.view(V, H)  # installed replica, zero copy
            # synthetic LIBERO-shaped observations -> features
            img = stage((n_traj * C, 224 * 224 * 3 // 64), torch.uint8)
            img.copy_(torch.randint(0, 256, img.shape, device=dev, generator=self.rng,
                                    dtype=torch.uint8))
            prop = torch.randn(n_traj * C, 8, device=dev, generator=self.rng)
            obs = torch.cat([img.float() / 255.0, prop], dim=1)
            feats = stage((n_traj * C, H), torch.bfloat16)
            feats.copy_(obs @ self.proj)                                # [n_traj*C, H]
            ftok = expand_token_features(feats, self.pos, stage((R, H), torch.bfloat16))
            logits = stage((R, V), torch.bfloat16)
            torch.matmul(ftok, W.t(), out=logits)
            rewards = torch.randint(0, 2, (n_traj,), device=dev, generator=self.rng).float()
            if poison:
                rewards[0] = float("nan")
            # action tokens ~ softmax(logits) + f32 behaviour log-probs in
            # one pass (csrc/sample.cu), Philox keyed by (seed, epoch, row)
            tokens, blp, _ = sample_action_tokens(
                logits, T, seed=cfg.seed * 1_000_003 + self.node, offset=epoch)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        msgs = []
        base = (epoch * self.nodes + self.node) * cfg.n_groups if group_base is None else group_base
        for gi in range(cfg.n_groups):
            sl = slice(gi * G, (gi + 1) * G)
            toks = tokens.view(n_traj, C, T)[sl]
            b = GroupBatch(
                group_id=base + gi, horizon=C * T, chunk=T,
                obs=feats.view(n_traj, C, H)[sl], actions=toks,
                behavior_log_prob=blp.view(n_traj, C)[sl],
                rewards=rewards[sl], behavior_version=snap.version, tokens=toks)
            b.ready = ev  # device-resident handoff: consumer waits on the event
            msgs.append(b)
        ev.synchronize()
        meta = {"roll_wall": time.perf_counter() - t0, "epoch": epoch,
                "behavior_version": snap.version,
                "success_rate": float(rewards.float().mean().item()) if not poison else 0.0,
                # the whole epoch as one message (cross-process hand-off)
                "epoch_batch": GroupBatch(
                    group_id=base, horizon=C * T, chunk=T, obs=feats.view(n_traj, C, H),
                    actions=tokens.view(n_traj, C, T), behavior_log_prob=blp.view(n_traj, C),
                    rewards=rewards, behavior_version=snap.version, tokens=None)}
        return msgs, meta


class TrainerWorker:
    """One per GPU: owns the head parameters and Adam state (MODEL_COMPUTE
    pool), the fused loss and the TRAINER stream (reference
    runtime.py:732-800).

    update() enqueues the whole learner step on the trainer stream and
    synchronises once at its end:
      per-token features -> logits GEMM (cuBLAS, bf16 weights kept by the
      optimizer tail) -> fused token loss fwd+bwd (csrc/token_loss.cu) ->
      skip word (loss abort) -> head gradient dW = dl^T feats as f32 GEMM
      output -> with N learners: ZeRO-1, the gradient's row blocks
      reduce-scattered together with every rank's skip word (so one rank's
      abort skips the step on every rank) -- by copy-engine pushes over
      NVLink as the blocks complete (exchange.PeerGradExchange) or NCCL --
      this rank's block stepped, the bf16 blocks all-gathered (pushed chunk
      by chunk behind the optimizer tail, or NCCL); with the switch-reduced
      / exact reducers: the
      mean of the whole gradient -> grad norm of the mean -> optimizer tail
      (clip, Adam, bf16 copy, non-finite flag; skipped on the device on
      abort or a non-finite gradient).  (GradReducer.reduce_async keeps a
      bucketed all-reduce available; overlapping it with the gradient GEMM
      measured slower.)
    Aborts surface after the one synchronisation: GrpoAbort (the caller
    quarantines; parameters and Adam state untouched) or RunAbort
    (non-finite parameters)."""

    def __init__(self, cfg: SwimlaneConfig, node: int, model_pool, reducer, stream, device,
                 act_pool=None, n_groups: int | None = None, torch_arena=None):
        import torch

        from . import _lib
        from .pools import Pool, PoolKind
        self.cfg, self.node, self.reducer = cfg, node, reducer
        self.stream, self.device = stream, device
        V, H, G, C, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.chunks, cfg.tokens
        nodes = reducer.nodes
        # ZeRO-1 over the learner GPUs when the gradient travels as NCCL f32
        # sums: reduce-scatter the gradient, step this rank's row block,
        # all-gather the bf16 weights (less traffic than all-reduce, and the
        # optimizer tail runs on 1/N of the parameters)
        self.sharded = nodes > 1 and reducer.backend == "nccl" and not reducer.exact
        if self.sharded:
            import torch.distributed as dist
            shard = (dist.get_rank(reducer.group), nodes)
        else:
            shard = None
        self.reducer_rank = shard[0] if shard else 0
        self.policy = TokenPolicy(cfg, model_pool, device, shard=shard)
        self.gcfg = GrpoConfig(group_size=cfg.group_size, lr=cfg.lr,
                               max_grad_norm=cfg.max_grad_norm)
        self.n_groups = cfg.n_groups if n_groups is None else int(n_groups)
        R = self.n_groups * G * C * T
        n = V * H
        self.loss = TokenLoss(self.n_groups, G, C, T, V, self.gcfg, dtype=torch.bfloat16,
                              device=device)
        if self.sharded:
            # reduce-scatter input: the gradient's N*Vs rows contiguous (rank j's
            # block = rows [j Vs, (j+1) Vs); rows past V stay zero), so a GEMM
            # can cover several owners' blocks at once; output: this rank's
            # block.  The skip words (loss aborts) travel with the block sums
            # of squares: scal = [sum of squares, skip] summed over the ranks.
            Vs = self.policy.Vs
            self.cs = Vs * H
            self.hg = model_pool.alloc(nodes * self.cs * 4 + self.cs * 4, align=256)
            allg = model_pool.view(self.hg, torch.float32)[: (nodes + 1) * self.cs]
            allg.zero_()
            self.gin = allg[: nodes * self.cs]
            self.gshard = allg[nodes * self.cs:]
            self.grad2d = None
            self.scal = torch.zeros(2, dtype=torch.float64, device=device)
            self.sumsq = self.scal[0:1]
            self.skip = torch.zeros(1, dtype=torch.float32, device=device)
            self._own_skip = torch.zeros(1, dtype=torch.float32, device=device)
            self.status_out = self._own_skip
            self.exchange = None
            if reducer.peer_scatter():
                from ._lib import NativeError
                from .exchange import PeerGradExchange
                try:
                    self.exchange = PeerGradExchange(self.gin.view(nodes, self.cs), model_pool,
                                                     group=reducer.group,
                                                     wbuf=self.policy.w16pad)
                except NativeError as e:   # raised on every rank alike: NCCL together
                    log.warning("peer gradient exchange unavailable (%s); NCCL collectives", e)
                    reducer.scatter = "nccl"
            if self.exchange is not None:
                # the bf16 all-gather: "kernel" = the optimizer tail stores its
                # rows into the peers' working copies itself; "ce" = copy-engine
                # pushes of each optimizer-tail chunk while the next is stepped
                self.gather_mode = os.environ.get("DVLA_GATHER_MODE", "kernel")
                self.gather_chunks = int(os.environ.get("DVLA_GATHER_CHUNKS", "4"))
                self._peer_rows = self.exchange.peer_rows(0)
        else:
            # f32 gradient + the skip word (one all-reduce buffer), long-lived
            self.hg = model_pool.alloc((n + 1) * 4, align=256)
            self.gbuf = model_pool.view(self.hg, torch.float32)[: n + 1]
            self.grad2d = self.gbuf[:n].view(V, H)
            self.skip = self.gbuf[n:n + 1]
            self.status_out = self.skip
        # activations of one update (logits, d loss / d logits, per-token
        # features): an activation pool of the recycled kind, reset per update
        act_bytes = R * (2 * V * 2 + H * 2) + (4 << 20)
        self.act_pool = act_pool or Pool(PoolKind.ENV_AUX, act_bytes, device=device)
        self._acts(R, V, H)
        # GEMMs per owner block of the head gradient (DVLA_GRAD_SUB; DESIGN §6:
        # at 4 learners two per block measured 0.15 ms faster, at 2 one)
        self.grad_sub = max(1, int(os.environ.get("DVLA_GRAD_SUB", "1")))
        self.grad_plan = os.environ.get("DVLA_GRAD_PLAN", "halves")
        self.pos = token_positions(cfg, device)
        self.norm_ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8,
                                   device=device)
        self.norm = torch.zeros(1, dtype=torch.float64, device=device)
        # grad / param non-finite, peer-exchange timeout (max-reduced over learners)
        self.flags = torch.zeros(3, dtype=torch.int32, device=device)
        if getattr(self, "exchange", None) is not None:
            self.exchange.err = self.flags[2:3]
        self.h_stats = torch.empty(_lib.ST_LEN, dtype=torch.float64, pin_memory=True)
        self.h_misc = torch.empty(2, dtype=torch.float64, pin_memory=True)  # norm, skip
        self.h_flags = torch.empty(3, dtype=torch.int32, pin_memory=True)
        self.h_skip = torch.empty(1, dtype=torch.float32, pin_memory=True)
        self.h_rw = None
        self.version = 0
        self.done_event = None
        self.timing = None  # optional: dict of CUDA event pairs per phase
        self.torch_arena = torch_arena
        # the initial weights / moments were written on the default stream,
        # which the worker's non-blocking streams do not order against
        torch.cuda.synchronize(device)

    def close(self):
        """Release the peer exchange's IPC mappings (collective with the
        other learners when sharded)."""
        ex = getattr(self, "exchange", None)
        if ex is not None:
            ex.close()
            self.exchange = None

    def _acts(self, R, V, H):
        import torch
        pool = self.act_pool
        pool.epoch_reset()
        self.logits = pool.view(pool.alloc(R * V * 2, align=256), torch.bfloat16).view(R, V)
        self.dl = pool.view(pool.alloc(R * V * 2, align=256), torch.bfloat16).view(R, V)
        self.feats_tok = pool.view(pool.alloc(R * H * 2, align=256), torch.bfloat16).view(R, H)

    def snapshot(self, out=None, stream=None) -> ParamSnapshot:
        """The bf16 head as a versioned device snapshot (fused copy +
        first-non-finite scan; reference snapshot_from_params)."""
        from .replicate import device_snapshot
        return device_snapshot(self.policy.weight_bf16().reshape(-1), self.version, out=out,
                               stream=stream)

    def _grad_tail(self, s, ev_t, mx):
        """One GPU (or the switch-reduced / exact reducers): dW = dl^T x as
        f32 GEMM output, the mean over nodes, norm, optimizer tail."""
        from . import _lib
        torch = __import__("torch")
        pol, nodes = self.policy, self.reducer.nodes
        V, H = pol.V, pol.H
        n = V * H
        torch.mm(self.dl.t(), self.feats_tok, out_dtype=torch.float32, out=self.grad2d)
        if ev_t is not None:
            ev_t["grad1"].record(s)
        if nodes > 1:  # switch-reduced / exact paths: the mean itself
            self.gbuf.copy_(self.reducer.reduce(self.gbuf))
        if ev_t is not None:
            ev_t["reduce1"].record(s)
        g = self.gcfg
        _lib.check(_lib.dvla_grad_norm_f32(self.gbuf.data_ptr(), n, 1.0, self.norm.data_ptr(),
                                           self.flags.data_ptr(), self.norm_ws.data_ptr(),
                                           s.cuda_stream), "dvla_grad_norm_f32")
        if ev_t is not None and "norm1" in ev_t:
            ev_t["norm1"].record(s)
        _lib.check(_lib.dvla_adam_tail_f32(
            pol.master.data_ptr(), self.gbuf.data_ptr(), pol.m.data_ptr(), pol.v.data_ptr(),
            n, pol.step + 1, g.lr, g.beta1, g.beta2, g.opt_eps, 1.0, self.norm.data_ptr(), mx,
            self.skip.data_ptr(), pol.w16.data_ptr(), self.flags.data_ptr() + 4,
            s.cuda_stream), "dvla_adam_tail_f32")
        if ev_t is not None and "adam1" in ev_t:
            ev_t["adam1"].record(s)

    def _grad_rows(self, a: int, b: int):
        """Rows [a, b) of dW = dl^T x (f32 GEMM output into the contiguous
        reduce-scatter input), as `grad_sub` row-split GEMMs."""
        import torch
        b = min(b, self.policy.V)
        if a >= b:
            return
        H = self.policy.H
        rows = self.gin.view(-1, H)
        step = max(128, (-(-(b - a) // self.grad_sub) + 127) // 128 * 128)
        for a2 in range(a, b, step):
            b2 = min(b, a2 + step)
            torch.mm(self.dl[:, a2:b2].t(), self.feats_tok, out_dtype=torch.float32,
                     out=rows[a2:b2])

    def _grad_segments(self):
        """The head-gradient GEMMs of this rank under ZeRO-1, in issue order,
        as (first row, end row, peer blocks complete after this GEMM); every
        peer block a GEMM completes is pushed right after it, and the last
        GEMM (part or all of the own block) hides the last pushes.
          "halves" (default): the owner blocks in two halves, each ~V/2 rows
            (a single owner block of V/N rows is a less efficient GEMM shape
            on B200 at 4 learners: DESIGN.md §6) -- the other half first;
            then, when the own block sits at an end of its half, the half
            minus the own block's outer half as one GEMM (its peer blocks
            pushed under the next one) and that outer half last;
          "halves1": the same with the own half as one GEMM (its peer blocks
            pushed after it, exposed);
          "runs": the peers' blocks as the (at most two) contiguous runs
            around the own block, larger first, then the own block alone."""
        N, r = self.reducer.nodes, self.reducer_rank
        Vs = self.policy.Vs
        plan = self.grad_plan
        if plan in ("halves", "halves1") and N > 2:
            h = N // 2
            halves = [(0, h), (h, N)]
            own = 0 if r < h else 1
            oa, ob = halves[1 - own]
            segs = [(oa * Vs, ob * Vs, list(range(oa, ob)))]
            ha, hb = halves[own]
            mates = [j for j in range(ha, hb) if j != r]
            cut = (Vs // 2 + 127) // 128 * 128      # the own block's outer part
            if plan == "halves" and mates and r in (ha, hb - 1) and 0 < cut < Vs:
                if r == ha:   # own block first in its half: its lower rows last
                    segs += [(r * Vs + cut, hb * Vs, mates), (r * Vs, r * Vs + cut, [])]
                else:         # own block last in its half: its upper rows last
                    segs += [(ha * Vs, r * Vs + Vs - cut, mates),
                             (r * Vs + Vs - cut, (r + 1) * Vs, [])]
            else:
                segs += [(ha * Vs, hb * Vs, mates)]
            return segs
        runs = [(r + 1, N), (0, r)]
        runs = sorted([x for x in runs if x[1] > x[0]], key=lambda x: x[0] - x[1])
        return ([(a * Vs, b * Vs, list(range(a, b))) for a, b in runs]
                + [(r * Vs, (r + 1) * Vs, [])])

    def _grad_tail_sharded(self, s, ev_t, mx):
        """N learner GPUs, ZeRO-1 (reference runtime.py:788-796 arithmetic):
        dW row blocks as f32 GEMM outputs straight into the reduce-scatter
        input -> reduce-scatter (sum): copy-engine pushes over NVLink as the
        blocks complete + a node-order f64 sum (exchange.PeerGradExchange),
        or NCCL reduce_scatter -> this rank's block / N -> global
        norm (block sums of squares summed over the ranks together with the
        skip words: in rank order over NVLink with the exchange, else NCCL)
        -> optimizer tail on the block (skipped on every rank when any
        rank's loss aborted) -> all-gather of the bf16 blocks (stored into
        the peers by the optimizer-tail kernel itself, or pushed per
        optimizer chunk by the copy engines, or NCCL) -> non-finite / timeout flags
        max-reduced (over NVLink with the exchange, else NCCL).  With the
        exchange the step makes no collective-library call."""
        import torch
        import torch.distributed as dist

        from . import _lib
        pol, nodes, grp = self.policy, self.reducer.nodes, self.reducer.group
        Vs = pol.Vs
        nloc = Vs * pol.H
        ex = self.exchange
        div = float(nodes)

        if ex is not None:
            # the GEMMs of _grad_segments (own block last); each finished peer
            # block pushed by a copy engine while the next GEMM runs; then the
            # node-order sum + this block's sum of squares in one pass
            ex.begin(s)
            for ra, rb, done in self._grad_segments():
                self._grad_rows(ra, rb)
                for j in done:
                    ex.pushed(j, s)
            if ev_t is not None:
                ev_t["grad1"].record(s)
            ex.finish(s, self.gshard, nloc, div, self.sumsq, self.flags, self.norm_ws)
        else:
            self._grad_rows(0, nodes * Vs)     # one GEMM: the rows are contiguous
            if ev_t is not None:
                ev_t["grad1"].record(s)
            dist.reduce_scatter_tensor(self.gshard, self.gin, op=dist.ReduceOp.SUM, group=grp)
            _lib.check(_lib.dvla_grad_sumsq_f32(self.gshard.data_ptr(), nloc, div,
                                                self.sumsq.data_ptr(), self.flags.data_ptr(),
                                                self.norm_ws.data_ptr(), s.cuda_stream),
                       "dvla_grad_sumsq_f32")
        if ev_t is not None:
            ev_t["reduce1"].record(s)
        g = self.gcfg
        # [sum of squares, skip] summed over the ranks: the global norm and
        # the number of ranks whose loss aborted (any -> the step is skipped
        # on every rank)
        self.scal[1:2].copy_(self._own_skip)
        if ex is not None:   # rank order, over NVLink
            ex.reduce_sum_f64(self.scal, s)
        else:
            dist.all_reduce(self.scal, op=dist.ReduceOp.SUM, group=grp)
        self.skip.copy_(self.scal[1:2])
        torch.sqrt(self.sumsq, out=self.norm)
        if ev_t is not None and "norm1" in ev_t:
            ev_t["norm1"].record(s)

        def adam(lo, hi):
            _lib.check(_lib.dvla_adam_tail_f32(
                pol.master.data_ptr() + 4 * lo, self.gshard.data_ptr() + 4 * lo,
                pol.m.data_ptr() + 8 * lo, pol.v.data_ptr() + 8 * lo, hi - lo, pol.step + 1,
                g.lr, g.beta1, g.beta2, g.opt_eps, div, self.norm.data_ptr(), mx,
                self.skip.data_ptr(), pol.w16_own.data_ptr() + 2 * lo, self.flags.data_ptr() + 4,
                s.cuda_stream), "dvla_adam_tail_f32")

        if ex is not None and ex.wbuf is not None and self.gather_mode == "kernel":
            # the all-gather inside the optimizer tail: its bf16 rows stored
            # into every peer's working copy by the same kernel
            _lib.check(_lib.dvla_adam_tail_f32_bcast(
                pol.master.data_ptr(), self.gshard.data_ptr(), pol.m.data_ptr(),
                pol.v.data_ptr(), nloc, pol.step + 1, g.lr, g.beta1, g.beta2, g.opt_eps, div,
                self.norm.data_ptr(), mx, self.skip.data_ptr(), pol.w16_own.data_ptr(),
                self._peer_rows, nodes - 1, self.flags.data_ptr() + 4, s.cuda_stream),
                "dvla_adam_tail_f32_bcast")
            if ev_t is not None and "adam1" in ev_t:
                ev_t["adam1"].record(s)
            ex.gather_finish(s, by_kernel=True)
        elif ex is not None and ex.wbuf is not None:
            # the all-gather as copy-engine pushes of each stepped chunk
            k = max(1, self.gather_chunks)
            step = max(64, (-(-nloc // k) + 63) // 64 * 64)   # 64-element aligned chunks
            for lo in range(0, nloc, step):
                hi = min(nloc, lo + step)
                adam(lo, hi)
                ex.gather_chunk(lo, hi, s)
            if ev_t is not None and "adam1" in ev_t:
                ev_t["adam1"].record(s)
            ex.gather_finish(s)
        else:
            adam(0, nloc)
            if ev_t is not None and "adam1" in ev_t:
                ev_t["adam1"].record(s)
            dist.all_gather_into_tensor(pol.w16pad, pol.w16_own, group=grp)
        if ex is not None:   # abort / non-finite / timeout words, max over the learners
            ex.reduce_max_u32(self.flags, s)
        else:
            dist.all_reduce(self.flags, op=dist.ReduceOp.MAX, group=grp)

    def update(self, batches: list, transport_nodes: int | None = None) -> dict:
        """One GRPO update on one epoch of groups (reference runtime.py:768-800).
        transport_nodes: the reference's argument; the node count here is
        the reducer's (GradReducer.nodes)."""
        import torch

        from . import _lib
        from .grpo import stats_from_vector
        cfg, pol, s = self.cfg, self.policy, self.stream
        H = cfg.hidden
        t0 = time.perf_counter()
        ids = [b.group_id for b in batches]
        if len(batches) != self.n_groups:
            raise ConfigError(f"update expects {self.n_groups} groups, got {len(batches)}")
        ev_t = self.timing
        with (self.torch_arena or contextlib.nullcontext()), torch.cuda.stream(s):
            seen = set()
            for b in batches:
                ev = getattr(b, "ready", None)
                if ev is not None and id(ev) not in seen:
                    seen.add(id(ev))
                    s.wait_event(ev)
            if ev_t is not None:
                ev_t["start"].record(s)
            feats = torch.cat([b.obs.reshape(-1, H) for b in batches])       # [n_traj*C, H]
            expand_token_features(feats, self.pos, self.feats_tok)
            torch.mm(self.feats_tok, pol.w16.t(), out=self.logits)
            self.loss.set_groups(ids)
            toks = torch.cat([b.actions.reshape(-1) for b in batches])
            blp = torch.cat([b.behavior_log_prob.reshape(-1) for b in batches])
            rw = torch.cat([b.rewards.reshape(-1) for b in batches])
            if self.h_rw is None or self.h_rw.dtype != rw.dtype or self.h_rw.shape != rw.shape:
                self.h_rw = torch.empty(rw.shape, dtype=rw.dtype, pin_memory=True)
            self.h_rw.copy_(rw, non_blocking=True)   # mean_reward, read after the sync
            if ev_t is not None:
                ev_t["loss0"].record(s)
            self.loss.launch(self.logits, toks, blp, rw, self.dl, stream=s)
            if ev_t is not None:
                ev_t["loss1"].record(s)
            _lib.check(_lib.dvla_loss_status(self.loss.stats_dev.data_ptr(),
                                             self.status_out.data_ptr(), s.cuda_stream),
                       "dvla_loss_status")
            self.flags.zero_()
            g = self.gcfg
            mx = float(g.max_grad_norm) if g.max_grad_norm is not None else 0.0
            if self.sharded:
                self._grad_tail_sharded(s, ev_t, mx)
            else:
                self._grad_tail(s, ev_t, mx)
            if ev_t is not None:
                ev_t["end"].record(s)
            self.h_stats.copy_(self.loss.stats_dev, non_blocking=True)
            self.h_misc[:1].copy_(self.norm, non_blocking=True)
            self.h_flags.copy_(self.flags, non_blocking=True)
            self.h_skip.copy_(self.skip, non_blocking=True)
        done = torch.cuda.Event()
        done.record(s)
        t_enq = time.perf_counter()
        done.synchronize()   # the update's one host synchronisation
        if ev_t is not None:
            ev_t["host_enqueue_s"] = t_enq - t0
            ev_t["host_wait_s"] = time.perf_counter() - t_enq
        hf = self.h_flags.numpy()
        if hf[2]:
            raise RunAbort("peer gradient exchange timed out (a learner stopped arriving)",
                           lane=LaneId.TRAINER.value, epoch=self.version)
        sv = self.h_stats.numpy().copy()
        skipped = float(self.h_skip.numpy()[0]) != 0.0
        grad_bad = bool(hf[0])
        norm = float(self.h_misc.numpy()[0])
        if skipped or grad_bad or not np.isfinite(norm):
            # the device skipped the step: parameters and moments untouched
            # (loss abort / non-finite loss on any rank, or a non-finite
            # gradient: reference grpo.py:237-283 -> quarantine)
            stats_from_vector(sv, self.loss.group_ids, self.loss.order,
                              self.n_groups * cfg.group_size)          # local abort -> raises
            if skipped:
                raise GrpoAbort(int(ids[0]), "a peer learner's batch aborted the update")
            raise GrpoAbort(int(ids[0]), "non-finite loss or gradient")
        rw_h = self.h_rw.numpy().reshape(self.n_groups, cfg.group_size)
        stats = stats_from_vector(sv, self.loss.group_ids, self.loss.order,
                                  self.n_groups * cfg.group_size, rw_h)
        if hf[1]:
            raise RunAbort("non-finite parameters after update",
                           lane=LaneId.TRAINER.value, epoch=self.version)
        pol.step += 1
        self.version += 1
        self.done_event = done
        return {"version": self.version, "loss": stats["loss"], "grad_norm": norm,
                "train_wall": time.perf_counter() - t0, "mean_ratio": stats["mean_ratio"],
                "clip_fraction": stats["clip_fraction"], "n_chunks": stats["n_chunks"],
                "mean_reward": stats["mean_reward"]}


class RunResult:
    def __init__(self):
        self.reports: list = []
        self.update_stats: list = []
        self.counters: dict = {}
        self.staleness_max = 0
        self.wall = 0.0
        self.lane_busy: dict = {}

    def summary(self) -> dict:
        """Throughput between the first and the last published update (wall
        clock), i.e. after the pipeline filled; the reference's per-epoch
        step-time sum (metrics.py:101-123) is reported beside it."""
        post = self.reports[1:] if len(self.reports) > 1 else self.reports
        trans = sum(r["transitions"] for r in post)
        traj = sum(r["trajectories"] for r in post)
        span = sum(r["step_time"] for r in post)
        pubs = [r["t_publish"] for r in self.reports]
        wall = (pubs[-1] - pubs[0]) if len(pubs) > 1 else max(self.wall, 1e-12)
        n = max(len(post), 1)
        return {"transitions_per_s": trans / max(wall, 1e-12),
                "rollout_time": sum(r.get("roll_wall", 0.0) for r in post) / n,
                "actor_time": sum(r.get("train_wall", 0.0) for r in post) / n,
                "trajectories_per_s": traj / max(wall, 1e-12),
                "transitions_per_s_steptime": trans / max(span, 1e-12),
                "wall": self.wall, "staleness_max": self.staleness_max,
                "updates": len(self.update_stats)}


@dataclass
class BubbleStats:
    sampler_idle_fraction: float
    trainer_idle_fraction: float
    wall: float
    warmup_dominated: bool


def barrier_free_handoff_audit(result: RunResult) -> BubbleStats:
    """Idle fraction of each lane over the run's wall clock (reference
    runtime.py:881-889): the bubbles the asynchronous handoff leaves."""
    wall = max(result.wall, 1e-12)
    return BubbleStats(
        sampler_idle_fraction=max(0.0, 1.0 - result.lane_busy.get("sampler", 0.0) / wall),
        trainer_idle_fraction=max(0.0, 1.0 - result.lane_busy.get("trainer", 0.0) / wall),
        wall=wall, warmup_dominated=len(result.reports) <= 1)


def run_swimlane(cfg: SwimlaneConfig, device=None, group=None, poison_epochs=frozenset()):
    """Asynchronous swimlane on one GPU (and, under torch.distributed, one
    closed loop per GPU with NCCL gradient reduction: topology replication,
    reference placement.py:197-205)."""
    import torch
    import torch.distributed as dist

    from .planes import Channel, ControlPlane, Plane, RunAborted, Transport, TransportMode
    from .pools import Pool, PoolKind
    from .replicate import device_snapshot

    cfg.validate()
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    torch.cuda.set_device(dev)
    nodes = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    V, H, G, C, T = cfg.vocab, cfg.hidden, cfg.group_size, cfg.chunks, cfg.tokens
    n_traj = cfg.n_groups * G
    R = n_traj * C * T

    # ---- dual pools: long-lived model state vs epoch-recycled rollout staging
    nbuf = cfg.staleness_limit + 2   # published-weight ring (see VersionBoard.retire)
    n = V * H
    model_bytes = n * (4 + 8 + 8 + 2) + (n + 1) * 4 + nbuf * n * 2 + (64 << 20)
    model_pool = Pool(PoolKind.MODEL_COMPUTE, model_bytes, device=dev)
    # ENV_AUX: one epoch-recycled arena per epoch the staleness gate lets be in
    # flight (limit + 2); each is reset wholesale when its epoch starts again
    env_bytes = R * (V * 2 + H * 2 + 64) + n_traj * C * (H * 2 + 224 * 224 * 3 // 64 * 5) + \
        (16 << 20)
    env_pools = [Pool(PoolKind.ENV_AUX, env_bytes, device=dev)
                 for _ in range(cfg.staleness_limit + 2)]
    abort = threading.Event()
    monitor = Monitor(abort)

    # the trainer stream (loss, gradient GEMM, all-reduce hand-off, optimizer
    # and snapshot) runs at high priority: its CTAs are scheduled ahead of the
    # sampler's GEMM CTAs whenever both have work pending
    s_train = torch.cuda.Stream(device=dev, priority=-1)
    s_sample, s_dist = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ctrl = ControlPlane(Transport(TransportMode.INPROC, Plane.CONTROL, name="ctrl"))
    mailbox = ctrl.subscribe("weights", abort_event=abort)
    chan = Channel(cfg.queue_capacity * cfg.n_groups,
                   Transport(TransportMode.INPROC, Plane.DATA, name="data"), abort_event=abort)
    reducer = GradReducer(nodes, group)
    tarena = None
    if cfg.torch_pool_bytes > 0:
        from .pools import TorchArena
        tarena = TorchArena.shared(dev, cfg.torch_pool_bytes)
    trainer = TrainerWorker(cfg, rank, model_pool, reducer, s_train, dev, torch_arena=tarena)
    sampler = SamplerWorker(cfg, rank, nodes, env_pools, s_sample, dev, torch_arena=tarena)
    # ring of published weights (bf16) in the MODEL_COMPUTE pool
    wbuf = [model_pool.view(model_pool.alloc(n * 2, align=256), torch.bfloat16)
            for _ in range(nbuf)]
    snap0 = trainer.snapshot(out=wbuf[0])
    board = VersionBoard(cfg.staleness_limit, monitor, snap0)
    result = RunResult()
    busy = {"sampler": 0.0, "trainer": 0.0}
    dist_q: list = []
    dist_cv = threading.Condition()

    def sampler_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            for epoch in range(cfg.epochs):
                snap, stal = board.wait_gate()
                monitor.beat(LaneId.SAMPLER.value, "rolling")
                msgs, meta = sampler.run_epoch(epoch, snap, poison=epoch in poison_epochs)
                busy["sampler"] += meta["roll_wall"]
                board.produce(epoch, {**meta, "staleness": stal})
                for m in msgs:
                    chan.put(m)
                board.boundary()
            board.mark_sampler_done()
            monitor.beat(LaneId.SAMPLER.value, "done")
        except RunAborted:
            pass
        except Exception as e:  # surface the failure through the watchdog
            monitor.fail(f"sampler: {e!r}", LaneId.SAMPLER.value, -1)

    def trainer_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            for epoch in range(cfg.epochs):
                batches = [chan.take() for _ in range(cfg.n_groups)]
                meta = board.take_meta(epoch)
                monitor.beat(LaneId.TRAINER.value, "train")
                t0 = time.perf_counter()
                try:
                    st = trainer.update(batches)
                except GrpoAbort as e:
                    log.warning("quarantined update: %s", e)
                    board.quarantine()
                    result.counters["quarantined_updates"] = \
                        result.counters.get("quarantined_updates", 0) + 1
                    continue
                board.wait_pacing(board.version + 1)
                nv = trainer.version
                board.retire(nv - nbuf)   # the ring slot nv % nbuf is free again
                # the published copy is taken on the trainer stream, so the
                # next update's optimizer step cannot overlap it (the bytes
                # are already verified finite by the optimizer tail)
                snap = device_snapshot(trainer.policy.weight_bf16().reshape(-1), nv,
                                       out=wbuf[nv % nbuf], stream=s_train, verified=True)
                v = board.publish()
                busy["trainer"] += time.perf_counter() - t0
                result.update_stats.append({"version": v, **{k: st[k] for k in (
                    "loss", "mean_ratio", "clip_fraction", "n_chunks", "grad_norm")}})
                with dist_cv:
                    dist_q.append((v, snap))
                    dist_cv.notify_all()
                step_time = max(meta["roll_wall"], time.perf_counter() - t0)
                result.reports.append({"epoch": epoch, "policy_version": meta["behavior_version"],
                                       "version_after": v, "step_time": step_time,
                                       "transitions": n_traj * C * T,
                                       "trajectories": n_traj, "staleness": meta["staleness"],
                                       "roll_wall": meta["roll_wall"],
                                       "train_wall": st["train_wall"],
                                       "t_publish": time.perf_counter()})
            with dist_cv:
                dist_q.append((None, None))
                dist_cv.notify_all()
            monitor.beat(LaneId.TRAINER.value, "done")
        except RunAborted:
            pass
        except Exception as e:
            monitor.fail(f"trainer: {e!r}", LaneId.TRAINER.value, -1)

    def dist_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            while True:
                with dist_cv:
                    while not dist_q:
                        if abort.is_set():
                            return
                        dist_cv.wait(0.05)
                    v, snap = dist_q.pop(0)
                if v is None:
                    break
                ctrl.broadcast(snap, stream=s_dist)  # INPROC: hand-off; ready event rides along
                monitor.beat(LaneId.WEIGHT_DIST.value)
            monitor.beat(LaneId.WEIGHT_DIST.value, "done")
        except RunAborted:
            pass
        except Exception as e:
            monitor.fail(f"dist: {e!r}", LaneId.WEIGHT_DIST.value, -1)

    def recv_lane():
        torch.cuda.set_device(dev)   # the current device is per host thread
        try:
            while not (board.sampler_done and mailbox._slot is None):
                snap = mailbox.take_newest(timeout=0.2)
                if snap is not None:
                    board.deposit(snap)
                    monitor.beat(LaneId.WEIGHT_RECV.value)
            monitor.beat(LaneId.WEIGHT_RECV.value, "done")
        except RunAborted:
            pass

    t_start = time.perf_counter()
    lanes = [threading.Thread(target=f, name=n, daemon=True) for f, n in (
        (sampler_lane, "sampler"), (recv_lane, "recv"), (trainer_lane, "trainer"),
        (dist_lane, "dist"))]
    for t in lanes:
        t.start()
    try:
        while any(t.is_alive() for t in lanes):
            time.sleep(0.05)
            stale = monitor.stale_lanes(cfg.watchdog_s)
            if stale:
                monitor.fail(f"watchdog: lanes silent for > {cfg.watchdog_s}s", stale[0], -1)
            if abort.is_set():
                for t in lanes:
                    t.join(timeout=2.0)
                raise RunAbort(monitor.abort_reason or "aborted", lane=monitor.abort_lane,
                               epoch=monitor.abort_epoch, lane_states=monitor.dump())
    finally:
        # the learners' peer-memory mappings (a later run may be handed the
        # same peer allocations: an open mapping would collide)
        trainer.close()
    torch.cuda.synchronize(dev)
    result.wall = time.perf_counter() - t_start
    result.staleness_max = board.staleness_max
    result.lane_busy = busy
    result.policy = trainer.policy   # final weights (multi-GPU: identical on every rank)
    if tarena is not None:
        st = tarena.pool.stats()
        result.counters["torch_arena"] = {"capacity": tarena.pool.capacity,
                                          "segments_allocated": st.alloc_count,
                                          "live_bytes": st.live_bytes}
    result.counters.update({"updates": board.version, "produced": board.produced,
                            "regressions_ignored": board.regressions_ignored})
    return result


_ = (math, field)
