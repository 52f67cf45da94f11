#!/usr/bin/env python
"""bench.py -- D-VLA data-plane hot path on B200.

Metric (BASELINE.json): "RL samples/sec; weight-replication GB/s vs NVLink
peak at 1/2/4/8 B200".  A step is one pass of the learner hot path over one
GRPO batch of BASELINE config 2 (OpenVLA-7B-shaped action-token head: 512
trajectories = 64 groups x G=8, C=1 chunk x T=56 action tokens, V=32,064,
bf16 logits): fused log-softmax gather + clipped-ratio / group-normalised
advantage loss + d loss/d logits (csrc/token_loss.cu).  RL samples are
trajectories (one GRPO sample each); `value` = trajectories/s summed over
all ranks (weak scaling: every rank trains its own 512-trajectory shard).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank drives one GPU; timing is CUDA events on the
launching stream with barrier + synchronize on both sides, max over ranks.
Inputs (1.84 GB of logits per rank) exceed the 126 MB L2, so no flush is
needed between steps.  `--impl reference` times the CPU oracle port of the
same step on the host cores (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GROUPS, G, C, T, V = 64, 8, 1, 56, 32064
METRIC = "RL samples/sec; weight-replication GB/s vs NVLink peak at 1/2/4/8 B200"
UNIT = "samples/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--no-repl", action="store_true")
    ap.add_argument("--no-swimlane", action="store_true")
    ap.add_argument("--no-gauss", action="store_true")
    ap.add_argument("--no-f32", action="store_true", help="skip the C2 f32 leg")
    ap.add_argument("--fixed-warmup", action="store_true",
                    help="exactly --warmup warm-up steps (for ncu launch lists)")
    return ap.parse_args()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _nvlink_traffic():
    """NVLink bytes the chain kernel puts on the wire per replicated byte
    (ncu nvltx__bytes_data_user.sum of one 1 GiB hop, profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "nvlink_traffic.json")) as f:
            t = json.load(f)["replicate_chain_kernel"]
        return {"nvltx_user_bytes_per_byte": t["user_over_S"],
                "nvltx_bytes_per_byte_incl_protocol": t["nvltx_bytes"] / t["S"],
                "source": t["source"]}
    except Exception:  # noqa: BLE001
        return None


def _traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, watts = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                try:
                    watts.append(float(parts[3]))
                except ValueError:
                    pass
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if watts:
            out["power_w"] = statistics.median(watts)
        return out


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_inputs(n_groups: int):
    """Seeded synthetic inputs for the oracle port: n_groups x 8 trajectories."""
    import numpy as np
    rng = np.random.default_rng(0)
    x = rng.normal(0, 2, (n_groups, G, C, T, V)).astype(np.float32)
    tok = rng.integers(31744, 32000, (n_groups, G, C, T))
    blp = rng.normal(-600, 5, (n_groups, G, C)).astype(np.float32)
    rw = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
    return x, tok, blp, rw, np.arange(n_groups)


def _cpu_sample(threads: int, inputs, reps: int = 1):
    """Oracle port over `reps` passes of the prepared sample; returns
    (trajectories/s, seconds)."""
    from oracle import grpo_oracle as O
    x, tok, blp, rw, ids = inputs
    t0 = time.perf_counter()
    for _ in range(reps):
        O.grpo_token_grad(x, tok, blp, rw, ids, threads=threads)
    dt = time.perf_counter() - t0
    return reps * x.shape[0] * G / dt, dt


CPU_GROUPS = 16                      # one resident CPU sample: 16 groups x 8 traj (918 MB f32)


def run_reference(a):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    # each step: the full C2 batch (64 groups x 8 trajectories) as four passes
    # over one resident 16-group sample, so host memory stays bounded
    inputs = _cpu_inputs(CPU_GROUPS)
    reps = N_GROUPS // CPU_GROUPS
    for _ in range(max(1, min(a.warmup, 1))):
        _cpu_sample(threads, inputs, 1)
    times = []
    for _ in range(a.steps):
        _, dt = _cpu_sample(threads, inputs, reps)
        times.append(dt)
    value = a.steps * reps * CPU_GROUPS * G / sum(times)
    sample = (f"full C2 batch per step: {reps} passes x {CPU_GROUPS} groups x 8 traj x 56 tokens "
              f"x 32064 vocab (oracle numpy f64, rows split over all host threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * sum(times) / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 token-head GRPO loss fwd+bwd (OpenVLA-7B-shaped)",
                   "n_groups": N_GROUPS, "G": G, "C": C, "T": T, "V": V,
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)
    return 0


NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction (fallback)
_LIVE_NVL_PEAK = [None]   # this run's measured copy-engine peer copy (N >= 2)


def _nvl_peak():
    return _LIVE_NVL_PEAK[0] or NVLINK_PEER_GBS
NVLINK_NOMINAL_GBS = 900.0
REPL_BYTES = 6_600_000_000  # pi0-3B-shaped bf16 weights (BASELINE config 3)


def _bench_replication(world, rank, dev, barrier, max_over_ranks, iters=5):
    """Weight replication GB/s: chain broadcast of REPL_BYTES from rank 0 to
    every other rank (N >= 2), or into a co-located replica region (N = 1).
    Bit-exactness is verified on every receiver."""
    import torch
    from paper_2605_13276_b200 import _lib
    from paper_2605_13276_b200.replicate import ChainReplicator, LocalChain, bytes_equal
    S = REPL_BYTES
    gen = torch.Generator(device=dev).manual_seed(4242)
    src = torch.randint(0, 256, (S,), dtype=torch.uint8, device=dev, generator=gen)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"bytes": S, "iters": iters}
    if world == 1:
        ch = LocalChain(S, 1, device=dev, chunk_bytes=64 << 20, ctas_per_hop=148)
        ch.broadcast(src)
        torch.cuda.synchronize()
        ch.check()
        mism, _ = bytes_equal(src, ch.dsts[0])
        _lib.dvla_profile_enable(1)
        e0.record(stream)
        for _ in range(iters):
            ch.broadcast(src)
        e1.record(stream)
        torch.cuda.synchronize()
        kms, kn = _lib.profile_collect()
        _lib.dvla_profile_enable(0)
        ms = e0.elapsed_time(e1) / iters
        dst_ce = ch.dsts[0]
        e0.record(stream)
        for _ in range(iters):
            _lib.dvla_memcpy_async(dst_ce.data_ptr(), src.data_ptr(), S, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ce_ms = e0.elapsed_time(e1) / iters
        peak, _ = _peaks()
        out.update({"mode": "co-located replica (intra-HBM chain hop, TMA)",
                    "gbs": S / (ms / 1e3) / 1e9, "ms": ms,
                    "roofline": {"bound": "hbm", "achieved": 2 * S / (ms / 1e3) / 1e9,
                                 "peak": peak, "unit": "GB/s",
                                 "frac": 2 * S / (ms / 1e3) / 1e9 / peak,
                                 "note": "2 bytes moved per replicated byte"},
                    "ce_memcpy_gbs": S / (ce_ms / 1e3) / 1e9, "bit_exact": mism == 0,
                    "kernel_ms": kms / max(kn, 1)})
        del ch
        return out
    # receivers' replica regions live in their MODEL_COMPUTE pool (the static
    # half of the dual-pool allocator): the chain writes straight into it
    from paper_2605_13276_b200.pools import Pool, PoolKind
    pool = None if rank == 0 else Pool(PoolKind.MODEL_COMPUTE, 2 * S + (64 << 20), device=dev)
    rep = ChainReplicator(S, n_buffers=2, ctas_per_hop=128, pool=pool)
    rep_engine = rep.engine
    expect = src  # every rank generated the same bytes (same seed)
    rep.broadcast(src, 0)
    torch.cuda.synchronize()
    barrier()
    rep.check()
    ok = True if rank == 0 else bytes_equal(expect, rep.replica(0))[0] == 0
    times = []
    for it in range(1, iters + 1):
        barrier()
        e0.record(stream)
        rep.broadcast(src, it)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(max_over_ranks(e0.elapsed_time(e1)))
    rep.check()
    if rank != 0:
        ok = ok and bytes_equal(expect, rep.replica(iters))[0] == 0
    ok_all = max_over_ranks(0.0 if ok else 1.0) == 0.0
    ms = sorted(times)[len(times) // 2]
    # the NVLink peak of this box, measured live: copy-engine peer copy
    # rank 0 -> rank 1, 1 GiB, best of 10 (SURVEY §8(d) replication roofline)
    peak_ms = []
    for it in range(10):
        barrier()
        if rank == 0:
            e0.record(stream)
            _lib.check(_lib.dvla_memcpy_async(rep.fan_bufs[0], src.data_ptr(), 1 << 30,
                                              stream.cuda_stream), "dvla_memcpy_async")
            e1.record(stream)
        torch.cuda.synchronize()
        peak_ms.append(max_over_ranks(e0.elapsed_time(e1) if rank == 0 else 0.0))
    ce_peak = (1 << 30) / (min(peak_ms) / 1e3) / 1e9
    _LIVE_NVL_PEAK[0] = ce_peak
    # copy-engine fan-out baseline (root pushes to every receiver)
    ce = []
    for it in range(3):
        barrier()
        e0.record(stream)
        rep.ce_fanout(src, 0)
        e1.record(stream)
        torch.cuda.synchronize()
        ce.append(max_over_ranks(e0.elapsed_time(e1)))
    barrier()
    rep.close()
    del rep, pool
    gbs = S / (ms / 1e3) / 1e9
    engine = "copy-engine hop" if rep_engine == "ce" else "TMA chain"
    out.update({"mode": f"{engine} 0->{'->'.join(str(r) for r in range(1, world))}",
                "replica_regions": "receivers' MODEL_COMPUTE pools (dual-pool allocator)",
                "gbs": gbs, "ms": ms, "bit_exact": ok_all,
                "roofline": {"bound": "nvlink", "achieved": gbs, "peak": round(ce_peak, 1),
                             "unit": "GB/s", "frac": gbs / ce_peak,
                             "frac_of_nominal_900": gbs / NVLINK_NOMINAL_GBS,
                             "peak_source": "measured in this run: copy-engine peer copy "
                                            "rank 0 -> 1, 1 GiB, best of 10",
                             "traffic": _nvlink_traffic()},
                "ce_fanout_gbs_per_receiver": S / (sorted(ce)[1] / 1e3) / 1e9})
    out["multicast"] = _bench_multicast(S, src, rank, world, barrier, max_over_ranks)
    if world >= 4:
        try:
            out["c3_split"] = _bench_c3_split(S, src, rank, world, barrier, max_over_ranks)
        except Exception as e:  # noqa: BLE001 - a secondary leg never sinks the line
            out["c3_split"] = {"error": repr(e)[:300]}
    return out


def _bench_c3_split(S, src, rank, world, barrier, max_over_ranks, iters=4):
    """BASELINE config 3 layout: learners on ranks 0 and 1 each source half
    of the weight region to the replicas on ranks 2..N-1 (the two chains run
    the replicas in opposite orders), bit-exact on every replica."""
    import torch
    from paper_2605_13276_b200.replicate import SplitReplicator, bytes_equal
    reps = list(range(2, world))
    chains = [[0] + reps, [1] + reps[::-1]]
    rep = SplitReplicator(S, chains, n_buffers=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for it in range(iters + 1):
        barrier()
        e0.record()
        rep.broadcast(src if rank in (0, 1) else None, it)
        e1.record()
        torch.cuda.synchronize()
        t = max_over_ranks(e0.elapsed_time(e1))
        if it:
            times.append(t)
    rep.check()
    ok = rank < 2 or bytes_equal(src, rep.replica(0))[0] == 0
    ok_all = max_over_ranks(0.0 if ok else 1.0) == 0.0
    barrier()
    rep.close()
    ms = sorted(times)[len(times) // 2]
    return {"layout": f"learners 0,1 -> replicas {reps[0]}..{reps[-1]} (two half-region chains)",
            "gbs_per_replica": S / (ms / 1e3) / 1e9, "ms": ms, "bit_exact": ok_all,
            "frac_of_peer_copy": S / (ms / 1e3) / 1e9 / _nvl_peak()}


def _bench_multicast(S, src, rank, world, barrier, max_over_ranks, iters=4):
    """Switch-multicast (NVLS) broadcast of the same region, beside the
    chain: one source write per byte, replicated by the NVSwitch."""
    import torch
    from paper_2605_13276_b200.replicate import McReplicator, bytes_equal, multicast_supported
    ok_local = multicast_supported()
    if max_over_ranks(0.0 if ok_local else 1.0) != 0.0:
        return {"unavailable": "no NVSwitch multicast / POSIX-fd handles on this box"}
    from paper_2605_13276_b200._lib import NativeError
    try:
        rep = McReplicator(S, n_buffers=1)
    except NativeError as e:  # every rank raises the same error (agreement in setup)
        return {"unavailable": str(e)[:200]}
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for it in range(iters + 1):
        barrier()
        e0.record(stream)
        rep.broadcast(src, it)
        e1.record(stream)
        torch.cuda.synchronize()
        t = max_over_ranks(e0.elapsed_time(e1))
        if it:
            times.append(t)
    rep.check()
    ok = bytes_equal(src, rep.replica(iters))[0] == 0
    ok_all = max_over_ranks(0.0 if ok else 1.0) == 0.0
    barrier()
    rep.close()
    ms = sorted(times)[len(times) // 2]
    gbs = S / (ms / 1e3) / 1e9
    return {"mode": f"NVLS multicast 0->{{{','.join(str(r) for r in range(1, world))}}}",
            "gbs": gbs, "ms": ms, "bit_exact": ok_all,
            "frac_of_peer_copy": gbs / _nvl_peak()}


def _bench_gauss_c3(dev, rank, steps=200, cpu=True):
    """C3 (pi0-shaped) Gaussian-head learner step on this GPU: chunk_log_prob
    -> group advantages -> canonical-order epilogue -> head backward, B = 512
    chunks x D = 1,600 (SURVEY §8 d: ~10 MB, latency-bound: report time).
    Timed eagerly and as a captured CUDA graph; the f64 oracle port of the
    same step (single host thread, like the reference's numba backend)
    beside it on rank 0."""
    import numpy as np
    import torch
    from paper_2605_13276_b200 import _lib
    n_groups, G, C, D = 64, 8, 1, 1600
    B = n_groups * G * C
    g = torch.Generator(device=dev).manual_seed(0)
    means = torch.randn(B, D, device=dev, generator=g)
    actions = torch.randn(B, D, device=dev, generator=g)
    log_std = torch.randn(D, device=dev, generator=g) * 0.1
    lp0 = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    _lib.check(_lib.dvla_chunk_log_prob(means.data_ptr(), log_std.data_ptr(), actions.data_ptr(),
                                        B, D, lp0.data_ptr(), st.cuda_stream), "clp")
    blp = (lp0 + (torch.rand(B, dtype=torch.float64, device=dev, generator=g) - 0.5) * 0.1).float()
    rewards = torch.randint(0, 2, (n_groups * G,), device=dev, generator=g).float()
    ids = np.arange(n_groups, dtype=np.int64)
    order_d = torch.from_numpy(ids).to(dev)
    ids_d = order_d.clone()
    lp = torch.empty(B, dtype=torch.float64, device=dev)
    stats = torch.zeros(_lib.ST_LEN, dtype=torch.float64, device=dev)
    dm = torch.empty(B, D, dtype=torch.float32, device=dev)
    dls = torch.zeros(D, dtype=torch.float64, device=dev)

    ws = torch.empty(_lib.dvla_gauss_loss_workspace_bytes(n_groups, G, C), dtype=torch.uint8,
                     device=dev)

    def step(s):  # one C-ABI call: advantages -> lp -> epilogue -> head backward
        _lib.dvla_gauss_loss_fwd_bwd(means.data_ptr(), log_std.data_ptr(), actions.data_ptr(),
                                     blp.data_ptr(), rewards.data_ptr(), order_d.data_ptr(),
                                     ids_d.data_ptr(), n_groups, G, C, D, 0.2, 1e-8, 0.0,
                                     dm.data_ptr(), dls.data_ptr(), lp.data_ptr(),
                                     stats.data_ptr(), ws.data_ptr(), ws.numel(), s)

    for _ in range(5):
        step(st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        step(st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    eager_us = e0.elapsed_time(e1) / steps * 1e3
    # CUDA graph: the four launches captured once, replayed per step
    gs = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        step(gs.cuda_stream)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=gs):
            step(gs.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(steps):
        graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    graph_us = e0.elapsed_time(e1) / steps * 1e3
    out = {"workload": "C3 Gaussian head (pi0-shaped): 64 groups x 8 x 1 chunk, D = 1600, f32 "
                       "means/actions, f64 accumulation",
           "us_per_step_eager": eager_us, "us_per_step_graph": graph_us,
           "loss": float(stats[_lib.ST_LOSS].item()), "launches_per_step": 4}
    if cpu and rank == 0:
        sys.path.insert(0, ROOT)
        from oracle import grpo_oracle as O
        m, a, ls = means.cpu().numpy(), actions.cpu().numpy(), log_std.cpu().numpy()
        b3 = blp.cpu().numpy().reshape(n_groups, G, C)
        r2 = rewards.cpu().numpy().reshape(n_groups, G)
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            lpo = O.chunk_log_prob(m, ls, a)
            _, entries = O._entries(ids, r2, b3, G, 1e-8)
            res = O._epilogue(lambda key: lpo[(key[0] * G + key[1]) * C:(key[0] * G + key[1] + 1) * C],
                              entries, n_groups * G, 0.2, 0.0)
            cs = np.empty(B)
            for (k, i), v in res[4].items():
                cs[(k * G + i) * C:(k * G + i + 1) * C] = v
            O.gauss_head_backward(m, ls, a, cs)
        cpu_ms = (time.perf_counter() - t0) / reps * 1e3
        out["cpu_oracle_ms"] = cpu_ms
        out["cpu_cores"] = 1
        out["gpu_over_cpu"] = cpu_ms * 1e3 / graph_us
        out["loss_oracle"] = float(res[0])
    return out


def _bench_sampler(dev, logits, steps=20):
    """Rollout-side action-token sampling + behaviour log-prob
    over the same C2 logits: one read pass, HBM-bound."""
    import torch
    from paper_2605_13276_b200.rollout import sample_action_tokens
    for _ in range(3):
        sample_action_tokens(logits, T, seed=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        sample_action_tokens(logits, T, seed=1, offset=i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    nbytes = logits.numel() * logits.element_size()
    peak, _ = _peaks()
    return {"workload": "C2 logits [28672, 32064] bf16 -> tokens, lp_tok, blp (f32)",
            "ms": ms, "gbs": nbytes / ms / 1e6, "frac_of_hbm_peak": nbytes / ms / 1e6 / peak,
            "launches_per_step": 2}


def _bench_optimizer(dev, iters=10):
    """Learner optimizer tail on the OpenVLA action-head size:
    Adam (f32 params, f64 grad / moments) and the
    gradient norm, HBM-bound (Adam reads p, g, m, v and writes p, m, v: 48 B
    per parameter)."""
    import torch
    from paper_2605_13276_b200 import _lib
    n = V * 4096
    p = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev, dtype=torch.float64) * 1e-3
    m = torch.zeros(n, device=dev, dtype=torch.float64)
    v = torch.zeros(n, device=dev, dtype=torch.float64)
    ws = torch.empty(_lib.dvla_grad_norm_workspace_bytes(n), dtype=torch.uint8, device=dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    peak, _ = _peaks()
    out = {"params": n}
    for name, fn, nbytes in (
            ("adam", lambda it: _lib.dvla_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(),
                                                    v.data_ptr(), n, it + 1, 1e-4, 0.9, 0.999,
                                                    1e-8, s), n * 48),
            ("grad_norm", lambda it: _lib.dvla_grad_norm(g.data_ptr(), n, 0.0, norm.data_ptr(),
                                                         bad.data_ptr(), ws.data_ptr(), s),
             n * 8)):
        for it in range(3):
            fn(it)
        torch.cuda.synchronize()
        e0.record()
        for it in range(iters):
            fn(it)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        out[name] = {"ms": ms, "gbs": nbytes / ms / 1e6, "frac_of_hbm_peak": nbytes / ms / 1e6 / peak}
    return out


def _bench_weight_plane_cpu(n_params=250_000_000):
    """CPU baseline of the weight plane (SURVEY §8 d, CPU item iii): the
    reference's host path -- snapshot_from_params (copy + isfinite) ->
    ControlPlane.broadcast in WIRE mode (weight frame encode) -> one
    mailbox -> take_newest (decode) -- through this repo's byte-identical
    port, single-threaded, on 1 GB of f32 parameters."""
    import numpy as np
    from paper_2605_13276_b200.core import snapshot_from_params
    from paper_2605_13276_b200.planes import ControlPlane, Plane, Transport, TransportMode
    params = np.random.default_rng(0).standard_normal(n_params, dtype=np.float32)
    plane = ControlPlane(Transport(TransportMode.WIRE, Plane.CONTROL))
    box = plane.subscribe(name="replica")
    t0 = time.perf_counter()
    snap = snapshot_from_params(params, 1)
    plane.broadcast(snap)
    got = box.take_newest()
    dt = time.perf_counter() - t0
    assert got.version == 1
    return {"gbs": params.nbytes / dt / 1e9, "seconds": round(dt, 3), "bytes": params.nbytes,
            "cores": 1, "kind": "port",
            "path": "snapshot_from_params -> ControlPlane.broadcast (WIRE) -> take_newest"}


def _bench_allocator(n_ops=20_000, capacity=1 << 18, reps=20):
    """§8 d (iv): the dual-pool allocator's batched trace (csrc/arena.cpp,
    host C++ -- integer bookkeeping, no device kernel) on the reference's
    random workload, bitwise against the C restatement of alloc_trace_run
    timed beside it on one host thread."""
    import numpy as np

    from oracle.arena import alloc_trace
    from paper_2605_13276_b200.pools import arena_trace, random_workload
    wl = random_workload(0, n_ops, capacity)

    def best(fn):
        out, ts = None, []
        for _ in range(reps):
            t0 = time.perf_counter()
            out = fn(capacity, *wl)
            ts.append(time.perf_counter() - t0)
        return out, min(ts)
    (ok, off, fin), t_ours = best(arena_trace)
    (ok2, off2, fin2), t_or = best(alloc_trace)
    same = bool(np.array_equal(ok, ok2) and np.array_equal(off, off2) and fin == fin2)
    return {"workload": f"random_workload(0, {n_ops}, 2^18) (reference pools.py:219-231)",
            "ops_per_s": n_ops / t_ours, "bit_exact_vs_oracle": same,
            "cpu_baseline": {"ops_per_s": n_ops / t_or, "cores": 1, "kind": "port",
                             "impl": "oracle/arena_oracle.c (alloc_trace_run restated)"}}


def _bench_allreduce(world, dev, barrier, max_over_ranks, nbytes=1 << 30, iters=5):
    """NCCL all-reduce of a learner gradient bucket (f32), busbw."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return None
    g = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
    dist.all_reduce(g)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        barrier()
        e0.record(stream)
        dist.all_reduce(g)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(max_over_ranks(e0.elapsed_time(e1)))
    ms = sorted(ts)[len(ts) // 2]
    busbw = nbytes * 2 * (world - 1) / world / (ms / 1e3) / 1e9
    out = {"bytes": nbytes, "ms": ms, "busbw_gbs": busbw, "dtype": "f32",
           "frac_of_nominal_900": busbw / NVLINK_NOMINAL_GBS, "impl": "NCCL (ring)"}
    del g
    # the switch-reduced all-reduce (GradReducer's default where available)
    from paper_2605_13276_b200.replicate import McAllReduce, multicast_supported
    from paper_2605_13276_b200._lib import NativeError
    ar = None
    if max_over_ranks(0.0 if multicast_supported() else 1.0) == 0.0:
        try:
            ar = McAllReduce(nbytes // 4)
        except NativeError as e:
            out["nvls"] = {"unavailable": str(e)[:200]}
    if ar is not None:
        ar.buf.fill_(1.0)
        ar.allreduce()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            barrier()
            e0.record(stream)
            ar.allreduce()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(max_over_ranks(e0.elapsed_time(e1)))
        ar.check()
        ok = bool(torch.all(ar.buf == float(world ** (iters + 1))).item())
        barrier()
        ar.close()
        nms = sorted(ts)[len(ts) // 2]
        nbus = nbytes * 2 * (world - 1) / world / (nms / 1e3) / 1e9
        out["nvls"] = {"impl": "switch-reduced (multimem.ld_reduce + multimem.st)", "ms": nms,
                       "busbw_gbs": nbus, "frac_of_nominal_900": nbus / NVLINK_NOMINAL_GBS,
                       "exact": ok}
    return out


def _bench_c2_f32(dev, rank, world, barrier, max_over_ranks, steps=20):
    """The C2 step with f32 logits (the north star's 1e-5 parity dtype):
    the fused kernel streams each 128 KB row as two pieces.  Same timing
    rules as the headline (CUDA events on the launching stream, the fused
    kernel's own events in an interleaved profiled run, max over ranks)."""
    import numpy as np
    import torch

    from paper_2605_13276_b200 import _lib, grpo
    R = N_GROUPS * G * C * T
    gen = torch.Generator(device=dev).manual_seed(99 + rank)
    logits = torch.randn(R, V, device=dev, generator=gen) * 2.0
    tokens = torch.randint(31744, 32000, (R,), device=dev, generator=gen, dtype=torch.int32)
    rewards = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=gen).float()
    tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, grpo.GrpoConfig(group_size=G),
                        dtype=torch.float32, device=dev)
    tl.set_groups(np.arange(N_GROUPS) + rank * N_GROUPS)
    tl.launch(logits, tokens, torch.zeros(N_GROUPS * G * C, device=dev), rewards, None)
    blp = (tl.lp_chunk + (torch.rand(tl.lp_chunk.shape, device=dev, generator=gen,
                                     dtype=torch.float64) - 0.5) * 0.1).float()
    dl = torch.empty_like(logits)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        tl.launch(logits, tokens, blp, rewards, dl)
    tl.stats(rewards)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        tl.launch(logits, tokens, blp, rewards, dl)
    e1.record(stream)
    _lib.dvla_profile_enable(1)
    for _ in range(steps):
        tl.launch(logits, tokens, blp, rewards, dl)
    torch.cuda.synchronize()
    km, kn = _lib.profile_collect()
    _lib.dvla_profile_enable(0)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps)
    kms = max_over_ranks(km / max(kn, 1))
    st = tl.stats(rewards)
    N = R * V
    algo = 2 * N * 4 + R * 4 + N_GROUPS * G * C * (4 + 8) + N_GROUPS * G * 4
    peak, kind = _peaks()
    ach = algo / (kms / 1e3) / 1e9
    del logits, dl
    torch.cuda.empty_cache()
    return {"value": world * N_GROUPS * G / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "dtype": "f32", "target_ms_70pct": 1.633,
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "kernel": "tok_fused_kernel<f32, 2 pieces>",
                         "kernel_ms": round(kms, 4), "algo_bytes": algo,
                         "traffic": _traffic().get("tok_fused_kernel<f32,2>"),
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({kind})"},
            "loss": st["loss"]}


SWIM_H = 4096                        # OpenVLA-7B hidden size (the action head's K)


def _bench_learner_step(world, rank, dev, barrier, max_over_ranks, steps=10, warmup=3,
                        scatter="auto"):
    """The learner step of BASELINE config 4 per GPU, timed as a unit with
    its collective (reference TrainerWorker.update, runtime.py:768-800):
    per-token features -> logits GEMM (V=32,064 x H=4,096 bf16 head) ->
    fused token loss fwd+bwd -> f32 head-gradient GEMM in row blocks, with
    N GPUs ZeRO-1: each peer's block pushed over NVLink by a copy engine as
    it completes, own block last, node-order sum (scatter "peer"; "nccl" =
    NCCL reduce-scatter after the GEMM) -> grad norm -> optimizer tail on
    the own block (clip + Adam + bf16 copy + non-finite flag) -> bf16
    all-gather, one host sync per step.
    CUDA events on the trainer stream, max over ranks; the same 512
    trajectories every step (inputs 1.84 GB of logits > L2)."""
    import torch

    from paper_2605_13276_b200.pools import Pool, PoolKind
    from paper_2605_13276_b200.runtime import (GradReducer, SamplerWorker, SwimlaneConfig,
                                               TrainerWorker)
    cfg = SwimlaneConfig(n_groups=N_GROUPS, group_size=G, chunks=C, tokens=T, vocab=V,
                         hidden=SWIM_H, seed=23)
    n = V * SWIM_H
    R = N_GROUPS * G * C * T
    model_pool = Pool(PoolKind.MODEL_COMPUTE, n * 26 + (64 << 20), device=dev)
    env_pool = Pool(PoolKind.ENV_AUX, R * (V * 2 + SWIM_H * 2 + 64) + (256 << 20), device=dev)
    s_train = torch.cuda.Stream(device=dev, priority=-1)
    s_sample = torch.cuda.Stream(device=dev)
    import torch.distributed as dist
    reducer = GradReducer(world, None, scatter=scatter)
    trainer = TrainerWorker(cfg, rank, model_pool, reducer, s_train, dev)
    sampler = SamplerWorker(cfg, rank, world, [env_pool], s_sample, dev)
    msgs, _ = sampler.run_epoch(0, trainer.snapshot())
    names = ("start", "loss0", "loss1", "grad1", "reduce1", "norm1", "adam1", "end")
    phases = {k: 0.0 for k in ("feats_logits_gemm", "loss", "grad_gemm_and_reduce",
                               "reduce_wait", "norm_adam_tail", "tail_norm", "tail_adam",
                               "tail_gather")}
    for _ in range(warmup):
        trainer.update(msgs)
    barrier()
    walls, devs = [], []
    host = {"enqueue": 0.0, "wait": 0.0, "wall": 0.0}
    for _ in range(steps):
        ev = {k: torch.cuda.Event(enable_timing=True) for k in names}
        trainer.timing = ev
        t0 = time.perf_counter()
        trainer.update(msgs)       # ends with its one host sync
        walls.append(time.perf_counter() - t0)
        devs.append(ev["start"].elapsed_time(ev["end"]))
        host["enqueue"] += 1e3 * ev.get("host_enqueue_s", 0.0)
        host["wait"] += 1e3 * ev.get("host_wait_s", 0.0)
        host["wall"] += 1e3 * walls[-1]
        phases["feats_logits_gemm"] += ev["start"].elapsed_time(ev["loss0"])
        phases["loss"] += ev["loss0"].elapsed_time(ev["loss1"])
        phases["grad_gemm_and_reduce"] += ev["loss1"].elapsed_time(ev["grad1"])
        phases["reduce_wait"] += ev["grad1"].elapsed_time(ev["reduce1"])
        phases["norm_adam_tail"] += ev["reduce1"].elapsed_time(ev["end"])
        phases["tail_norm"] += ev["reduce1"].elapsed_time(ev["norm1"])
        phases["tail_adam"] += ev["norm1"].elapsed_time(ev["adam1"])
        phases["tail_gather"] += ev["adam1"].elapsed_time(ev["end"])
    trainer.timing = None
    barrier()
    dev_ms = max_over_ranks(sum(devs) / steps)
    wall_ms = max_over_ranks(1e3 * sum(walls) / steps)
    flops = 2 * 2 * R * SWIM_H * V            # logits GEMM + head-gradient GEMM
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            tf_peak = float(json.load(f)["bf16_tflops_sustained"])
    except Exception:  # noqa: BLE001
        tf_peak = 1394.0
    out = {"metric": "learner step (RL samples/s through update(), incl. the all-reduce)",
           "value": world * N_GROUPS * G / (wall_ms / 1e3), "unit": UNIT,
           "ms_per_step_wall": wall_ms, "ms_per_step_device": dev_ms,
           "phases_ms_rank0": {k: round(v / steps, 4) for k, v in phases.items()},
           "host_ms_rank0": {"enqueue": round(host["enqueue"] / steps, 4),
                             "wait_for_device": round(host["wait"] / steps, 4),
                             "after_sync": round((host["wall"] - host["enqueue"] - host["wait"])
                                                 / steps, 4)},
           "gemm_tflop_per_step": flops / 1e12,
           "gemm_roofline": {"bound": "tensor", "peak_tflops": tf_peak,
                             "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                             "achieved_tflops_step": round(flops / (dev_ms / 1e3) / 1e12, 1),
                             "frac_step": round(flops / (dev_ms / 1e3) / 1e12 / tf_peak, 4)},
           "config": f"V={V} x H={SWIM_H} bf16 head, {N_GROUPS}x{G} traj x {T} tokens per GPU; "
                     f"grad f32 {n * 4 / 1e9:.2f} GB reduce-scattered over {world} GPU(s)",
           "grad_gemms_per_block": getattr(trainer, "grad_sub", 1),
           "reduce_scatter": (("peer (exchange.PeerGradExchange): gradient GEMMs in plan "
                               f"'{getattr(trainer, 'grad_plan', '')}', each finished peer "
                               "block pushed over NVLink by a copy engine under the next GEMM, "
                               "node-order f64 sum; norm / abort scalars reduced over peer "
                               "memory; bf16 all-gather "
                               + ("stored into the peers by the optimizer-tail kernel"
                                  if getattr(trainer, "gather_mode", "") == "kernel" else
                                  "as copy-engine pushes per optimizer chunk")
                               + "; no collective-library call")
                              if getattr(trainer, "exchange", None) is not None else
                              ("NCCL: one gradient GEMM, reduce_scatter_tensor, all-reduce of "
                               "the scalars, all_gather_into_tensor" if world > 1 else None)),
           "steps": steps}
    trainer.close()
    del trainer, sampler, model_pool, env_pool, msgs
    torch.cuda.empty_cache()
    _ = dist
    return out


C3_WEIGHT_BYTES = 6_600_000_000     # pi0-3B-shaped bf16 weights (BASELINE config 3)


def _bench_disaggregated(world, rank, dev, epochs=8, keep_timeline=False, engine="ce_head",
                         staleness_limit=1):
    """BASELINE config 3 layout inside the RL loop (disagg.run_disaggregated):
    learner ranks {0, 1} (from 4 GPUs; {0} below) and rollout ranks, the
    C4-shaped action head trained on the rollout ranks' trajectories, and
    every published version -- the head plus a constant body blob up to the
    pi0-3B weight volume (6.6 GB) -- pushed over NVLink by the split TMA
    chains into the rollout ranks' MODEL_COMPUTE replica rings, checksummed
    on every receiver.  Rank 0 (learner 0) reports."""
    from paper_2605_13276_b200.disagg import default_learners, run_disaggregated
    from paper_2605_13276_b200.runtime import SwimlaneConfig
    cfg = SwimlaneConfig(n_groups=N_GROUPS, group_size=G, chunks=C, tokens=T, vocab=V,
                         hidden=SWIM_H, epochs=epochs, seed=29, staleness_limit=staleness_limit)
    body = max(0, C3_WEIGHT_BYTES - V * SWIM_H * 2)
    res = run_disaggregated(cfg, verify=True, body_bytes=body, timeout_s=300.0, engine=engine)
    tl = None
    import torch.distributed as dist
    mism = [None] * world
    dist.all_gather_object(mism, res.mismatched)
    if keep_timeline:
        tl = [None] * world
        dist.all_gather_object(tl, res.timeline)
    if rank != 0:
        return None
    sm = res.summary()
    L = default_learners(world)
    peak = _nvl_peak()
    S = V * SWIM_H * 2 + body
    gbs = S / (sm["receiver_ms_median_max"] / 1e3) / 1e9 if sm["receiver_ms_median_max"] else None
    return {"layout": f"learners {L}, rollout ranks {[r for r in range(world) if r not in L]}",
            "engine": engine, "staleness_limit": staleness_limit,
            "trajectories_per_s_total": sm["trajectories_per_s"],
            "updates": sm["updates"], "quarantined": sm["quarantined"],
            "weight_bytes_per_version": V * SWIM_H * 2 + body,
            "replication_ms_per_iteration_median": sm["receiver_ms_median_max"],
            "replication_gbs_per_receiver": gbs,
            "replication_frac_of_nvlink_peak": (gbs / peak) if gbs else None,
            "source_hop_ms_median": sm["replication_ms_median"],
            "lane_s_rank0": sm["lane_s"],
            "nvlink_peak_gbs": peak,
            "replication_overlapped_with_updates": sm["overlap"],
            "checksum_mismatches": sm["checksum_mismatches"],
            "mismatched_versions": {r: [m[0] for m in x] for r, x in enumerate(mism) if x},
            **({"timeline": tl} if tl else {}),
            "timing": "learner 0: host clock between first and last publish (traj/s); "
                      "replication: CUDA events around each rollout rank's hop launch on its "
                      "receive stream (launched once the chain heads run) until every chunk "
                      "landed, median per rank, max over ranks"}


def _bench_swimlane(world, rank, dev, max_over_ranks, epochs=8):
    """End-to-end RL samples/s of the four-lane swimlane (BASELINE config 4
    shape: OpenVLA-7B-sized action head V=32,064 x H=4,096, 64 groups x 8
    trajectories x 56 action tokens per GPU per epoch; one closed loop per
    GPU, NCCL gradient mean across GPUs).  Host-clock lane timing (the
    reference's transitions/s definition, metrics.py:101-123)."""
    from paper_2605_13276_b200.runtime import SwimlaneConfig, run_swimlane
    out = {}
    for mode, limit in (("async", 1), ("sync", 0)):
        cfg = SwimlaneConfig(n_groups=N_GROUPS, group_size=G, chunks=C, tokens=T, vocab=V,
                             hidden=SWIM_H, epochs=epochs, seed=17, staleness_limit=limit)
        s = run_swimlane(cfg, device=dev).summary()
        out[mode] = s
    traj = out["async"]["trajectories_per_s"]
    return {"trajectories_per_s_rank0": traj,
            "transitions_per_s_rank0": out["async"]["transitions_per_s"],
            "trajectories_per_s_total": traj * world,
            "sync_trajectories_per_s_rank0": out["sync"]["trajectories_per_s"],
            "async_over_sync": traj / max(out["sync"]["trajectories_per_s"], 1e-12),
            "epochs": epochs, "staleness_max": out["async"]["staleness_max"],
            "lanes": {m: {k: out[m][k] for k in ("transitions_per_s", "trajectories_per_s",
                                                 "rollout_time", "actor_time")}
                      for m in out},
            "config": "V=32064, H=4096, 64 groups x 8 traj x 56 tokens per GPU per epoch; "
                      "sync = the same lanes with staleness limit 0 (strict alternation)",
            "timing": "host clock per lane (reference transitions/s definition)"}


def _swim_model(swim, world, roofline, sampler, optimizer):
    """the swimlane's discrete-event model (sim.py, the
    reference DES rules) with lane costs from this run's measured B200
    rates, checked against the live lanes above (fit_check)."""
    from paper_2605_13276_b200 import sim
    kw = {}
    if isinstance(roofline, dict) and roofline.get("frac"):
        kw["loss_frac"] = roofline["frac"]
    if isinstance(sampler, dict) and sampler.get("frac_of_hbm_peak"):
        kw["sample_frac"] = sampler["frac_of_hbm_peak"]
    if isinstance(optimizer, dict) and isinstance(optimizer.get("adam"), dict):
        kw["adam_frac"] = optimizer["adam"]["frac_of_hbm_peak"]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            kw["gemm_tflops"] = float(json.load(f)["bf16_tflops"])
    except Exception:  # noqa: BLE001 - the dataclass default stands
        pass
    rates = sim.B200Rates(hbm_gbs=_peaks()[0], **kw)
    costs = sim.b200_costs(N_GROUPS, G, C, T, V, SWIM_H, nodes=world, rates=rates)
    R = N_GROUPS * G * C * T
    per_traj = N_GROUPS * G / R
    ep = swim["epochs"]

    def fit(res, mode):
        live = swim["lanes"][mode]
        f = sim.fit_check(res, {"mode": mode, "throughput": live["transitions_per_s"],
                                "rollout_time": live["rollout_time"],
                                "actor_time": live["actor_time"]}, threshold=0.25)
        out = {"predicted_trajectories_per_s": res.throughput * per_traj,
               "live_trajectories_per_s": live["trajectories_per_s"],
               "fit": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in f.items()}}
        if mode == "async":
            # both lanes run on one GPU here: a live lane's host time includes
            # waiting for the GPU the other lane holds, which the DES books as
            # slot waiting, not lane time -- the overlapped run is judged on
            # throughput
            out["fit"]["pass_throughput"] = f["throughput_dev"] <= 0.25
            out["fit"]["note"] = ("lane times include waiting for the shared GPU; "
                                  "judged on throughput")
        return out

    # one closed loop per GPU, coupled only through the gradient mean: each
    # GPU is modelled as its own node with the all-reduce inside the trainer
    # lane (the reference's multi-node pacing model counts versions, not
    # per-GPU epochs)
    akw = {"epochs": ep, "staleness_limit": 1}

    def per_gpu(c, reduce_s):
        return sim.LaneCosts(rollout_s=c.rollout_s, actor_s=c.actor_s + reduce_s,
                             shared_slots=True, transitions_per_epoch=R)
    a1 = per_gpu(costs, costs.reduce_s)
    # (1) analytic: lane costs from the measured kernel / GEMM / link rates
    out = {"analytic": {"rates": rates.__dict__, "rollout_s": a1.rollout_s,
                        "actor_s": a1.actor_s, "reduce_s": costs.reduce_s,
                        "sync": fit(sim.simulate(a1, "sync", epochs=ep), "sync"),
                        "async": fit(sim.simulate(a1, "async", **akw), "async")}}
    # (2) calibrated: the live strict-alternation (sync) lane times are the
    # lanes' isolated costs (the trainer's includes its all-reduce); the
    # model predicts the overlapped (async) run
    sl = swim["lanes"]["sync"]
    cal = sim.LaneCosts(rollout_s=sl["rollout_time"], actor_s=sl["actor_time"],
                        shared_slots=True, transitions_per_epoch=R)
    out["calibrated"] = {"rollout_s": cal.rollout_s, "actor_s": cal.actor_s,
                         "async": fit(sim.simulate(cal, "async", **akw), "async")}
    # the calibrated lanes at 8 GPUs: the analytic difference of the learner
    # lane between this run's N and 8 (ZeRO-1: the reduce-scatter /
    # all-gather grows to 7/8 of the bytes, the optimizer tail shrinks to
    # 1/8 of the parameters) applied to the live trainer lane
    c8 = sim.b200_costs(N_GROUPS, G, C, T, V, SWIM_H, nodes=8, rates=rates)
    d8 = (c8.actor_s + c8.reduce_s) - (costs.actor_s + costs.reduce_s)
    cal8 = sim.LaneCosts(rollout_s=cal.rollout_s, actor_s=max(cal.actor_s + d8, 1e-6),
                         shared_slots=True, transitions_per_epoch=R)
    r8 = sim.simulate(cal8, "async", **akw)
    out["predicted_8gpu_trajectories_per_s_total"] = r8.throughput * per_traj * 8
    return out


def run_ours(a):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_13276_b200 import _lib, grpo

    world, rank, local = _dist()
    if world > 1:
        torch.cuda.set_device(local)
        # NCCL's internal streams at high priority: the all-reduce kernels
        # are scheduled ahead of concurrently queued sampler work
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        dist.init_process_group("nccl", init_method="env://", world_size=world, rank=rank,
                                device_id=torch.device("cuda", local), pg_options=opts)
    dev = torch.device("cuda", torch.cuda.current_device())
    torch.cuda.set_device(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    R = N_GROUPS * G * C * T
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    logits = (torch.randn(R, V, device=dev, generator=gen) * 2.0).to(torch.bfloat16)
    tokens = torch.randint(31744, 32000, (R,), device=dev, generator=gen, dtype=torch.int32)
    rewards = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=gen).float()
    cfg = grpo.GrpoConfig(group_size=G)
    tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, cfg, dtype=torch.bfloat16, device=dev,
                        fused=not a.unfused)
    tl.set_groups(np.arange(N_GROUPS) + rank * N_GROUPS)
    # behaviour log-probs close to the current policy (as after one rollout)
    tl.launch(logits, tokens, torch.zeros(N_GROUPS * G * C, device=dev), rewards, None)
    blp = (tl.lp_chunk + (torch.rand(tl.lp_chunk.shape, device=dev, generator=gen,
                                     dtype=torch.float64) - 0.5) * 0.1).float()
    dl = torch.empty_like(logits)
    stream = torch.cuda.current_stream()

    clocks = Clocks(dev.index if dev.index is not None else 0)
    clocks.start()  # samples the warm-up tail and the whole timed region
    t_warm = time.perf_counter()
    w = 0
    min_warm_s = 0.0 if a.fixed_warmup else 0.5
    while w < max(a.warmup, 3) or time.perf_counter() - t_warm < min_warm_s:
        tl.launch(logits, tokens, blp, rewards, dl)
        w += 1
        if w % 16 == 0:
            torch.cuda.synchronize()
    st = tl.stats(rewards)  # raises GrpoAbort on bad data
    # Timed region: the K headline steps run in up to 4 chunks, each
    # followed by an equal chunk with a CUDA event pair around every fused
    # launch (the dominant kernel's own time).  The profiled chunks are not
    # part of the K steps -- an event between the PDL-linked launches would
    # serialise them -- and interleaving keeps both in the same thermal /
    # power state.  Barrier + synchronize on both sides of the whole region.
    n_chunks = 4 if a.steps >= 4 else 1
    sizes = [a.steps // n_chunks + (1 if i < a.steps % n_chunks else 0) for i in range(n_chunks)]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in sizes]
    barrier()
    torch.cuda.synchronize()
    kern_ms, kern_n = 0.0, 0
    for (c0, c1), k in zip(ev, sizes):
        c0.record(stream)
        for _ in range(k):
            tl.launch(logits, tokens, blp, rewards, dl)
        c1.record(stream)
        _lib.dvla_profile_enable(1)
        for _ in range(k):
            tl.launch(logits, tokens, blp, rewards, dl)
        torch.cuda.synchronize()
        km, kn = _lib.profile_collect()
        _lib.dvla_profile_enable(0)
        kern_ms, kern_n = kern_ms + km, kern_n + kn
    torch.cuda.synchronize()
    # reference: a plain device copy of the same bytes under the same
    # (warm, possibly power-capped) conditions, right after the timed region
    nbytes_rows = logits.numel() * logits.element_size()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(a.steps):
        _lib.dvla_memcpy_async(dl.data_ptr(), logits.data_ptr(), nbytes_rows, stream.cuda_stream)
    c1.record(stream)
    torch.cuda.synchronize()
    copy_gbs = 2 * nbytes_rows * a.steps / (c0.elapsed_time(c1) / 1e3) / 1e9
    clk = clocks.stop()
    barrier()
    ms = sum(c0.elapsed_time(c1) for c0, c1 in ev)
    ms_max = max_over_ranks(ms)
    kern_avg_ms = max_over_ranks(kern_ms / max(kern_n, 1))
    value = world * N_GROUPS * G * a.steps / (ms_max / 1e3)
    st = tl.stats(rewards)

    # ---- roofline of the dominant kernel (the fused loss kernel)
    N = R * V
    algo_bytes = 2 * N * 2 + R * 4 + N_GROUPS * G * C * (4 + 8) + N_GROUPS * G * 4
    peak, peak_kind = _peaks()
    achieved = algo_bytes / (kern_avg_ms / 1e3) / 1e9
    traffic = _traffic().get("tok_fused_kernel<bf16,1>")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "tok_fused_kernel<bf16, 1 piece>" if not a.unfused else "tok_rows+tok_bwd",
                "kernel_ms": round(kern_avg_ms, 4), "algo_bytes": algo_bytes,
                "kernel_timing": "CUDA events around each fused launch on its stream, in K "
                                 "profiled steps interleaved chunk by chunk with the K "
                                 "headline steps (events inside the headline steps would "
                                 "serialise the PDL launches)",
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "copy_gbs_same_conditions": round(copy_gbs, 1),
                "frac_of_copy_same_conditions": round(achieved / copy_gbs, 4)}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        h_logits = torch.empty((R, V), dtype=torch.bfloat16, pin_memory=True)
        h_logits.copy_(logits)
        h_tok = tokens.cpu().pin_memory()
        h_blp = blp.cpu().pin_memory()
        h_rw = rewards.cpu().pin_memory()
        h_stats = [torch.empty(_lib.ST_LEN, dtype=torch.float64, pin_memory=True)
                   for _ in range(2)]
        # two input slots: step k + 1's host->device copy (copy stream) runs
        # while step k's kernel runs (the copy, not the kernel, is the bound)
        slots = [(torch.empty_like(logits), torch.empty_like(tokens), torch.empty_like(blp),
                  torch.empty_like(rewards)) for _ in range(2)]
        s_copy = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        e_steps = max(2, min(a.steps, 5))
        e_k = [0]

        def e2e_step():
            k = e_k[0] % 2
            e_k[0] += 1
            d_logits, d_tok, d_blp, d_rw = slots[k]
            with torch.cuda.stream(s_copy):
                if e_k[0] > 2:
                    s_copy.wait_event(consumed[k])   # the kernel that read this slot
                d_logits.copy_(h_logits, non_blocking=True)
                d_tok.copy_(h_tok, non_blocking=True)
                d_blp.copy_(h_blp, non_blocking=True)
                d_rw.copy_(h_rw, non_blocking=True)
                copied[k].record(s_copy)
            stream.wait_event(copied[k])
            tl.launch(d_logits, d_tok, d_blp, d_rw, dl)
            consumed[k].record(stream)
            h_stats[k].copy_(tl.stats_dev, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_copy.wait_event(e0)
        for _ in range(e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1))
        barrier()
        # the last step's result as read back on the host vs the device one
        e2e_ok = bool(torch.equal(h_stats[(e_k[0] - 1) % 2], tl.stats_dev.cpu()))
        # the bound: a plain pinned host -> device copy of the logits alone
        h2d_best = 1e9
        for _ in range(2):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            slots[0][0].copy_(h_logits, non_blocking=True)
            c1.record(stream)
            torch.cuda.synchronize()
            h2d_best = min(h2d_best, c0.elapsed_time(c1))
        h2d_gbs = R * V * 2 / (h2d_best / 1e3) / 1e9
        h2d = R * V * 2 + R * 4 + N_GROUPS * G * C * 4 + N_GROUPS * G * 4
        e2e = {"value": world * N_GROUPS * G * e_steps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": _lib.ST_LEN * 8,
               "steps": e_steps, "ms_per_step": ems / e_steps,
               "pipelining": "two input slots: step k+1's H2D copy overlaps step k's kernel",
               "result_read_back": e2e_ok,
               "roofline": {"bound": "pcie_h2d", "unit": "GB/s",
                            "achieved": round(h2d / (ems / e_steps / 1e3) / 1e9, 2),
                            "peak": round(h2d_gbs, 2),
                            "frac": round(h2d / (ems / e_steps / 1e3) / 1e9 / h2d_gbs, 4),
                            "peak_source": "measured in this run: one pinned 1.84 GB "
                                           "host->device copy, best of 2 (split over 2-8 "
                                           "streams it is no faster: tools/h2d_probe.py)"}}
        del h_logits, slots

    del dl
    c2_f32 = None if a.no_f32 else _guarded(_bench_c2_f32, dev, rank, world, barrier,
                                            max_over_ranks)
    repl = None if a.no_repl else _bench_replication(world, rank, dev, barrier, max_over_ranks)
    allreduce = _bench_allreduce(world, dev, barrier, max_over_ranks)
    learner = None if a.no_swimlane else _guarded(_bench_learner_step, world, rank, dev, barrier,
                                                  max_over_ranks)
    if learner and world > 1 and "value" in learner:
        # the same step with NCCL's reduce-scatter (the collective-library baseline)
        alt = _guarded(_bench_learner_step, world, rank, dev, barrier, max_over_ranks,
                       scatter="nccl")
        if alt and "value" in alt:
            learner["nccl_reduce_scatter"] = {k: alt[k] for k in (
                "value", "ms_per_step_wall", "ms_per_step_device", "phases_ms_rank0")}
    # secondary per-GPU measurements: a failure is reported, never fatal to
    # the headline line
    gauss = None if a.no_gauss else _guarded(_bench_gauss_c3, dev, rank, cpu=not a.no_cpu)
    sampler = None if a.no_gauss else _guarded(_bench_sampler, dev, logits)
    optimizer = None if a.no_gauss else _guarded(_bench_optimizer, dev)
    swim = None
    if not a.no_swimlane:
        barrier()
        swim = _guarded(_bench_swimlane, world, rank, dev, max_over_ranks)
        barrier()
        if "error" not in swim:
            swim["model"] = _guarded(_swim_model, swim, world, roofline, sampler, optimizer)
        if world >= 2:
            barrier()
            swim["disaggregated"] = _guarded(_bench_disaggregated, world, rank, dev)
            barrier()
            # the same layout with one more version of slack in the gate: the
            # push leaves the rollout epochs' critical path (learner-bound)
            swim["disaggregated_staleness2"] = _guarded(_bench_disaggregated, world, rank, dev,
                                                        staleness_limit=2)
            barrier()
            # strict alternation in the same layout (staleness limit 0: every
            # epoch waits for the previous update's version to arrive)
            swim["disaggregated_sync"] = _guarded(_bench_disaggregated, world, rank, dev,
                                                  staleness_limit=0)
            barrier()
            try:
                swim["disaggregated_async_over_sync"] = (
                    swim["disaggregated"]["trajectories_per_s_total"]
                    / swim["disaggregated_sync"]["trajectories_per_s_total"])
            except (TypeError, KeyError, ZeroDivisionError):
                pass
        # the GPU-work bound of one epoch on one GPU: the sampler's device
        # work (the strict-alternation rollout lane) + the learner step
        if (isinstance(learner, dict) and "ms_per_step_device" in learner
                and "lanes" in swim):
            t_epoch = swim["lanes"]["sync"]["rollout_time"] + learner["ms_per_step_device"] / 1e3
            bound = N_GROUPS * G / t_epoch
            swim["gpu_work_bound_trajectories_per_s_rank0"] = bound
            swim["async_frac_of_gpu_work_bound"] = swim["trajectories_per_s_rank0"] / bound

    if rank == 0 and world == 1 and not a.no_cpu and isinstance(repl, dict):
        repl["cpu_baseline"] = _guarded(_bench_weight_plane_cpu)
    allocator = _guarded(_bench_allocator) if rank == 0 and not a.no_cpu else None

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        def cpu_leg():
            # passes over one resident 16-group sample until >= 10 s of CPU work
            threads = len(os.sched_getaffinity(0))
            inputs = _cpu_inputs(CPU_GROUPS)
            _, dt1 = _cpu_sample(threads, inputs, 1)
            reps = max(1, min(60, int(10.0 / max(dt1, 1e-3)) + 1))
            v, dt = _cpu_sample(threads, inputs, reps)
            return {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                    "sample": f"{reps} passes x {CPU_GROUPS} groups x 8 trajectories x 56 tokens "
                              f"x 32064 vocab (C2 rows; oracle numpy f64, rows split over all "
                              f"host threads)",
                    "seconds": round(dt, 3)}
        cpu = _guarded(cpu_leg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "C2 token-head GRPO loss fwd+bwd (OpenVLA-7B-shaped action head)",
                       "n_groups_per_gpu": N_GROUPS, "G": G, "C": C, "T": T, "V": V,
                       "trajectories_per_gpu_step": N_GROUPS * G,
                       "parallelism": f"dp{world} (group-sharded learner)",
                       "l2": "inputs 1.84 GB/rank > 126 MB L2 (no flush needed)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "c2_f32": c2_f32, "learner_step": learner,
            "rl_samples_per_s_end_to_end": (swim or {}).get("trajectories_per_s_total"),
            "replication": repl, "grad_allreduce": allreduce, "swimlane": swim,
            "gauss_c3": gauss, "sampler": sampler, "optimizer": optimizer,
            "allocator": allocator,
            "gpu_launches": 3 * a.steps, "clocks": clk,
            "loss": st["loss"], "mean_ratio": st["mean_ratio"],
            "clip_fraction": st["clip_fraction"],
        }
        _emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


_JSON_FD = None


def _guarded(fn, *args, **kw):
    """Run a secondary, single-rank measurement; report its failure in the
    JSON line instead of losing the whole line."""
    try:
        return fn(*args, **kw)
    except Exception as e:  # noqa: BLE001 - any failure of a secondary leg
        import traceback
        traceback.print_exc()
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def _quiet_stdout():
    """Keep stdout for the one JSON line: anything else written to fd 1 (the
    NCCL version banner, library chatter) goes to stderr."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def _emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    _quiet_stdout()
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
