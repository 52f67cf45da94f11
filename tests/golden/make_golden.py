"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs small .npz fixtures next to this script; they are committed and are
what the oracle (oracle/) and the GPU parity tests are pinned against.
Every fixture records which reference function produced it.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from dvla import grpo, kernels, pools, wire  # noqa: E402
from dvla.core import Rng, snapshot_from_params  # noqa: E402
from dvla.grpo import GrpoConfig  # noqa: E402
from dvla.policy import flatten  # noqa: E402
from helpers import GRAD_CHECK_GRPO, brute_force_trace, make_gradient_case  # noqa: E402


def advantages():
    """compute_advantages (grpo.py:89-99) on ragged reward groups."""
    rng = np.random.Generator(np.random.Philox(key=2024))
    sizes = list(range(2, 40)) + [64, 127, 128, 129, 256, 300, 1000]
    rewards, offs, kinds = [], [0], []
    for g in sizes:
        for kind in range(5):
            if kind == 0:
                r = rng.integers(0, 2, g).astype(np.float64)          # binary
            elif kind == 1:
                r = rng.uniform(0, 1, g).astype(np.float32).astype(np.float64)
            elif kind == 2:
                r = rng.integers(-64, 65, g).astype(np.float64) / 8.0  # dyadic
            elif kind == 3:
                r = rng.normal(1.5, 3.0, g)
            else:
                r = np.full(g, rng.uniform(-100, 100))                 # constant
            rewards.append(r)
            offs.append(offs[-1] + g)
            kinds.append(kind)
    # Appendix B.2 quirk: three identical non-dyadic rewards -> tiny non-zero A
    rewards.append(np.array([86.0426146651424] * 3))
    offs.append(offs[-1] + 3)
    kinds.append(9)
    flat = np.concatenate(rewards)
    adv = np.concatenate([grpo.compute_advantages(r, 1e-8) for r in rewards])
    np.savez_compressed(OUT / "advantages.npz", rewards=flat, offsets=np.array(offs),
                        kinds=np.array(kinds), adv=adv, delta=1e-8)


def grpo_cases():
    """grpo_grad (grpo.py:217-294) on helpers.make_gradient_case seeds."""
    out = {}
    for seed in range(10):
        for kl in (0.0, 0.5):
            if kl and seed not in (3, 7):
                continue
            params, batches = make_gradient_case(seed)
            cfg = GrpoConfig(**{**GRAD_CHECK_GRPO.__dict__, "kl_coeff": kl})
            loss, grad, st = grpo.grpo_grad(params, batches, cfg)
            tag = f"s{seed}_kl{int(kl * 10)}"
            out[f"{tag}_w1"] = params.w1
            out[f"{tag}_b1"] = params.b1
            out[f"{tag}_w2"] = params.w2
            out[f"{tag}_b2"] = params.b2
            out[f"{tag}_log_std"] = params.log_std
            out[f"{tag}_group_ids"] = np.array([b.group_id for b in batches])
            out[f"{tag}_obs"] = np.stack([b.obs for b in batches])
            out[f"{tag}_actions"] = np.stack([b.actions for b in batches])
            out[f"{tag}_blp"] = np.stack([b.behavior_log_prob for b in batches])
            out[f"{tag}_rewards"] = np.stack([b.rewards for b in batches])
            out[f"{tag}_loss"] = np.float64(loss)
            out[f"{tag}_grad"] = grad.copy()
            out[f"{tag}_stats"] = np.array([st["loss"], st["mean_ratio"], st["clip_fraction"],
                                            st["n_chunks"], st["mean_reward"]])
            out[f"{tag}_kl"] = np.float64(kl)
            if kl == 0.0:
                # one Adam step of grpo_update on the same case
                adam = grpo.AdamState.zeros(params.n_params)
                newp, ust = grpo.grpo_update(params, batches, cfg, adam, 4)
                out[f"{tag}_updated"] = flatten(newp)
                out[f"{tag}_grad_norm"] = np.float64(ust.grad_norm)
    np.savez_compressed(OUT / "grpo_gauss.npz", **out)


def kernel_cases():
    """chunk_log_prob / mlp_forward / policy_backward (numba default backend)."""
    rng = Rng(3)
    means = rng.gaussian2d((37, 8))
    log_std = (rng.gaussian(8) * 0.1).astype(np.float32)
    actions = rng.gaussian2d((37, 8))
    lp = kernels.chunk_log_prob(means, log_std, actions)
    r2 = Rng(4)
    w1 = r2.gaussian2d((8, 4)) * 0.3
    b1 = r2.gaussian(8) * 0.1
    w2 = r2.gaussian2d((8, 8)) * 0.3
    b2 = r2.gaussian(8) * 0.1
    ls2 = r2.gaussian(8) * 0.1
    obs = r2.gaussian2d((29, 4))
    act = r2.gaussian2d((29, 8))
    coeffs = r2.gaussian(29).astype(np.float64)
    mf = kernels.mlp_forward(w1, b1, w2, b2, obs)
    out = np.zeros(w1.size + b1.size + w2.size + b2.size + ls2.size)
    kernels.policy_backward(w1, b1, w2, b2, ls2, obs, act, coeffs, out)
    np.savez_compressed(OUT / "kernels.npz", means=means, log_std=log_std, actions=actions,
                        lp=lp, w1=w1, b1=b1, w2=w2, b2=b2, ls2=ls2, obs=obs, act=act,
                        coeffs=coeffs, mlp_out=mf, backward=out, backend=kernels.BACKEND)


def alloc_traces():
    """alloc_trace_run (numba_backend.py:139-247) == brute_force_trace."""
    out = {}
    for seed, n, cap in ((0, 20000, 1 << 18), (1, 20000, 1 << 18), (11, 3000, 1 << 16),
                         (17, 20000, 1 << 18), (5, 2000, 1 << 12)):
        is_alloc, size, align, pick = pools.random_workload(seed, n, cap)
        ok = np.zeros(n, np.uint8)
        off = np.zeros(n, np.int64)
        final = kernels.alloc_trace_run(cap, is_alloc, size, align, pick, ok, off)
        ok_b = np.zeros(n, np.uint8)
        off_b = np.zeros(n, np.int64)
        final_b = brute_force_trace(cap, is_alloc, size, align, pick, ok_b, off_b)
        assert np.array_equal(ok, ok_b) and np.array_equal(off, off_b)
        tag = f"s{seed}"
        out[f"{tag}_cap"] = np.int64(cap)
        out[f"{tag}_n"] = np.int64(n)
        out[f"{tag}_ok"] = ok
        out[f"{tag}_off"] = off
        out[f"{tag}_final"] = np.array([int(x) for x in final], dtype=np.int64)
    # churn (pools.py:281-315)
    for unified in (True, False):
        failed, st = pools.run_churn(unified)
        m = st["model"]
        out[f"churn_{int(unified)}"] = np.array(
            [failed, m.total_free, m.largest_free_block, m.failed_allocs,
             int(m.fragmentation * 1e12)], dtype=np.int64)
    np.savez_compressed(OUT / "alloc_traces.npz", **out)


def wire_frames():
    """Weight-snapshot frame (wire.py:144-147) bytes."""
    snap = snapshot_from_params(Rng(1).gaussian(37).astype(np.float32), 9)
    frame = wire.encode(snap)
    assert len(frame) == wire.weight_frame_size(37)
    np.savez_compressed(OUT / "wire.npz", params=snap.params, version=np.int64(9),
                        frame=np.frombuffer(frame, dtype=np.uint8),
                        meta=np.frombuffer(wire.encode(wire.MetadataMsg(entries=())), np.uint8),
                        ack=np.frombuffer(wire.encode(wire.AckMsg(epoch_id=77)), np.uint8))


if __name__ == "__main__":
    advantages()
    grpo_cases()
    kernel_cases()
    alloc_traces()
    wire_frames()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
