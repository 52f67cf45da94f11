"""The kernel seam, B200 edition.

Reference pkg/src/dvla/kernels/__init__.py:41-51 binds a module-level
function table once at import (numba or numpy backend, chosen by
DVLA_BACKEND).  This module keeps the in-scope entries of that table with
the same signatures and semantics, all bound to libdvla_b200.so; there is
exactly one backend and no environment switch (no multi-backend dispatch,
no CPU fallback).  Out of scope: `spin` (synthetic cost) and
`env_step_chunk` (toy physics); `alloc_oracle_run` is a test oracle.

Arrays may be numpy (copied to/from the device around the call, like the
reference's host arrays) or CUDA tensors (zero-copy).
"""

from __future__ import annotations

import numpy as np

from . import _lib  # noqa: F401  (fails loudly without the native library)

BACKEND = "b200"


def _is_t(x) -> bool:
    return type(x).__module__.startswith("torch")


def mlp_forward(w1, b1, w2, b2, obs):
    """(B, obs_dim) -> (B, out_dim) f32 means (numba_backend.py:27-46)."""
    from .policy import PolicyParams, forward
    return forward(PolicyParams(w1=w1, b1=b1, w2=w2, b2=b2, log_std=b2), obs)


def chunk_log_prob(means, log_std, actions):
    """Joint diagonal-Gaussian log density per row, f64 (numba_backend.py:49-61)."""
    from .policy import chunk_log_prob_dev, to_dev
    out = chunk_log_prob_dev(to_dev(means), to_dev(log_std), to_dev(actions))
    return out if _is_t(means) else out.cpu().numpy()


def policy_backward(w1, b1, w2, b2, log_std, obs, actions, coeffs, out):
    """out += sum_b coeffs[b] * d log_prob_b / d params (numba_backend.py:64-113)."""
    from .policy import PolicyParams, backward_batch
    backward_batch(PolicyParams(w1=w1, b1=b1, w2=w2, b2=b2, log_std=log_std), obs, actions,
                   coeffs, out)


def gauss_head_backward(means, log_std, actions, coeffs):
    """Head-only Gaussian backward: (dmeans f32 [B,D], dlog_std f64 [D])."""
    import torch
    from .policy import to_dev
    m, ls, a = to_dev(means), to_dev(log_std), to_dev(actions)
    c = to_dev(coeffs, torch.float64)
    B, D = m.shape
    dm = torch.empty((B, D), dtype=torch.float32, device=m.device)
    dls = torch.zeros(D, dtype=torch.float64, device=m.device)
    _lib.check(_lib.dvla_gauss_head_backward(m.data_ptr(), ls.data_ptr(), a.data_ptr(),
                                             c.data_ptr(), B, D, dm.data_ptr(), dls.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream),
               "dvla_gauss_head_backward")
    if _is_t(means):
        return dm, dls
    return dm.cpu().numpy(), dls.cpu().numpy()


def alloc_trace_run(capacity, is_alloc, size, align, pick, out_ok, out_off):
    """Batched allocator trace (numba_backend.py:139-247): fills out_ok /
    out_off and returns (total_free, largest_free, n_extents)."""
    from .pools import arena_trace
    ok, off, fin = arena_trace(capacity, is_alloc, size, align, pick)
    out_ok[:] = ok
    out_off[:] = off
    return fin


def token_loss_fwd_bwd(logits, tokens, behavior_log_prob, rewards, group_ids, cfg,
                       dlogits=None):
    """The north-star kernel: fused action-token GRPO loss fwd + bwd."""
    from .grpo import grpo_token_grad
    return grpo_token_grad(logits, tokens, behavior_log_prob, rewards, group_ids, cfg,
                           dlogits=dlogits)


def warmup():
    """Kernels are compiled ahead of time (sm_100a cubins in the .so)."""
    return None


__all__ = ["BACKEND", "mlp_forward", "chunk_log_prob", "policy_backward", "gauss_head_backward",
           "alloc_trace_run", "token_loss_fwd_bwd", "warmup"]
_ = np
