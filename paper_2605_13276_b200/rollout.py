"""Rollout side of the token head: sample action tokens and record their
behaviour log-probs in one pass over the logits (csrc/sample.cu).

Token-head analogue of reference policy.sample_chunk_batch
(policy.py:150-158) + the sampler's f32 behaviour log-prob store
(runtime.py:696-698).  Draws come from a counter-based Philox stream keyed by
(seed, offset, row), so a rollout is reproducible bit for bit regardless of
stream or thread scheduling (the reference's Rng substream contract,
core.py:46-64).
"""

from __future__ import annotations

from .core import UsageError


def sample_action_tokens(logits, T: int, seed: int, offset: int = 0, want_lp_tok: bool = False):
    """logits [R, V] (bf16/f32 CUDA) -> (tokens int32 [R], blp f32 [R//T],
    lp_chunk f64 [R//T][, lp_tok f64 [R]])."""
    import torch

    from . import _lib
    if not (isinstance(logits, torch.Tensor) and logits.is_cuda and logits.dim() == 2):
        raise UsageError("logits must be a 2-D CUDA tensor")
    if logits.dtype not in (torch.bfloat16, torch.float32):
        raise UsageError(f"logits dtype must be bf16 or f32, got {logits.dtype}")
    lg = logits.contiguous()
    R, V = lg.shape
    if T < 1 or R % T:
        raise UsageError(f"rows ({R}) must be a multiple of T ({T})")
    dev = lg.device
    tokens = torch.empty(R, dtype=torch.int32, device=dev)
    lp_tok = torch.empty(R, dtype=torch.float64, device=dev)
    blp = torch.empty(R // T, dtype=torch.float32, device=dev)
    lp_chunk = torch.empty(R // T, dtype=torch.float64, device=dev)
    code = _lib.BF16 if lg.dtype == torch.bfloat16 else _lib.F32
    with torch.cuda.device(dev):
        _lib.check(_lib.dvla_token_sample(
            lg.data_ptr(), code, R, V, T, int(seed) & (2**64 - 1), int(offset) & (2**64 - 1),
            tokens.data_ptr(), lp_tok.data_ptr(), blp.data_ptr(), lp_chunk.data_ptr(),
            torch.cuda.current_stream().cuda_stream), "dvla_token_sample")
    if want_lp_tok:
        return tokens, blp, lp_chunk, lp_tok
    return tokens, blp, lp_chunk
