"""ctypes binding of libdvla_b200.so (the C-ABI in include/dvla_b200.h).

This is the only place Python touches native code.  There is no fallback:
if the shared library is missing or fails to load, importing the package's
compute modules raises immediately (the product path must never route
through a CPU implementation).  ctypes releases the GIL for the duration of
every call, which gives the four swimlane threads the same concurrency the
reference gets from numba's nogil kernels (reference
kernels/numba_backend.py:1-5).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .core import ConfigError, UsageError

_LIB_PATH = Path(os.environ["DVLA_B200_LIB"]) if os.environ.get("DVLA_B200_LIB") else Path(__file__).resolve().parent / "libdvla_b200.so"

# status codes (include/dvla_b200.h: enum dvla_status)
OK = 0
ERR_USAGE = 1
ERR_CONFIG = 2
ERR_GRPO_ABORT = 3
ERR_ALLOC_FAILURE = 4
ERR_POOL_USAGE = 5
ERR_CUDA = 6
ERR_DECODE = 7
ERR_TIMEOUT = 8

F32, BF16, U8, F64 = 0, 1, 2, 3
TL_WRITE_DLOGITS = 1
TL_UNFUSED = 2

ST_LOSS, ST_RATIO_SUM, ST_CLIP_COUNT, ST_CHUNK_COUNT = 0, 1, 2, 3
ST_ABORT, ST_ABORT_GROUP, ST_KERNEL_ERR, ST_RESERVED, ST_LEN = 4, 5, 6, 7, 8


class NativeError(RuntimeError):
    """CUDA-level failure inside libdvla_b200 (no reference analogue)."""


class ReplicationTimeout(RuntimeError):
    """A replication flag wait exceeded its deadline (peer never delivered)."""


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -m paper_2605_13276_b200.build` "
            "(there is no CPU fallback)")
    return C.CDLL(str(_LIB_PATH), mode=os.RTLD_LOCAL)


lib = _load()

_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_f64 = C.c_double
_sz = C.c_size_t


def _proto(name, args, res=C.c_int):
    fn = getattr(lib, name)
    fn.argtypes = args
    fn.restype = res
    return fn


dvla_last_error = _proto("dvla_last_error", [], C.c_char_p)
dvla_abi_version = _proto("dvla_abi_version", [], C.c_int)

dvla_profile_enable = _proto("dvla_profile_enable", [_i32])
dvla_profile_collect = _proto("dvla_profile_collect", [C.POINTER(C.c_double), C.POINTER(_i64)])
dvla_advantages = _proto("dvla_advantages", [_vp, _i64, _i64, _f64, _vp, _vp])
dvla_group_advantages = _proto("dvla_group_advantages", [_vp, _i64, _i64, _f64, _vp, _vp, _vp])
dvla_token_loss_workspace_bytes = _proto(
    "dvla_token_loss_workspace_bytes", [_i64, _i64, _i64, _i64], _sz)
dvla_token_loss_workspace_layout = _proto(
    "dvla_token_loss_workspace_layout", [_i64, _i64, _i64, _i64, C.POINTER(_sz)])
dvla_token_loss_fwd_bwd = _proto("dvla_token_loss_fwd_bwd", [
    _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64,
    _f64, _f64, _f64, _i32, _vp, _vp, _vp, _vp, _sz, _vp])
dvla_grpo_epilogue = _proto("dvla_grpo_epilogue", [
    _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _f64, _vp, _vp, _vp])


def last_error() -> str:
    msg = dvla_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a dvla status onto the reference's exception types."""
    if status == OK:
        return
    msg = last_error() or what
    if status == ERR_CONFIG:
        raise ConfigError(msg)
    if status == ERR_USAGE:
        raise UsageError(msg)
    if status == ERR_POOL_USAGE:
        from .pools import PoolUsageError
        raise PoolUsageError(msg)
    if status == ERR_TIMEOUT:
        raise ReplicationTimeout(msg)
    if status == ERR_DECODE:
        from .wire import DecodeError
        raise DecodeError(-1, msg)
    raise NativeError(f"{what}: {msg} (status {status})")


def profile_collect() -> tuple[float, int]:
    ms = C.c_double(0.0)
    n = _i64(0)
    check(dvla_profile_collect(C.byref(ms), C.byref(n)), "dvla_profile_collect")
    return ms.value, n.value


def exported_symbols() -> list[str]:
    """Every dvla_* symbol the header declares (parsed from include/)."""
    import re
    hdr = (Path(__file__).resolve().parent.parent / "include" / "dvla_b200.h").read_text()
    return sorted(set(re.findall(r"\b(dvla_[a-z0-9_]+)\s*\(", hdr)))


# ------------------------------------------------------------- arena / pools
POOL_MODEL_COMPUTE, POOL_ENV_AUX, POOL_UNIFIED_BASELINE = 0, 1, 2
_pp = C.c_void_p
_i64p = C.POINTER(_i64)
dvla_arena_create = _proto("dvla_arena_create", [_i32, _i64, C.POINTER(_pp), _i64p])
dvla_arena_destroy = _proto("dvla_arena_destroy", [_pp])
dvla_arena_alloc = _proto("dvla_arena_alloc", [_pp, _i64, _i64, _i64p, _i64p, _i64p])
dvla_arena_free = _proto("dvla_arena_free", [_pp, _i64, _i64, _i64, _i64, _i64])
dvla_arena_epoch_reset = _proto("dvla_arena_epoch_reset", [_pp])
dvla_arena_is_live = _proto("dvla_arena_is_live", [_pp, _i64, _i64, C.POINTER(C.c_int)])
dvla_arena_stats = _proto("dvla_arena_stats", [_pp, _i64p])
dvla_arena_trace = _proto("dvla_arena_trace", [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp])

# ------------------------------------------------------- weight replication
class Hop(C.Structure):
    _fields_ = [("src", _vp), ("dst", _vp), ("wait_flags", _vp), ("signal_flags", _vp)]


dvla_dev_alloc = _proto("dvla_dev_alloc", [_i32, _sz, C.POINTER(_pp)])
dvla_dev_free = _proto("dvla_dev_free", [_pp])
dvla_ipc_handle = _proto("dvla_ipc_handle", [_vp, C.c_char_p])
dvla_ipc_open = _proto("dvla_ipc_open", [C.c_char_p, C.POINTER(_pp)])
dvla_ipc_close = _proto("dvla_ipc_close", [_pp])
dvla_enable_peer_access = _proto("dvla_enable_peer_access", [_i32, _i32])
dvla_replicate_chain = _proto("dvla_replicate_chain", [
    C.POINTER(Hop), _i32, _i64, _i64, C.c_uint32, _i32, C.c_uint64, _vp, _vp])
dvla_snapshot_copy = _proto("dvla_snapshot_copy", [_vp, _vp, _i64, _i32, _vp, _vp])
dvla_bytes_equal = _proto("dvla_bytes_equal", [_vp, _vp, _i64, _vp, _vp])
dvla_checksum64 = _proto("dvla_checksum64", [_vp, _i64, _vp, _vp])
dvla_checksum64_at = _proto("dvla_checksum64_at", [_vp, _i64, _i64, _vp, _vp])
dvla_torch_pool_bind = _proto("dvla_torch_pool_bind", [_i32, _vp, _vp])
dvla_memcpy_async = _proto("dvla_memcpy_async", [_vp, _vp, _i64, _vp])
dvla_nccl_init = _proto("dvla_nccl_init", [_i32, C.POINTER(_i32)])
dvla_nccl_group_start = _proto("dvla_nccl_group_start", [])
dvla_nccl_group_end = _proto("dvla_nccl_group_end", [])
dvla_nccl_allreduce_sum = _proto("dvla_nccl_allreduce_sum", [_i32, _vp, _i64, _i32, _vp])
dvla_nccl_destroy = _proto("dvla_nccl_destroy", [])
dvla_replicate = _proto("dvla_replicate", [_i32, _vp, _i32, C.POINTER(_i32), C.POINTER(_vp), _i64,
                                           _i64, _i32, C.POINTER(_vp)])
dvla_replicate_status = _proto("dvla_replicate_status", [C.POINTER(_i32)])
dvla_replicate_hop_ce = _proto("dvla_replicate_hop_ce", [_vp, _vp, _vp, _vp, _i64, _i64,
                                                         C.c_uint32, _vp])
dvla_stream_wait_u32 = _proto("dvla_stream_wait_u32", [_vp, C.c_uint32, _vp])
dvla_stream_write_u32 = _proto("dvla_stream_write_u32", [_vp, C.c_uint32, _vp])
dvla_wait_flags_u32 = _proto("dvla_wait_flags_u32", [_vp, C.c_uint32, C.c_uint32, C.c_uint64, _vp,
                                                       _vp])
dvla_peer_reduce = _proto("dvla_peer_reduce", [_i32, _vp, _i32, C.POINTER(_vp), C.POINTER(_vp), _i32,
                                                 _i32, _vp, _vp, C.c_uint32, C.c_uint64, _vp, _vp,
                                                 _vp])
dvla_mc_supported = _proto("dvla_mc_supported", [_i32, C.POINTER(_i32)])
dvla_mc_create = _proto("dvla_mc_create", [_i32, _sz, C.POINTER(_i32), C.POINTER(_sz),
                                           C.POINTER(_pp)])
dvla_mc_import = _proto("dvla_mc_import", [_i32, _i32, _i32, _sz, C.POINTER(_pp)])
dvla_mc_add_device = _proto("dvla_mc_add_device", [_vp, _i32])
dvla_mc_bind = _proto("dvla_mc_bind", [_vp, _i32, C.POINTER(_pp)])
dvla_mc_map = _proto("dvla_mc_map", [_vp, _i32, C.POINTER(_pp)])
dvla_mc_destroy = _proto("dvla_mc_destroy", [_vp])
dvla_mc_broadcast = _proto("dvla_mc_broadcast", [_vp, _vp, _i64, _vp, C.c_uint32, _i32, _vp,
                                                 _vp])
dvla_mc_allreduce_f32 = _proto("dvla_mc_allreduce_f32", [
    _vp, _i64, _i32, _i32, _vp, _vp, C.c_uint32, C.c_float, _i32, _vp, C.c_uint64, _vp, _vp])
dvla_mc_wait = _proto("dvla_mc_wait", [_vp, C.c_uint32, C.c_uint64, _vp, _vp])

# ---------------------------------------------- Gaussian head / MLP policy
dvla_mlp_forward = _proto("dvla_mlp_forward", [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32,
                                               _vp, _vp])
dvla_chunk_log_prob = _proto("dvla_chunk_log_prob", [_vp, _vp, _vp, _i64, _i32, _vp, _vp])
dvla_policy_backward_workspace_bytes = _proto("dvla_policy_backward_workspace_bytes",
                                              [_i64, _i32, _i32], _sz)
dvla_policy_backward = _proto("dvla_policy_backward", [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                                       _i64, _i32, _i32, _i32, _vp, _vp, _vp])
dvla_gauss_loss_workspace_bytes = _proto("dvla_gauss_loss_workspace_bytes", [_i64, _i64, _i64],
                                         _sz)
dvla_gauss_loss_fwd_bwd = _proto("dvla_gauss_loss_fwd_bwd", [
    _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _f64, _f64, _f64, _vp, _vp, _vp,
    _vp, _vp, _sz, _vp])
dvla_gauss_head_backward = _proto("dvla_gauss_head_backward", [_vp, _vp, _vp, _vp, _i64, _i32,
                                                               _vp, _vp, _vp])
# ------------------------------------------------------------ optimizer
dvla_adam_step = _proto("dvla_adam_step", [_vp, _vp, _vp, _vp, _i64, _i64, _f64, _f64, _f64,
                                           _f64, _vp])
dvla_grad_norm_workspace_bytes = _proto("dvla_grad_norm_workspace_bytes", [_i64], _sz)
dvla_grad_norm = _proto("dvla_grad_norm", [_vp, _i64, _f64, _vp, _vp, _vp, _vp])
dvla_f32_nonfinite = _proto("dvla_f32_nonfinite", [_vp, _i64, _vp, _vp])
dvla_grad_norm_f32 = _proto("dvla_grad_norm_f32", [_vp, _i64, _f64, _vp, _vp, _vp, _vp])
dvla_grad_sumsq_f32 = _proto("dvla_grad_sumsq_f32", [_vp, _i64, _f64, _vp, _vp, _vp, _vp])
dvla_grad_sum_f32 = _proto("dvla_grad_sum_f32", [C.POINTER(_vp), _i32, _i64, _i64, _f64, _vp, _vp,
                                                   _vp, _vp, _vp])
dvla_adam_tail_f32 = _proto("dvla_adam_tail_f32", [
    _vp, _vp, _vp, _vp, _i64, _i64, _f64, _f64, _f64, _f64, _f64, _vp, _f64, _vp, _vp, _vp, _vp])
dvla_adam_tail_f32_bcast = _proto("dvla_adam_tail_f32_bcast", [
    _vp, _vp, _vp, _vp, _i64, _i64, _f64, _f64, _f64, _f64, _f64, _vp, _f64, _vp, _vp,
    C.POINTER(_vp), _i32, _vp, _vp])
dvla_loss_status = _proto("dvla_loss_status", [_vp, _vp, _vp])

# ---------------------------------------------------- rollout token sampling
dvla_token_sample = _proto("dvla_token_sample", [_vp, _i32, _i64, _i64, _i64, C.c_uint64,
                                                 C.c_uint64, _vp, _vp, _vp, _vp, _vp])
