"""Dual-pool VRAM arenas: a long-lived MODEL_COMPUTE pool beside an
epoch-recycled ENV_AUX pool, each one device slab.

Same API and placement decisions as reference pkg/src/dvla/pools.py
(PoolKind :23-26, AllocFailure :29-36, PoolUsageError :39-40, PoolHandle
:43-49, PoolStats :52-62, Pool :72-212, pool_create :215-216,
random_workload :219-231, churn_script :234-273, run_churn :281-315).  The
bookkeeping is the C++ arena behind the C-ABI (csrc/arena.cpp); the backing
store is a cudaMalloc'd slab (so regions can be shared with peer GPUs over
CUDA IPC for weight replication) exposed to torch as zero-copy views.

On B200 the MODEL_COMPUTE pool holds parameters, gradients, optimizer
moments and the double-buffered replica regions the weight plane writes
into; ENV_AUX holds rollout staging and activations and is reset wholesale
at every epoch boundary.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .core import ConfigError, UsageError


class PoolKind(Enum):
    MODEL_COMPUTE = "model_compute"
    ENV_AUX = "env_aux"
    UNIFIED_BASELINE = "unified_baseline"


_KIND_CODE = {PoolKind.MODEL_COMPUTE: 0, PoolKind.ENV_AUX: 1, PoolKind.UNIFIED_BASELINE: 2}


class AllocFailure(Exception):
    """No free extent fits the request; the caller decides the fallback."""

    def __init__(self, kind: PoolKind, size: int, align: int):
        super().__init__(f"{kind.value} pool cannot place {size} bytes @align {align}")
        self.kind = kind
        self.size = size
        self.align = align


class PoolUsageError(UsageError):
    """Double free, stale generation, or lifecycle misuse."""


@dataclass(frozen=True)
class PoolHandle:
    pool_id: int
    offset: int
    size: int
    generation: int
    serial: int


@dataclass(frozen=True)
class PoolStats:
    live_bytes: int
    total_free: int
    largest_free_block: int
    fragmentation: float  # 1 - largest/total_free; 0 when total_free == 0
    failed_allocs: int
    alloc_count: int
    free_count: int
    churn_bytes: int
    generation: int


class _DeviceSlab:
    """A cudaMalloc'd slab exposed through __cuda_array_interface__."""

    def __init__(self, nbytes: int, device: int):
        from . import _lib
        ptr = C.c_void_p()
        _lib.check(_lib.dvla_dev_alloc(device, nbytes, C.byref(ptr)), "dvla_dev_alloc")
        self.ptr = ptr.value
        self.nbytes = nbytes
        self.device = device
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3,
            "strides": None,
        }

    def __del__(self):
        try:
            from . import _lib
            _lib.dvla_dev_free(self.ptr)
        except Exception:
            pass


def _torch_dtype(dtype):
    import torch
    if isinstance(dtype, torch.dtype):
        return dtype
    m = {np.dtype(np.uint8): torch.uint8, np.dtype(np.float32): torch.float32,
         np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
         np.dtype(np.int64): torch.int64, np.dtype(np.float16): torch.float16}
    try:
        return m[np.dtype(dtype)]
    except (KeyError, TypeError):
        raise UsageError(f"unsupported view dtype {dtype!r}") from None


class Pool:
    """Single-owner arena over one slab (device by default; `device="cpu"`
    backs it with host memory for tooling and CPU tests)."""

    def __init__(self, kind: PoolKind, capacity: int, device=None):
        from . import _lib
        import torch
        if capacity <= 0:
            raise ConfigError(f"pool capacity must be > 0, got {capacity}")
        self.kind = kind
        self.capacity = int(capacity)
        h = C.c_void_p()
        pid = C.c_int64()
        _lib.check(_lib.dvla_arena_create(_KIND_CODE[kind], self.capacity, C.byref(h),
                                          C.byref(pid)), "dvla_arena_create")
        self._arena = h
        self.pool_id = int(pid.value)
        if device is None:
            device = "cuda" if torch.cuda.is_available() else "cpu"
        dev = torch.device(device)
        if dev.type == "cuda":
            idx = dev.index if dev.index is not None else torch.cuda.current_device()
            self._slab = _DeviceSlab(self.capacity, idx)
            self.data = torch.as_tensor(self._slab, device=torch.device("cuda", idx))
        else:
            self._slab = None
            self.data = torch.zeros(self.capacity, dtype=torch.uint8)
        self.device = self.data.device

    def __del__(self):
        try:
            from . import _lib
            _lib.dvla_arena_destroy(self._arena)
        except Exception:
            pass

    # -------------------------------------------------------------- handles
    def alloc(self, size: int, align: int = 1) -> PoolHandle:
        """First-fit allocate; raises AllocFailure when nothing fits."""
        from . import _lib
        off, serial, gen = C.c_int64(), C.c_int64(), C.c_int64()
        st = _lib.dvla_arena_alloc(self._arena, int(size), int(align), C.byref(off),
                                   C.byref(serial), C.byref(gen))
        if st == _lib.ERR_ALLOC_FAILURE:
            raise AllocFailure(self.kind, size, align)
        _lib.check(st, "dvla_arena_alloc")
        return PoolHandle(pool_id=self.pool_id, offset=off.value, size=int(size),
                          generation=gen.value, serial=serial.value)

    def free(self, handle: PoolHandle) -> None:
        from . import _lib
        _lib.check(_lib.dvla_arena_free(self._arena, handle.pool_id, handle.offset, handle.size,
                                        handle.generation, handle.serial), "dvla_arena_free")

    def epoch_reset(self) -> None:
        """Invalidate every handle and return to one free extent; ENV_AUX only."""
        from . import _lib
        _lib.check(_lib.dvla_arena_epoch_reset(self._arena), "dvla_arena_epoch_reset")

    @property
    def generation(self) -> int:
        return self.stats().generation

    def _live(self, handle: PoolHandle) -> bool:
        from . import _lib
        out = C.c_int()
        _lib.check(_lib.dvla_arena_is_live(self._arena, handle.generation, handle.serial,
                                           C.byref(out)), "dvla_arena_is_live")
        return bool(out.value) and handle.pool_id == self.pool_id

    def view(self, handle: PoolHandle, dtype=None, count: int | None = None):
        """Zero-copy torch view of a live allocation (device or host)."""
        import torch
        if not self._live(handle):
            raise PoolUsageError(f"view of dead or stale handle {handle}")
        td = torch.uint8 if dtype is None else _torch_dtype(dtype)
        item = torch.empty((), dtype=td).element_size()
        n = handle.size // item if count is None else int(count)
        if n * item > handle.size:
            raise PoolUsageError(f"view of {n}x{dtype} exceeds {handle.size} bytes")
        raw = self.data[handle.offset:handle.offset + n * item]
        return raw.view(td) if n else raw[:0].view(td)

    def stats(self) -> PoolStats:
        from . import _lib
        out = (C.c_int64 * 9)()
        _lib.check(_lib.dvla_arena_stats(self._arena, out), "dvla_arena_stats")
        total, largest = int(out[1]), int(out[2])
        frag = 0.0 if total == 0 else 1.0 - largest / total
        return PoolStats(live_bytes=int(out[0]), total_free=total, largest_free_block=largest,
                         fragmentation=frag, failed_allocs=int(out[3]), alloc_count=int(out[4]),
                         free_count=int(out[5]), churn_bytes=int(out[6]), generation=int(out[7]))

    def run_trace(self, is_alloc, size, align, pick):
        """Batched trace through the native arena (alloc_trace_run contract)."""
        return arena_trace(self.capacity, is_alloc, size, align, pick)


class TorchArena:
    """Torch's own allocations in an ENV_AUX pool.

    A torch.cuda.MemPool over a CUDAPluggableAllocator whose segments the
    pool's first-fit arena places in its device slab (dvla_torch_alloc /
    dvla_torch_free, csrc/arena.cpp): inside `with arena:` every tensor the
    current thread allocates on the pool's device (activations,
    concatenations, sampling outputs) lands in the recycled pool instead of
    torch's private cudaMalloc segments.  Torch caches and sub-allocates
    within its segments, so the pool is not epoch-reset while bound (the
    C-ABI refuses it); close() returns the segments and unbinds.  Several
    lane threads may use one arena at once (one MemPool per thread, all
    drawing from the arena)."""

    def __init__(self, pool: "Pool"):
        import torch

        from . import _lib
        if pool.kind is not PoolKind.ENV_AUX or pool._slab is None:
            raise PoolUsageError("torch allocations go to an ENV_AUX device pool")
        self.pool = pool
        self.device = pool.data.device.index
        _lib.check(_lib.dvla_torch_pool_bind(self.device, pool._arena, pool.data.data_ptr()),
                   "dvla_torch_pool_bind")
        self._alloc = torch.cuda.memory.CUDAPluggableAllocator(
            str(_lib._LIB_PATH), "dvla_torch_alloc", "dvla_torch_free")
        # one MemPool per thread (torch records one thread into a pool at a
        # time); every one of them draws its segments from this arena
        self._pools: dict = {}
        self._lock = threading.Lock()
        self._ctx = threading.local()

    @property
    def mempool(self):
        import torch
        tid = threading.get_ident()
        with self._lock:
            mp = self._pools.get(tid)
            if mp is None:
                mp = self._pools[tid] = torch.cuda.MemPool(self._alloc.allocator())
        return mp

    def __enter__(self):
        import torch
        ctx = torch.cuda.use_mem_pool(self.mempool, device=self.device)
        ctx.__enter__()
        stack = getattr(self._ctx, "stack", None) or []
        stack.append(ctx)
        self._ctx.stack = stack
        return self

    def __exit__(self, *exc):
        return self._ctx.stack.pop().__exit__(*exc)

    _shared: dict = {}

    @classmethod
    def shared(cls, device, nbytes: int) -> "TorchArena":
        """The process's torch arena on `device` (one binding per device),
        created with an ENV_AUX pool of `nbytes` on first use."""
        import torch
        idx = torch.device(device).index
        if idx is None:
            idx = torch.cuda.current_device()
        a = cls._shared.get(idx)
        if a is None:
            a = cls(Pool(PoolKind.ENV_AUX, int(nbytes), device=torch.device("cuda", idx)))
            cls._shared[idx] = a
        return a

    def holds(self, t) -> bool:
        """True when tensor t's storage lies in the pool's slab."""
        base = self.pool.data.data_ptr()
        return base <= t.data_ptr() < base + self.pool.capacity

    def close(self):
        """Release torch's segments back to the arena and unbind (every
        tensor allocated inside must be gone)."""
        import gc

        import torch

        from . import _lib
        torch.cuda.synchronize(self.device)
        with self._lock:
            self._pools.clear()      # ~MemPool releases the pool; empty_cache then
        gc.collect()                 # hands its segments back through dvla_torch_free
        torch.cuda.empty_cache()
        _lib.check(_lib.dvla_torch_pool_bind(self.device, None, None), "dvla_torch_pool_bind")


def arena_trace(capacity: int, is_alloc, size, align, pick):
    """kernels.alloc_trace_run replacement: (out_ok, out_off, final triple)."""
    from . import _lib
    a = np.ascontiguousarray(is_alloc, dtype=np.uint8)
    s = np.ascontiguousarray(size, dtype=np.int64)
    al = np.ascontiguousarray(align, dtype=np.int64)
    pk = np.ascontiguousarray(pick, dtype=np.uint64)
    n = a.shape[0]
    ok = np.zeros(n, dtype=np.uint8)
    off = np.zeros(n, dtype=np.int64)
    fin = np.zeros(3, dtype=np.int64)
    _lib.check(_lib.dvla_arena_trace(int(capacity), n, a.ctypes.data, s.ctypes.data,
                                     al.ctypes.data, pk.ctypes.data, ok.ctypes.data,
                                     off.ctypes.data, fin.ctypes.data), "dvla_arena_trace")
    return ok, off, tuple(int(x) for x in fin)


def pool_create(kind: PoolKind, capacity: int, device=None) -> Pool:
    return Pool(kind, capacity, device=device)


def random_workload(seed: int, n_ops: int, capacity: int):
    """Deterministic alloc/free trace arrays (reference pools.py:219-231):
    60% allocs, log-uniform sizes 16..4096, aligns from {1, 8, 64, 256},
    free picks as u63 draws resolved modulo the live count."""
    g = np.random.Generator(np.random.Philox(key=seed))
    is_alloc = (g.random(n_ops) < 0.6).astype(np.uint8)
    size = np.exp(g.uniform(np.log(16), np.log(4096), n_ops)).astype(np.int64)
    align = np.choose(g.integers(0, 4, n_ops), [1, 8, 64, 256]).astype(np.int64)
    pick = g.integers(0, 1 << 63, n_ops).astype(np.uint64)
    return is_alloc, size, align, pick


def churn_script(n_rounds: int = 7):
    """The scripted scratch/model interleaving of reference pools.py:234-273:
    each round one strictly growing scratch buffer, from round 2 two small
    ephemeral scratch blocks, one model block of the scratch size, then the
    previous round's big scratch is released; finally a 128 KiB model
    request.  Returns (ops, model_request)."""
    ops: list[tuple] = []
    births = 0
    prev = None
    for r in range(n_rounds):
        big = 104448 + 2048 * r
        ops.append(("alloc_scratch", big))
        mine = births
        births += 1
        if r >= 2:
            ops.append(("alloc_scratch", 3072))
            ops.append(("alloc_scratch", 5120))
            births += 2
            ops.append(("alloc_model", big))
            ops.append(("free_scratch", births - 2))
            ops.append(("free_scratch", births - 1))
        else:
            ops.append(("alloc_model", big))
        if prev is not None:
            ops.append(("free_scratch", prev))
        prev = mine
    ops.append(("free_scratch", prev))
    return ops, 131072


UNIFIED_CAPACITY = (1 << 20) + (1 << 19)
MODEL_CAPACITY = 1 << 20
ENV_CAPACITY = 1 << 19


def run_churn(unified: bool, device=None):
    """Replay churn_script on one unified pool or the dual split; returns
    (final model request failed, {"model": stats[, "env": stats]})."""
    if unified:
        model = scratch = Pool(PoolKind.UNIFIED_BASELINE, UNIFIED_CAPACITY, device=device)
    else:
        model = Pool(PoolKind.MODEL_COMPUTE, MODEL_CAPACITY, device=device)
        scratch = Pool(PoolKind.ENV_AUX, ENV_CAPACITY, device=device)
    ops, request = churn_script()
    handles: dict[int, PoolHandle] = {}
    birth = 0
    for kind, arg in ops:
        if kind == "alloc_scratch":
            try:
                handles[birth] = scratch.alloc(arg, align=64)
            except AllocFailure:
                pass
            birth += 1
        elif kind == "free_scratch":
            h = handles.pop(arg, None)
            if h is not None:
                scratch.free(h)
        else:
            try:
                model.alloc(arg, align=256)
            except AllocFailure:
                pass
    try:
        model.alloc(request, align=256)
        failed = False
    except AllocFailure:
        failed = True
    stats = {"model": model.stats()}
    if not unified:
        stats["env"] = scratch.stats()
    return failed, stats
