"""Weight snapshots and learner -> replica replication on B200.

B200 replacement of the reference weight plane's data path:
  core.snapshot_from_params (core.py:120-129)  -> device_snapshot (fused copy
      + isfinite into a MODEL_COMPUTE region, csrc/replicate.cu)
  ControlPlane.broadcast + Transport WIRE + wire weight frames
      (planes.py:294-321, 101-128; wire.py:144-147, 227-237)
      -> a chunked, pipelined TMA chain over NVLink into every replica's
         pre-allocated region (ChainReplicator, LocalChain)
  messages_equal on parameter bytes (wire.py:279-281) -> bytes_equal

Process model: one process per GPU (torchrun).  Each rank owns its replica
region(s) and a per-chunk flag array in device slabs; CUDA IPC handles are
exchanged once over torch.distributed, after which a broadcast is one kernel
per rank: the root streams its parameters into the first receiver, every
receiver forwards each chunk to the next as soon as it landed, and the last
receiver just waits for its flags.  n_buffers = staleness_limit + 1 replica
regions per receiver give the latest-wins mailbox its double buffer.
"""

from __future__ import annotations

import ctypes as C

from .core import ConfigError, ParamSnapshot, UsageError

_DTYPE_CODE = None


def _torch():
    import torch
    return torch


def _code(t) -> int:
    torch = _torch()
    from . import _lib
    return {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16, torch.float64: _lib.F64}.get(
        t.dtype, _lib.U8)


def _stream_ptr(stream=None):
    torch = _torch()
    return (stream or torch.cuda.current_stream()).cuda_stream


def device_snapshot(params, version: int, out=None, stream=None,
                    verified: bool = False) -> ParamSnapshot:
    """snapshot_from_params for a device tensor: fused copy + isfinite.

    Raises ConfigError("non-finite parameter at flat index {i}") exactly as
    the reference (core.py:123-125).  `out` may be a pool region view of at
    least params.nbytes bytes (same dtype or uint8).  The copy runs on
    `stream` (default: current); the check synchronises that stream.
    verified=True: the caller has already established that every parameter
    is finite (the optimizer tail's flag, runtime.TrainerWorker) -- no host
    synchronisation; the snapshot's `ready` event marks when its bytes are
    valid."""
    from . import _lib
    torch = _torch()
    if version < 0:
        raise ConfigError(f"snapshot version must be >= 0, got {version}")
    src = params.detach().reshape(-1)
    if not src.is_contiguous():
        src = src.contiguous()
    nbytes = src.numel() * src.element_size()
    dst = torch.empty_like(src) if out is None else out
    if dst.numel() * dst.element_size() < nbytes:
        raise UsageError(f"snapshot destination holds {dst.numel() * dst.element_size()} bytes, "
                         f"need {nbytes}")
    st = stream if stream is not None else torch.cuda.current_stream(src.device)
    with torch.cuda.device(src.device), torch.cuda.stream(st):
        bad = torch.empty(1, dtype=torch.int64, device=src.device)
        _lib.check(_lib.dvla_snapshot_copy(src.data_ptr(), dst.data_ptr(), nbytes, _code(src),
                                           bad.data_ptr(), _stream_ptr(st)),
                   "dvla_snapshot_copy")
        ready = torch.cuda.Event()
        ready.record(st)
        if not verified:
            b = int(bad.item()) & 0xFFFFFFFFFFFFFFFF   # .item() on `st`: ordered after the copy
            if b != 0xFFFFFFFFFFFFFFFF:
                raise ConfigError(f"non-finite parameter at flat index {b}")
    if out is not None and dst.dtype != src.dtype:
        dst = dst[:nbytes].view(src.dtype)
    return ParamSnapshot(version=int(version), params=dst[:src.numel()] if out is not None
                         else dst, ready=ready)


def checksum64_async(t, stream=None, first_word: int = 0):
    """Device u64[2] checksum of a tensor's bytes (dvla_checksum64_at), on
    `stream`; compare two GPUs' copies of a region without moving either.
    first_word: the tensor's 8-byte-word offset inside a larger region
    (sub-range checksums add up mod 2^64)."""
    from . import _lib
    torch = _torch()
    out = torch.empty(2, dtype=torch.int64, device=t.device)
    _lib.check(_lib.dvla_checksum64_at(t.data_ptr(), t.numel() * t.element_size(),
                                       int(first_word), out.data_ptr(), _stream_ptr(stream)),
               "dvla_checksum64_at")
    return out


def bytes_equal(a, b, stream=None) -> tuple[int, int]:
    """(number of differing 16-byte words, first differing byte or -1)."""
    from . import _lib
    torch = _torch()
    na = a.numel() * a.element_size()
    nb = b.numel() * b.element_size()
    if na != nb:
        return 1, min(na, nb)
    out = torch.empty(2, dtype=torch.int64, device=a.device)
    with torch.cuda.device(a.device):
        _lib.check(_lib.dvla_bytes_equal(a.data_ptr(), b.data_ptr(), na, out.data_ptr(),
                                         _stream_ptr(stream)), "dvla_bytes_equal")
    mism, first = (int(x) for x in out.cpu().tolist())
    return mism, (-1 if mism == 0 else first)


def _hops(specs):
    from . import _lib
    arr = (_lib.Hop * len(specs))()
    for i, (src, dst, wait, sig) in enumerate(specs):
        arr[i].src, arr[i].dst, arr[i].wait_flags, arr[i].signal_flags = src, dst, wait, sig
    return arr


def _gather_by_rank(obj, group):
    """all_gather_object over `group` (default: world), returned as a dict
    global rank -> object."""
    import torch.distributed as dist
    ranks = (list(range(dist.get_world_size())) if group is None
             else dist.get_process_group_ranks(group))
    out = [None] * len(ranks)
    dist.all_gather_object(out, obj, group=group)
    return dict(zip(ranks, out))


class _Slab:
    """Device slab (cudaMalloc) + torch view; IPC-shareable."""

    def __init__(self, nbytes: int, device: int):
        torch = _torch()
        from .pools import _DeviceSlab
        self.slab = _DeviceSlab(nbytes, device)
        self.t = torch.as_tensor(self.slab, device=torch.device("cuda", device))
        self.ptr = self.slab.ptr

    def ipc(self) -> bytes:
        from . import _lib
        buf = C.create_string_buffer(64)
        _lib.check(_lib.dvla_ipc_handle(self.ptr, buf), "dvla_ipc_handle")
        return buf.raw


class _PoolRegion:
    """A replica region inside a (MODEL_COMPUTE) pool's device slab: the
    allocator's placement, shared over IPC as (slab handle, offset)."""

    def __init__(self, pool, nbytes: int):
        if pool._slab is None:
            raise UsageError("replica regions need a device pool")
        self.pool = pool
        self.handle = pool.alloc(nbytes, align=256)
        self.t = pool.view(self.handle)
        self.ptr = self.t.data_ptr()
        self.offset = self.handle.offset

    def ipc(self) -> bytes:
        from . import _lib
        buf = C.create_string_buffer(64)
        _lib.check(_lib.dvla_ipc_handle(self.pool._slab.ptr, buf), "dvla_ipc_handle")
        return buf.raw


_IPC_OPEN = {}   # handle bytes -> [mapped pointer, references] (one mapping per process)
_IPC_PTR = {}    # mapped pointer -> handle bytes


def _open_ipc(handle: bytes) -> int:
    """Map a peer allocation (CUDA IPC).  A process may map an allocation
    only once (cudaIpcOpenMemHandle refuses a second mapping), so mappings
    are shared and reference-counted: every _open_ipc pairs with one
    _close_ipc."""
    from . import _lib
    ent = _IPC_OPEN.get(handle)
    if ent is not None:
        ent[1] += 1
        return ent[0]
    p = C.c_void_p()
    _lib.check(_lib.dvla_ipc_open(handle, C.byref(p)), "dvla_ipc_open")
    _IPC_OPEN[handle] = [p.value, 1]
    _IPC_PTR[p.value] = handle
    return p.value


def _close_ipc(ptr: int) -> None:
    from . import _lib
    handle = _IPC_PTR.get(ptr)
    if handle is None:
        _lib.dvla_ipc_close(ptr)
        return
    ent = _IPC_OPEN[handle]
    ent[1] -= 1
    if ent[1] == 0:
        del _IPC_OPEN[handle], _IPC_PTR[ptr]
        _lib.dvla_ipc_close(ptr)


class LocalChain:
    """Chain replication between regions of ONE process (one GPU, or several
    GPUs with peer access): all hops run in a single launch, so hops that
    wait on each other are co-resident by construction.  Used for the
    1-GPU parity tests and the co-located (N=1) replica."""

    def __init__(self, nbytes: int, n_dst: int, device=None, chunk_bytes: int = 8 << 20,
                 ctas_per_hop: int = 16, dsts=None):
        torch = _torch()
        if nbytes % 16:
            raise UsageError("replicated regions must be a multiple of 16 bytes")
        self.nbytes, self.n_dst = int(nbytes), int(n_dst)
        self.chunk = int(chunk_bytes)
        self.ctas = int(ctas_per_hop)
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        self.n_chunks = (self.nbytes + self.chunk - 1) // self.chunk
        self.dsts = dsts if dsts is not None else [
            torch.empty(self.nbytes, dtype=torch.uint8, device=dev) for _ in range(n_dst)]
        self.flags = torch.zeros((max(n_dst, 1), self.n_chunks), dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0

    def broadcast(self, src, stream=None, timeout_s: float = 10.0):
        """Copy src's bytes into every destination through the chain."""
        from . import _lib
        if src.numel() * src.element_size() != self.nbytes:
            raise UsageError("source size differs from the replicated region")
        self.epoch += 1
        specs = []
        prev = src.data_ptr()
        for i, d in enumerate(self.dsts):
            wait = None if i == 0 else self.flags[i - 1].data_ptr()
            specs.append((prev, d.data_ptr(), wait, self.flags[i].data_ptr()))
            prev = d.data_ptr()
        hops = _hops(specs)
        torch = _torch()
        with torch.cuda.device(self.device):
            _lib.check(_lib.dvla_replicate_chain(hops, len(specs), self.nbytes, self.chunk,
                                                 self.epoch, self.ctas, int(timeout_s * 1e9),
                                                 self.err.data_ptr(), _stream_ptr(stream)),
                       "dvla_replicate_chain")

    def check(self):
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout("replication chain flag wait timed out")


def chain_chunk_bytes(nbytes: int, ctas_per_hop: int = 128) -> int:
    """Chunk size for the TMA chain: the pipeline fill costs (hops - 1) chunk
    transfers at the per-CTA rate, so chunks shrink with the region (about 16
    chunks per CTA), within [128 KB, 1 MB] (tools/repl_sweep.py, 4 B200:
    6.6 GB -> 1 MB 680 GB/s vs 2 MB 659; 1 GB -> 256 KB 607 vs 2 MB 482)."""
    target = max(1, nbytes // (ctas_per_hop * 16))
    c = 1 << (target.bit_length() - 1)
    return int(min(max(c, 128 << 10), 1 << 20))


class ChainReplicator:
    """Cross-process chain broadcast over NVLink (one process per GPU).

    Collective construction: every rank of `ranks` (default: all) calls it.
    ranks[0] is the source; the others hold `n_buffers` replica regions of
    `nbytes` each, allocated in `pool` (the receiver's MODEL_COMPUTE pool of
    the dual-pool allocator: the weights land directly in the pre-allocated
    static region, and the pool's slab is what is IPC-shared) or, without a
    pool, in a dedicated device slab.

    engine: "sm" (default) = the TMA-staged chain kernel on every hop;
    "ce" = copy-engine hops (stream memory operations carry the flags);
    "auto" = one copy-engine peer copy for a 2-GPU team (measured 750-758
    vs 713 GB/s), the TMA chain beyond.
    """

    def __init__(self, nbytes: int, ranks=None, n_buffers: int = 2, chunk_bytes=None,
                 ctas_per_hop: int = 128, group=None, engine: str = "sm", pool=None):
        import torch.distributed as dist
        torch = _torch()
        if nbytes % 16:
            raise UsageError("replicated regions must be a multiple of 16 bytes")
        self.rank = dist.get_rank()
        world = dist.get_world_size()
        if engine not in ("auto", "sm", "ce"):
            raise UsageError(f"engine must be 'auto', 'sm' (TMA kernel) or 'ce' (copy engines), "
                             f"got {engine!r}")
        self.ranks = list(range(world)) if ranks is None else list(ranks)
        # measured on B200 (tools/repl_sweep.py): a single hop is fastest as one
        # copy-engine peer copy (758 vs 713 GB/s); longer chains need the
        # per-chunk forwarding of the TMA kernel (CE chain: 498 vs 667 at N = 4)
        if engine == "auto":
            engine = "ce" if len(self.ranks) == 2 else "sm"
        self.engine = engine
        self.nbytes, self.nb = int(nbytes), int(n_buffers)
        self.ctas = int(ctas_per_hop)
        self.chunk = int(chunk_bytes) if chunk_bytes else chain_chunk_bytes(self.nbytes, self.ctas)
        if engine == "ce" and len(self.ranks) == 2:
            self.chunk = max(16, self.nbytes)  # one copy, one flag
        self.n_chunks = (self.nbytes + self.chunk - 1) // self.chunk
        self.dev = torch.cuda.current_device()
        self.pos = self.ranks.index(self.rank) if self.rank in self.ranks else -1
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.buf = None
        self.flags = None
        self.pool_handle = None
        handles = None
        if self.pos > 0:
            if pool is not None:
                self.buf = _PoolRegion(pool, self.nb * self.nbytes)
                self.pool_handle = self.buf.handle
            else:
                self.buf = _Slab(self.nb * self.nbytes, self.dev)
            flag_bytes = ((self.nb * self.n_chunks * 4 + 255) // 256) * 256
            self.flags = _Slab(flag_bytes, self.dev)
            self.flags.t.zero_()
            torch.cuda.synchronize()
            handles = (self.buf.ipc(), getattr(self.buf, "offset", 0), self.flags.ipc())
        allh = _gather_by_rank(handles, group)
        self.next_buf = self.next_flags = None
        self._opened = []
        if 0 <= self.pos < len(self.ranks) - 1:
            nxt = self.ranks[self.pos + 1]
            bh, boff, fh = allh[nxt]
            base = _open_ipc(bh)
            self._opened.append(base)
            self.next_buf = base + boff
            self.next_flags = _open_ipc(fh)
        self.epochs = [0] * self.nb
        # root also maps every receiver region (copy-engine fan-out baseline)
        self.fan_bufs = []
        if self.pos == 0:
            for r in self.ranks[1:]:
                if r == self.ranks[1]:
                    self.fan_bufs.append(self.next_buf)
                else:
                    base = _open_ipc(allh[r][0])
                    self._opened.append(base)
                    self.fan_bufs.append(base + allh[r][1])

    def ce_fanout(self, src, version: int, stream=None):
        """Baseline: root copies into every receiver with cudaMemcpyAsync
        (copy engines, 1 -> k direct fan-out).  No flags: time it with a
        barrier + synchronize.  Root only."""
        from . import _lib
        if self.pos != 0:
            return
        off = (version % self.nb) * self.nbytes
        for p in self.fan_bufs:
            _lib.check(_lib.dvla_memcpy_async(p + off, src.data_ptr(), self.nbytes,
                                              _stream_ptr(stream)), "dvla_memcpy_async")

    def replica(self, version: int):
        """This receiver's region holding `version` (after broadcast)."""
        if self.buf is None:
            raise UsageError("the source rank holds no replica region")
        b = version % self.nb
        return self.buf.t[b * self.nbytes:(b + 1) * self.nbytes]

    def broadcast(self, src, version: int, stream=None, timeout_s: float = 30.0):
        """Enqueue this rank's hop of the chain for `version` (all ranks)."""
        from . import _lib
        if self.pos < 0:
            return
        b = version % self.nb
        epoch = version + 1
        off = b * self.nbytes
        fl_off = b * self.n_chunks * 4
        if self.pos == 0:
            if src.numel() * src.element_size() != self.nbytes:
                raise UsageError("source size differs from the replicated region")
            s_ptr, wait = src.data_ptr(), None
        else:
            s_ptr, wait = self.buf.ptr + off, self.flags.ptr + fl_off
        if self.engine == "ce":
            nxt = self.next_buf is not None
            _lib.check(_lib.dvla_replicate_hop_ce(
                s_ptr if nxt else None, self.next_buf + off if nxt else None, wait,
                self.next_flags + fl_off if nxt else None, self.nbytes, self.chunk, epoch,
                _stream_ptr(stream)), "dvla_replicate_hop_ce")
            return
        if self.next_buf is not None:
            spec = (s_ptr, self.next_buf + off, wait, self.next_flags + fl_off)
        else:  # last receiver: wait until every chunk landed
            spec = (None, None, wait, None)
        hops = _hops([spec])
        _lib.check(_lib.dvla_replicate_chain(hops, 1, self.nbytes, self.chunk, epoch, self.ctas,
                                             int(timeout_s * 1e9), self.err.data_ptr(),
                                             _stream_ptr(stream)), "dvla_replicate_chain")

    def check(self):
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout(f"rank {self.rank}: replication flag wait timed out")

    def close(self):
        from . import _lib
        for p in set(self._opened + [self.next_flags]):
            if p:
                _close_ipc(p)
        self._opened = []
        self.next_buf = self.next_flags = None
        self.fan_bufs = []


class _CudaView:
    """__cuda_array_interface__ over memory this module does not own."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
            "strides": None,
        }


def multicast_supported(device=None) -> bool:
    """NVSwitch multicast (NVLS) + POSIX-fd handle export on `device`."""
    from . import _lib
    torch = _torch()
    out = C.c_int()
    dev = torch.cuda.current_device() if device is None else int(device)
    _lib.check(_lib.dvla_mc_supported(dev, C.byref(out)), "dvla_mc_supported")
    return bool(out.value)


class _McRegion:
    """One multicast object over `ranks` (one process per GPU) with a bound
    region of `total` bytes on every member, mapped locally; the multicast
    VA is mapped on the ranks in `map_on` (positions in `ranks`).

    Every setup phase ends with an agreement among the participating ranks:
    if any rank fails (no multicast support, no pidfd_getfd permission, out
    of memory ...), all of them release what they built and raise the same
    NativeError, so callers can fall back collectively instead of hanging."""

    def __init__(self, total: int, ranks, group, map_on):
        import os
        from . import _lib
        torch = _torch()
        import torch.distributed as dist
        self.rank = dist.get_rank()
        self.ranks = list(ranks)
        self.pos = self.ranks.index(self.rank) if self.rank in self.ranks else -1
        self.dev = torch.cuda.current_device()
        self.group = group
        n = len(self.ranks)
        self.obj = self.local = self.mc = None
        self.t = None
        self.size = 0

        def phase(fn):
            err = None
            try:
                out = fn()
            except Exception as e:  # noqa: BLE001 - reported to every rank below
                out, err = None, f"rank {self.rank}: {e}"
            errs = [e for e in _gather_by_rank(err, group).values() if e]
            if errs:
                self.close()
                raise _lib.NativeError("multicast setup failed: " + "; ".join(errs))
            return out

        def create():
            if self.pos != 0:
                return None
            fd, size, obj = C.c_int(), C.c_size_t(), C.c_void_p()
            _lib.check(_lib.dvla_mc_create(n, total, C.byref(fd), C.byref(size), C.byref(obj)),
                       "dvla_mc_create")
            self.obj = obj.value
            return (os.getpid(), fd.value, size.value)

        info = phase(create)
        pid, fd, size = _gather_by_rank(info, group)[self.ranks[0]]
        self.size = size

        def join():
            if os.environ.get("DVLA_TEST_MC_FAIL_RANK") == str(self.rank):
                raise RuntimeError("injected failure (DVLA_TEST_MC_FAIL_RANK)")
            if self.pos > 0:
                obj = C.c_void_p()
                _lib.check(_lib.dvla_mc_import(pid, fd, n, size, C.byref(obj)), "dvla_mc_import")
                self.obj = obj.value
            if self.pos >= 0:
                _lib.check(_lib.dvla_mc_add_device(self.obj, self.dev), "dvla_mc_add_device")

        phase(join)

        def bind():
            if self.pos >= 0:
                local = C.c_void_p()
                _lib.check(_lib.dvla_mc_bind(self.obj, self.dev, C.byref(local)), "dvla_mc_bind")
                self.local = local.value
                self.t = torch.as_tensor(_CudaView(self.local, self.size),
                                         device=torch.device("cuda", self.dev))

        phase(bind)

        def map_mc():
            if self.pos in map_on:
                mc = C.c_void_p()
                _lib.check(_lib.dvla_mc_map(self.obj, self.dev, C.byref(mc)), "dvla_mc_map")
                self.mc = mc.value

        phase(map_mc)

    def close(self):
        from . import _lib
        _torch().cuda.synchronize()
        self.t = None
        if self.obj:
            _lib.dvla_mc_destroy(self.obj)
        self.obj = self.local = self.mc = None


class McReplicator:
    """Cross-process switch-multicast (NVLS) broadcast (one process per GPU).

    ranks[0] writes each byte once into a multicast mapping and the NVSwitch
    replicates it into the bound region of every member; the root then
    release-stores the epoch into every member's flag through the same
    mapping and receivers acquire-poll their local copy (reference
    ControlPlane.broadcast -> WeightMailbox.deliver, planes.py:294-321,
    244-275).  Collective construction: every rank of `ranks` calls it.
    The root is a member too (its own bound copy is the cost of the team).
    """

    def __init__(self, nbytes: int, ranks=None, n_buffers: int = 2, ctas: int = 0, group=None):
        import torch.distributed as dist
        torch = _torch()
        if nbytes % 16:
            raise UsageError("replicated regions must be a multiple of 16 bytes")
        ranks = list(range(dist.get_world_size())) if ranks is None else list(ranks)
        self.nbytes, self.nb, self.ctas = int(nbytes), int(n_buffers), int(ctas)
        self.flag_off = (self.nb * self.nbytes + 255) // 256 * 256
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.done = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.region = _McRegion(self.flag_off + self.nb * 256, ranks, group, map_on=(0,))
        self.rank, self.ranks, self.pos = self.region.rank, self.region.ranks, self.region.pos
        self.size, self.local, self.mc, self.t = (self.region.size, self.region.local,
                                                  self.region.mc, self.region.t)
        if self.t is not None:
            self.t[self.flag_off:].zero_()
            torch.cuda.synchronize()
        dist.barrier(group=group)

    def replica(self, version: int):
        """This member's bound copy of `version` (after broadcast + wait)."""
        b = version % self.nb
        return self.t[b * self.nbytes:(b + 1) * self.nbytes]

    def broadcast(self, src, version: int, stream=None, timeout_s: float = 30.0):
        """Root: multicast `src`; receivers: stream-ordered wait for it."""
        from . import _lib
        if self.pos < 0:
            return
        b = version % self.nb
        epoch = version + 1
        flag = self.flag_off + b * 256
        if self.pos == 0:
            if src.numel() * src.element_size() != self.nbytes:
                raise UsageError("source size differs from the replicated region")
            _lib.check(_lib.dvla_mc_broadcast(src.data_ptr(), self.mc + b * self.nbytes,
                                              self.nbytes, self.mc + flag, epoch, self.ctas,
                                              self.done.data_ptr(), _stream_ptr(stream)),
                       "dvla_mc_broadcast")
        else:
            _lib.check(_lib.dvla_mc_wait(self.local + flag, epoch, int(timeout_s * 1e9),
                                         self.err.data_ptr(), _stream_ptr(stream)),
                       "dvla_mc_wait")

    def check(self):
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout(f"rank {self.rank}: multicast flag wait timed out")

    def close(self):
        self.t = None
        self.region.close()
        self.local = self.mc = None


class McAllReduce:
    """Switch-reduced all-reduce of an f32 buffer over NVSwitch multicast
    (one process per GPU; GradReducer's collective, runtime.py:569-637).

    `buf` is this rank's f32 [n] view inside its bound region: write the
    local gradient there, call `allreduce(scale)`, read the (scaled) sum back.
    Collective construction and calls: every rank of `ranks`."""

    def __init__(self, n: int, ranks=None, ctas: int = 0, group=None):
        import torch.distributed as dist
        torch = _torch()
        if n % 4:
            raise UsageError("the all-reduce length must be a multiple of 4 floats")
        ranks = list(range(dist.get_world_size())) if ranks is None else list(ranks)
        self.n, self.ctas = int(n), int(ctas)
        self.flag_off = (self.n * 4 + 255) // 256 * 256
        self.region = _McRegion(self.flag_off + 256, ranks, group,
                                map_on=tuple(range(len(ranks))))
        self.pos, self.world = self.region.pos, len(ranks)
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.done = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.epoch = 0
        self.buf = None
        if self.region.t is not None:
            self.region.t[self.flag_off:].zero_()
            self.buf = self.region.t[: self.n * 4].view(torch.float32)
            torch.cuda.synchronize()
        dist.barrier(group=group)

    def allreduce(self, scale: float = 1.0, stream=None, timeout_s: float = 30.0):
        from . import _lib
        if self.pos < 0:
            return
        self.epoch += 1
        r = self.region
        _lib.check(_lib.dvla_mc_allreduce_f32(
            r.mc, self.n, self.pos, self.world, r.local + self.flag_off, r.mc + self.flag_off,
            self.epoch, float(scale), self.ctas, self.done.data_ptr(), int(timeout_s * 1e9),
            self.err.data_ptr(), _stream_ptr(stream)), "dvla_mc_allreduce_f32")

    def check(self):
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout("multicast all-reduce barrier timed out")

    def close(self):
        self.buf = None
        self.region.close()


class SplitReplicator:
    """Several learners source one weight region (BASELINE config 3: two
    learners, six replicas): part i of the region (1/len(chains) of it) flows
    along chains[i], whose head holds the full source and sends only part i,
    so every receiver takes in parts over several links at once.  Every rank
    of the union of the chains constructs it and calls `broadcast`; each
    rank's hops run in one kernel launch (one CTA group per hop)."""

    def __init__(self, nbytes: int, chains, n_buffers: int = 2, chunk_bytes=None,
                 ctas_per_hop: int = 64, group=None, pool=None, engine: str = "sm"):
        import torch.distributed as dist
        torch = _torch()
        parts = len(chains)
        if parts < 1 or nbytes % (16 * parts):
            raise UsageError("the region must split into 16-byte-aligned equal parts")
        if engine not in ("sm", "ce", "ce_head"):
            raise UsageError(f"engine must be 'sm' (TMA kernel), 'ce' (copy engines) or "
                             f"'ce_head' (copy engines at the chain heads, TMA kernel on the "
                             f"forwarding hops), got {engine!r}")
        self.rank = dist.get_rank()
        self.chains = [list(c) for c in chains]
        self.nbytes, self.parts, self.nb = int(nbytes), parts, int(n_buffers)
        self.part = self.nbytes // parts
        self.ctas = int(ctas_per_hop)
        self.engine = engine
        if chunk_bytes:
            self.chunk = int(chunk_bytes)
        elif engine in ("ce", "ce_head") and all(len(c) == 2 for c in chains):
            self.chunk = self.part    # single hops: one copy-engine copy, one flag (no pipeline)
        elif engine in ("ce", "ce_head"):   # three stream operations per chunk: keep them few
            self.chunk = int(min(max(self.part // 64, 4 << 20), 64 << 20)) // 16 * 16
        else:
            self.chunk = chain_chunk_bytes(self.part, self.ctas)
        self.n_chunks = (self.part + self.chunk - 1) // self.chunk
        receivers = sorted({r for c in self.chains for r in c[1:]})
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.buf = self.flags = None
        handles = None
        if self.rank in receivers:
            # the replica ring lands in the receiver's MODEL_COMPUTE pool when
            # one is given (the pool's slab is what is IPC-shared)
            if pool is not None:
                self.buf = _PoolRegion(pool, self.nb * self.nbytes)
            else:
                self.buf = _Slab(self.nb * self.nbytes, torch.cuda.current_device())
            fb = ((self.nb * parts * self.n_chunks * 4 + 255) // 256) * 256
            self.flags = _Slab(fb, torch.cuda.current_device())
            self.flags.t.zero_()
            torch.cuda.synchronize()
            handles = (self.buf.ipc(), getattr(self.buf, "offset", 0), self.flags.ipc())
        allh = _gather_by_rank(handles, group)
        self.peer = {}
        self._opened = []
        for c in self.chains:
            if self.rank in c and c.index(self.rank) < len(c) - 1:
                nxt = c[c.index(self.rank) + 1]
                if nxt not in self.peer:
                    base = _open_ipc(allh[nxt][0])
                    self._opened.append(base)
                    self.peer[nxt] = (base + allh[nxt][1], _open_ipc(allh[nxt][2]))

    def _flag_off(self, b: int, c: int) -> int:
        return (b * self.parts + c) * self.n_chunks * 4

    def replica(self, version: int):
        if self.buf is None:
            raise UsageError("this rank holds no replica region")
        b = version % self.nb
        return self.buf.t[b * self.nbytes:(b + 1) * self.nbytes]

    def broadcast(self, src, version: int, stream=None, timeout_s: float = 30.0):
        from . import _lib
        b = version % self.nb
        epoch = version + 1
        specs = []
        heads = []   # specs of hops this rank sources as a chain head
        for c, chain in enumerate(self.chains):
            if self.rank not in chain:
                continue
            pos = chain.index(self.rank)
            off = c * self.part
            if pos == 0:
                if src is None or src.numel() * src.element_size() != self.nbytes:
                    raise UsageError("a chain head needs the full source region")
                s_ptr, wait = src.data_ptr() + off, None
            else:
                s_ptr = self.buf.ptr + b * self.nbytes + off
                wait = self.flags.ptr + self._flag_off(b, c)
            if pos < len(chain) - 1:
                nb_ptr, nf_ptr = self.peer[chain[pos + 1]]
                spec = (s_ptr, nb_ptr + b * self.nbytes + off, wait, nf_ptr + self._flag_off(b, c))
            else:
                spec = (None, None, wait, None)
            (heads if pos == 0 else specs).append(spec)
        ce = list(heads) if self.engine in ("ce", "ce_head") else []
        if self.engine == "ce":
            ce += specs
            specs = []
        elif self.engine == "sm":
            specs = heads + specs
        # copy engines: stream-ordered waits, peer copies and flag writes; no
        # SMs are held while the bytes move (the GEMMs keep them)
        for s_ptr, d_ptr, wait, nf in ce:
            _lib.check(_lib.dvla_replicate_hop_ce(s_ptr, d_ptr, wait, nf, self.part,
                                                  self.chunk, epoch, _stream_ptr(stream)),
                       "dvla_replicate_hop_ce")
        if not specs:
            return
        _lib.check(_lib.dvla_replicate_chain(_hops(specs), len(specs), self.part, self.chunk,
                                             epoch, self.ctas, int(timeout_s * 1e9),
                                             self.err.data_ptr(), _stream_ptr(stream)),
                   "dvla_replicate_chain")

    def check(self):
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout(f"rank {self.rank}: split replication timed out")

    def close(self):
        from . import _lib
        for p in self._opened:
            _close_ipc(p)
        for _, fp in self.peer.values():
            _close_ipc(fp)
        self.peer = {}
        self._opened = []


def replicate_devices(src, dsts, mode: str = "chain", chunk_bytes: int = 0, streams=None):
    """One process, several GPUs (`dvla_replicate`): copy `src` (a CUDA
    tensor) into every tensor of `dsts` (same byte size, any devices) by a
    device-to-device chain (each hop on its source GPU) or copy-engine
    fan-out.  Synchronous: returns once every destination holds the bytes;
    raises ReplicationTimeout if a chain hop timed out."""
    from . import _lib
    torch = _torch()
    n = src.numel() * src.element_size()
    if n % 16:
        raise UsageError("replicated regions must be a multiple of 16 bytes")
    for d in dsts:
        if d.numel() * d.element_size() != n or not d.is_cuda:
            raise UsageError("every destination must be a CUDA tensor of the source's size")
    k = len(dsts)
    devs = (C.c_int * max(k, 1))(*[d.device.index for d in dsts])
    ptrs = (C.c_void_p * max(k, 1))(*[d.data_ptr() for d in dsts])
    st = None
    if streams is not None:
        st = (C.c_void_p * (k + 1))(*[s.cuda_stream for s in streams])
    code = {"chain": 0, "ce": 1}[mode]
    _lib.check(_lib.dvla_replicate(src.device.index, src.data_ptr(), k, devs, ptrs, n,
                                   int(chunk_bytes), code, st), "dvla_replicate")
    for d in {src.device.index, *[t.device.index for t in dsts]}:
        torch.cuda.synchronize(d)
    bad = C.c_int()
    _lib.check(_lib.dvla_replicate_status(C.byref(bad)), "dvla_replicate_status")
    if bad.value:
        from ._lib import ReplicationTimeout
        raise ReplicationTimeout("dvla_replicate: a chain hop timed out")


def make_replicator(nbytes: int, ranks=None, n_buffers: int = 2, group=None):
    """The replication engine the C5 size sweep favours for this region and
    team (profiles/r01_replication_size_sweep_n{2,4}.txt): NVSwitch
    multicast for regions below 0.5 GB on teams of 4 or more GPUs (no
    pipeline fill), else the chain (one copy-engine hop for 2 GPUs, the TMA
    chain beyond).  Collective: every rank of `ranks` calls it."""
    import torch.distributed as dist
    team = len(ranks) if ranks is not None else dist.get_world_size()
    if team >= 4 and nbytes < 500_000_000:
        ok = _torch().tensor([1.0 if multicast_supported() else 0.0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if ok.item() == 1.0:
            from ._lib import NativeError
            try:
                return McReplicator(nbytes, ranks=ranks, n_buffers=n_buffers, group=group)
            except NativeError:
                pass  # raised on every rank alike: fall back together
    return ChainReplicator(nbytes, ranks=ranks, n_buffers=n_buffers, group=group)
