"""Learner-gradient reduce-scatter over NVLink peer memory, overlapped with
the gradient GEMM (ZeRO-1 path of TrainerWorker.update).

Reference: GradReducer.reduce / reduce_serial (runtime.py:569-637) -- every
node's gradient travels as an f32 frame (runtime.py:590), the frames are
summed in f64 in node order and divided by the node count (runtime.py:618-
627); TrainerWorker.update divides by w and reduces (runtime.py:788).  SURVEY
§8 a10 / e.

B200 design.  The head gradient dW = dl^T x is a row-blocked GEMM: block j
(the rows rank j owns under ZeRO-1) is computed by every rank and needed,
summed, only by rank j.  Each rank computes its gradient in a few large
GEMMs ordered so that its own block comes last (TrainerWorker's plans: the
other half of the blocks, then its own half; or the peer runs, then its
own block); as soon as a GEMM is in HBM a copy engine pushes each of its
peer blocks over NVLink into the owner's staging slot for r -- no SMs are
taken from the GEMMs, and the last GEMM hides the earlier pushes.
Then one HBM-bound kernel on rank j sums its own block and the N - 1 staged
ones in f64 in NODE order (the reference's arithmetic, deterministic) and
computes the block's sum of squares in the same pass
(`dvla_grad_sum_f32`).  Per GPU the links carry (N - 1) / N of the gradient
each way, the same as a ring reduce-scatter, but in one step with no
SM-driven pipeline.

The bf16 weight all-gather after the optimizer tail either rides in the
tail kernel itself (it stores its rows into every peer's working copy
through the mappings, `peer_rows`, then `gather_finish(by_kernel=True)`)
or goes as copy-engine pushes per optimizer chunk (`gather_chunk`).

Synchronisation is stream-ordered, with one u32 flag per peer and direction
in device memory (the same CUDA IPC + stream memory-operation protocol as
the copy-engine replication chain, replicate.SplitReplicator):
  ready[p] on rank j  = step e  after p's push into j's slot p landed
                                (written by p's copy stream)
  ack[j]   on rank p  = step e  after j's sum read its slot p
                                (written by j's trainer stream)
so a push of step e + 1 never overwrites a slot before the step-e sum read
it, and a GEMM of step e + 1 never overwrites a block before its step-e push
(a local event).  The flag waits are bounded (`dvla_wait_flags_u32`, one
polling warp per wait): a peer that stops arriving sets an error word after
the timeout instead of hanging the stream.
"""

from __future__ import annotations

import ctypes as C
import os

from .core import UsageError


class PeerGradExchange:
    """Reduce-scatter of `gin` ([N, cs] f32, this rank's GEMM output; row j
    goes to rank j) into rank r's sum, over CUDA IPC + copy engines.

    Collective construction: every rank of `group` calls it (one process
    per GPU).  `stage_pool` (a device Pool, e.g. MODEL_COMPUTE) holds the
    N x cs f32 staging slots; per step:
        begin(s)                       # before anything writes gin
        GEMMs into gin's blocks, the own block last (order(): one per block);
        pushed(j, s) for each peer block j as soon as it is complete
        finish(s, out, n_norm, div, sumsq, nonfinite, workspace)
    """

    def __init__(self, gin, stage_pool, group=None, wbuf=None, err=None,
                 timeout_s: float | None = None):
        import torch
        import torch.distributed as dist

        from . import _lib
        from .replicate import _gather_by_rank, _open_ipc, _PoolRegion, _Slab
        if gin.dim() != 2 or gin.dtype != torch.float32 or not gin.is_contiguous():
            raise UsageError("gin must be a contiguous [N, cs] f32 tensor")
        self.N, self.cs = gin.shape
        if (self.cs * 4) % 16 or gin.data_ptr() % 16:
            raise UsageError("gradient blocks must be 16-byte aligned")
        self.rank = dist.get_rank(group)
        if dist.get_world_size(group) != self.N:
            raise UsageError("gin needs one block per rank of the group")
        if self.N > 32:
            raise UsageError("at most 32 ranks per exchange")
        self.gin = gin
        self.dev = gin.device
        self.group = group
        N, cs, r = self.N, self.cs, self.rank
        self._opened = []
        self.peer = {}   # group rank -> (stage base of that rank, flags base of that rank)
        self.peer_w = {}  # group rank -> that rank's wbuf
        ranks = (list(range(dist.get_world_size())) if group is None
                 else dist.get_process_group_ranks(group))

        def agree(err):
            """Every setup phase ends with an agreement: a failure on any rank
            (out of pool memory, no IPC / peer access ...) raises the same
            NativeError on every rank, so the caller can fall back together
            instead of leaving the others in a collective."""
            errs = [e for e in _gather_by_rank(err, group).values() if e]
            if errs:
                self.close()
                raise _lib.NativeError("peer gradient exchange setup failed: "
                                       + "; ".join(errs))

        err = None
        try:
            if os.environ.get("DVLA_TEST_EXCHANGE_FAIL_RANK") == str(r):
                raise RuntimeError("injected failure (DVLA_TEST_EXCHANGE_FAIL_RANK)")
            self.stage = _PoolRegion(stage_pool, N * cs * 4)
            self.stage_t = self.stage.t[: N * cs * 4].view(torch.float32).view(N, cs)
            # u32 words: ready[0:N) | ack[32:32+N) | weights landed[64:64+N) |
            # scalar-sum flags [96:96+N) | scalar-max flags [128:128+N); bytes
            # [1024, 2048): f64 scalar-sum slots [N][k]; [2048, 2560): u32 max slots
            self.flags = _Slab(4096, self.dev.index)
            self.flags.t.zero_()
            torch.cuda.synchronize(self.dev)
            # the bf16 weights all-gathered after the optimizer tail
            # (optional): [N * nloc] in the same pool, rank p's rows at p * nloc
            self.wbuf = wbuf
            w_off = None
            if wbuf is not None:
                slab = stage_pool._slab
                w_off = wbuf.data_ptr() - slab.ptr
                if (wbuf.dtype != torch.bfloat16 or wbuf.numel() % N or w_off < 0
                        or w_off + wbuf.numel() * 2 > slab.nbytes):
                    raise UsageError("wbuf must be an [N * nloc] bf16 view inside the pool")
                self.nloc = wbuf.numel() // N
            mine = (self.dev.index, self.stage.ipc(), self.stage.offset, self.flags.ipc(), w_off)
        except Exception as e:  # noqa: BLE001 - agreed on below
            err, mine = f"rank {r}: {e}", None
        agree(err)
        allh = _gather_by_rank(mine, group)
        try:
            # peer access for the copy engines and the kernels' peer stores
            # (IPC mappings enable it lazily too)
            for g in ranks:
                if allh[g][0] != self.dev.index:
                    _lib.dvla_enable_peer_access(self.dev.index, allh[g][0])
            for p, g in enumerate(ranks):
                if p == r:
                    continue
                base = _open_ipc(allh[g][1])
                self._opened.append(base)
                fl = _open_ipc(allh[g][3])
                self._opened.append(fl)
                self.peer[p] = (base + allh[g][2], fl)
                if allh[g][4] is not None:
                    self.peer_w[p] = base + allh[g][4]
        except Exception as e:  # noqa: BLE001 - agreed on below
            err = f"rank {r}: {e}"
        agree(err)
        self.copy_stream = torch.cuda.Stream(device=self.dev, priority=-1)
        # bounded waits: a peer that stops arriving sets this word (device
        # int32; the caller's, e.g. a slot of TrainerWorker's flags that is
        # max-reduced and read after its one sync) instead of hanging
        self.err = err if err is not None else torch.zeros(1, dtype=torch.int32,
                                                           device=self.dev)
        if timeout_s is None:
            timeout_s = float(os.environ.get("DVLA_EXCHANGE_TIMEOUT_S", "120"))
        self.timeout_ns = int(timeout_s * 1e9)
        self.peer_mask = ((1 << N) - 1) & ~(1 << r)
        self.ev_block = [torch.cuda.Event() for _ in range(N)]
        self.ev_pushed = None     # the previous step's last push (gin reusable)
        self.epoch = 0
        self._npushed = 0
        # peer tables of the scalar reductions (the own entry unused)
        self._sum_slots = (C.c_void_p * N)(*[self.peer[p][1] + 1024 if p != r else 0
                                              for p in range(N)])
        self._sum_flags = (C.c_void_p * N)(*[self.peer[p][1] + 4 * 96 if p != r else 0
                                              for p in range(N)])
        self._max_slots = (C.c_void_p * N)(*[self.peer[p][1] + 2048 if p != r else 0
                                              for p in range(N)])
        self._max_flags = (C.c_void_p * N)(*[self.peer[p][1] + 4 * 128 if p != r else 0
                                              for p in range(N)])
        self.srcs = (C.c_void_p * N)(*[
            (gin[r].data_ptr() if p == r else self.stage_t[p].data_ptr()) for p in range(N)])
        dist.barrier(group=group)

    def order(self):
        """Block order for this rank's GEMM: every peer's block first, in
        the order (r + 1, r + 2, ...), its own block last."""
        return [(self.rank + k) % self.N for k in range(1, self.N + 1)]

    def begin(self, stream):
        """Start of a step on the trainer stream: the previous step's pushes
        must have read gin before the GEMMs overwrite it, and (copy stream)
        every peer's previous sum must have read its slot for this rank
        before this step's pushes overwrite it."""
        self.epoch += 1
        self._npushed = 0
        if self.ev_pushed is not None:
            stream.wait_event(self.ev_pushed)
        if self.epoch > 1:
            self._wait(32, self.epoch - 1, self.copy_stream)

    def _wait(self, word: int, target: int, stream):
        from . import _lib
        _lib.check(_lib.dvla_wait_flags_u32(self.flags.ptr + 4 * word, self.peer_mask, target,
                                            self.timeout_ns, self.err.data_ptr(),
                                            stream.cuda_stream), "dvla_wait_flags_u32")

    def pushed(self, j: int, stream):
        """Block j of gin is complete on `stream`: push it to rank j."""
        from . import _lib
        if j == self.rank:
            return
        e, c = self.epoch, self.copy_stream
        self.ev_block[j].record(stream)
        c.wait_event(self.ev_block[j])
        stage_j, flags_j = self.peer[j]
        _lib.check(_lib.dvla_memcpy_async(stage_j + self.rank * self.cs * 4,
                                          self.gin[j].data_ptr(), self.cs * 4, c.cuda_stream),
                   "dvla_memcpy_async")
        _lib.check(_lib.dvla_stream_write_u32(flags_j + 4 * self.rank, e, c.cuda_stream),
                   "dvla_stream_write_u32")
        self._npushed += 1
        if self._npushed == self.N - 1:   # the last peer block of the step
            ev = __import__("torch").cuda.Event()
            ev.record(c)
            self.ev_pushed = ev

    def finish(self, stream, out, n_norm: int, div: float, sumsq, nonfinite, workspace):
        """On `stream` (after this rank's own block): wait for every peer's
        push, out = f32(f64 sum of the N blocks in node order), *sumsq =
        sum of (out[:n_norm] / div)^2, then release the slots to the peers."""
        from . import _lib
        e, r = self.epoch, self.rank
        self._wait(0, e, stream)
        if out.numel() != self.cs or out.dtype != self.gin.dtype:
            raise UsageError("the reduce-scatter output is one f32 block")
        _lib.check(_lib.dvla_grad_sum_f32(self.srcs, self.N, int(n_norm), self.cs, float(div),
                                          out.data_ptr(),
                                          sumsq.data_ptr(), nonfinite.data_ptr(),
                                          workspace.data_ptr(), stream.cuda_stream),
                   "dvla_grad_sum_f32")
        for p in range(self.N):
            if p != r:
                _lib.check(_lib.dvla_stream_write_u32(self.peer[p][1] + 4 * (32 + r), e,
                                                      stream.cuda_stream),
                           "dvla_stream_write_u32")

    def gather_chunk(self, lo: int, hi: int, stream):
        """Elements [lo, hi) of this rank's weight rows are final on
        `stream` (an optimizer-tail chunk): a copy engine pushes them into
        every peer's wbuf while the next chunk is being stepped."""
        from . import _lib
        if self.wbuf is None:
            raise UsageError("this exchange has no weight buffer")
        if hi <= lo:
            return
        c = self.copy_stream
        ev = __import__("torch").cuda.Event()
        ev.record(stream)
        c.wait_event(ev)
        off = (self.rank * self.nloc + lo) * 2
        src = self.wbuf.data_ptr() + off
        for k in range(1, self.N):
            p = (self.rank + k) % self.N
            _lib.check(_lib.dvla_memcpy_async(self.peer_w[p] + off, src, (hi - lo) * 2,
                                              c.cuda_stream), "dvla_memcpy_async")

    def peer_rows(self, lo: int = 0):
        """Device pointers (a ctypes array, one per peer) to element `lo` of
        this rank's rows inside every peer's wbuf: the targets of an
        optimizer tail that stores its bf16 rows straight into the peers
        (dvla_adam_tail_f32_bcast)."""
        if self.wbuf is None:
            raise UsageError("this exchange has no weight buffer")
        off = (self.rank * self.nloc + lo) * 2
        peers = [p for p in range(self.N) if p != self.rank]
        return (C.c_void_p * max(len(peers), 1))(*[self.peer_w[p] + off for p in peers])

    def gather_finish(self, stream, by_kernel: bool = False):
        """After the last gather_chunk (or, by_kernel, after the optimizer
        tail that stored the rows into the peers itself, on `stream`): tell
        every peer this rank's rows landed, then make `stream` wait until
        this rank's pushes are done and every peer's rows have landed here."""
        from . import _lib
        torch = __import__("torch")
        e, r = self.epoch, self.rank
        c = stream if by_kernel else self.copy_stream
        for p in range(self.N):
            if p != r:
                _lib.check(_lib.dvla_stream_write_u32(self.peer[p][1] + 4 * (64 + r), e,
                                                      c.cuda_stream), "dvla_stream_write_u32")
        if not by_kernel:
            ev = torch.cuda.Event()
            ev.record(c)
            stream.wait_event(ev)
        self._wait(64, e, stream)

    def reduce_sum_f64(self, vals, stream):
        """vals (device f64, k <= 4 values) <- their sum over the ranks in
        rank order, identical on every rank (in place; once per step)."""
        self._reduce(0, vals, 1024, 96, self._sum_slots, self._sum_flags, stream)

    def reduce_max_u32(self, vals, stream):
        """vals (device int32/uint32 flags, k <= 4) <- their max over the
        ranks (in place; once per step)."""
        self._reduce(1, vals, 2048, 128, self._max_slots, self._max_flags, stream)

    def _reduce(self, kind, vals, slot_off, flag_word, peer_slots, peer_flags, stream):
        from . import _lib
        k = vals.numel()
        _lib.check(_lib.dvla_peer_reduce(kind, vals.data_ptr(), k, peer_slots, peer_flags,
                                         self.rank, self.N, self.flags.ptr + slot_off,
                                         self.flags.ptr + 4 * flag_word, self.epoch,
                                         self.timeout_ns, self.err.data_ptr(), vals.data_ptr(),
                                         stream.cuda_stream), "dvla_peer_reduce")

    def check(self):
        """Host side, after the stream has been synchronised: raise if a
        bounded wait timed out."""
        if int(self.err.item()):
            from ._lib import ReplicationTimeout
            raise ReplicationTimeout(f"rank {self.rank}: peer gradient exchange timed out")

    def close(self):
        import torch

        from .replicate import _close_ipc
        torch.cuda.synchronize(self.dev)
        for p in getattr(self, "_opened", []):
            _close_ipc(p)
        self._opened = []
        self.peer = {}
