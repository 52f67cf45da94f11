"""Per-rank body of tests/test_multigpu.py (run under torch.distributed.run).

Checks, on N >= 2 GPUs over NCCL/NVLink: (1) the cross-process TMA chain
broadcast is bit-exact on every receiver for two versions (double buffer),
and so is the switch-multicast (NVLS) broadcast where the box supports it;
(2) GradReducer's NCCL mean equals the reference semantics; (3) the
group-sharded token loss gives every rank its own shard's oracle result and
the NCCL-averaged f32 head gradient equals the full-batch gradient; (4) the
swimlane runs one closed loop per GPU with NCCL gradient reduction and ends
with bitwise-identical weights on every rank."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def _sharded_learner_step(rank, world):
    """(3): the full batch (4 groups per rank, same seed everywhere) is
    sharded by group; each rank's TokenLoss on its shard matches the f64
    oracle run on that shard alone; the head gradient dW_r = dl_r^T x_r (f32
    GEMM output) is all-reduced by NCCL through TrainerWorker's bucketed
    path and divided by N; it equals (a) the f64 mean of every rank's own
    product (f32 accumulation only, 1e-5) and (b) the single-GPU full-batch
    gradient (reference runtime.py:775-788: mean of equal shards = full
    batch; 1e-3 for N a power of two, 5e-3 otherwise: the two bf16 dlogits
    roundings differ)."""
    from oracle import grpo_oracle as O
    from oracle.check import assert_dlogits_close
    from paper_2605_13276_b200 import grpo
    from paper_2605_13276_b200.runtime import GradReducer
    k, G, T, V, H = 4, 4, 8, 2048, 64
    n_groups = k * world
    R = n_groups * G * T
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(77)
    feats = (torch.randn(R, H, device=dev, generator=g)).to(torch.bfloat16)
    W = (torch.randn(V, H, device=dev, generator=g) * 0.3).to(torch.bfloat16)
    logits = feats @ W.t()
    tokens = torch.randint(0, V, (R,), device=dev, generator=g, dtype=torch.int32)
    rewards = torch.rand(n_groups * G, device=dev, generator=g)
    cfg = grpo.GrpoConfig(group_size=G)
    full = grpo.TokenLoss(n_groups, G, 1, T, V, cfg, dtype=torch.bfloat16, device=dev)
    full.launch(logits, tokens, torch.zeros(n_groups * G, device=dev), rewards, None)
    blp = (full.lp_chunk + (torch.rand(full.lp_chunk.shape, device=dev, generator=g,
                                       dtype=torch.float64) - 0.5) * 0.2).float()
    rows = slice(rank * k * G * T, (rank + 1) * k * G * T)
    trj = slice(rank * k * G, (rank + 1) * k * G)
    ids = np.arange(rank * k, (rank + 1) * k)
    tl = grpo.TokenLoss(k, G, 1, T, V, cfg, dtype=torch.bfloat16, device=dev)
    tl.set_groups(ids)
    dl = torch.empty(k * G * T, V, dtype=torch.bfloat16, device=dev)
    tl.launch(logits[rows].contiguous(), tokens[rows].contiguous(), blp[trj].contiguous(),
              rewards[trj].contiguous(), dl)
    st = tl.stats(rewards[trj])
    torch.cuda.synchronize()
    x = logits[rows].float().cpu().numpy().reshape(k, G, 1, T, V)
    oloss, odl, ost = O.grpo_token_grad(x, tokens[rows].cpu().numpy().reshape(k, G, 1, T),
                                        blp[trj].cpu().numpy().reshape(k, G, 1),
                                        rewards[trj].cpu().numpy().reshape(k, G), ids)
    scale = float(np.abs(ost["coeff"]).mean())
    assert abs(st["loss"] - oloss) <= 1e-5 * max(abs(oloss), scale), (rank, st["loss"], oloss)
    np.testing.assert_allclose(tl.lp_chunk.cpu().numpy(), ost["lp_chunk"].reshape(-1),
                               rtol=0, atol=1e-5)
    assert st["group_ids"] == ost["group_ids"] == ids.tolist()
    assert_dlogits_close(dl.float().cpu().numpy(), odl.reshape(-1, V), 1e-2)
    # NCCL mean of the f32 head gradients, bucketed as TrainerWorker.update
    n = V * H
    gbuf = torch.zeros(n + 1, dtype=torch.float32, device=dev)
    red = GradReducer(world)
    assert red.overlappable(gbuf)
    step = -(-V // 4)
    works = []
    for j in range(4):
        a, b = j * step, min(V, (j + 1) * step)
        torch.mm(dl[:, a:b].t(), feats[rows], out_dtype=torch.float32,
                 out=gbuf[:n].view(V, H)[a:b])
        works.append(red.reduce_async(gbuf[a * H:(b * H if b < V else n + 1)]))
    for w in works:
        w.wait()
    mean = gbuf[:n].double() / world
    own = (dl.double().t() @ feats[rows].double()).reshape(-1)
    allown = [torch.empty_like(own) for _ in range(world)]
    dist.all_gather(allown, own)
    want = sum(allown) / world
    assert float((mean - want).norm() / want.norm()) <= 1e-5, rank
    assert float(gbuf[n]) == 0.0
    if rank == 0:
        dl_full = torch.empty(R, V, dtype=torch.bfloat16, device=dev)
        full.launch(logits, tokens, blp, rewards, dl_full)
        gfull = (dl_full.double().t() @ feats.double()).reshape(-1)
        # the shards' dlogits carry w_r = N w_full: for N a power of two the
        # bf16 roundings match the full batch's; otherwise each element is
        # rounded independently twice (RMS 2^-9 / sqrt(3) each)
        tol = 1e-3 if (world & (world - 1)) == 0 else 5e-3
        assert float((mean - gfull).norm() / gfull.norm()) <= tol
    dist.barrier()


def _zero1_matches_full_gradient(rank, world):
    from paper_2605_13276_b200.grpo import GroupBatch
    from paper_2605_13276_b200.pools import Pool, PoolKind
    from paper_2605_13276_b200.runtime import GradReducer, SwimlaneConfig, TrainerWorker
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1003, action_bins=256,
                         hidden=64, seed=31, lr=1e-3)
    dev = torch.device("cuda", torch.cuda.current_device())
    G, T, H, V = cfg.group_size, cfg.tokens, cfg.hidden, cfg.vocab
    n_traj = cfg.n_groups * G

    def batches(step):
        g = torch.Generator(device=dev).manual_seed(1000 * step + rank)
        feats = torch.randn(n_traj, 1, H, device=dev, generator=g).to(torch.bfloat16)
        toks = torch.randint(0, V, (n_traj, 1, T), device=dev, generator=g, dtype=torch.int32)
        blp = (torch.randn(n_traj, 1, device=dev, generator=g) - 60.0).float()
        rw = torch.rand(n_traj, device=dev, generator=g)
        return [GroupBatch(group_id=rank * cfg.n_groups + k, horizon=T, chunk=T,
                           obs=feats[k * G:(k + 1) * G], actions=toks[k * G:(k + 1) * G],
                           behavior_log_prob=blp[k * G:(k + 1) * G], rewards=rw[k * G:(k + 1) * G],
                           behavior_version=0, tokens=toks[k * G:(k + 1) * G])
                for k in range(cfg.n_groups)]

    out = {}
    for name, red in (("zero1", GradReducer(world)),
                      ("zero1_ce_gather", GradReducer(world)),
                      ("zero1_runs", GradReducer(world)),
                      ("zero1_nccl", GradReducer(world, scatter="nccl")),
                      ("full", GradReducer(world, exact=True))):
        pool = Pool(PoolKind.MODEL_COMPUTE, 64 << 20, device=dev)
        if name == "zero1_runs":   # the other GEMM plan of the peer exchange
            os.environ["DVLA_GRAD_PLAN"] = "runs"
        if name == "zero1_ce_gather":   # the all-gather by copy-engine pushes
            os.environ["DVLA_GATHER_MODE"] = "ce"
        tr = TrainerWorker(cfg, rank, pool, red, torch.cuda.Stream(device=dev), dev)
        os.environ.pop("DVLA_GRAD_PLAN", None)
        os.environ.pop("DVLA_GATHER_MODE", None)
        assert tr.sharded == name.startswith("zero1")
        if tr.sharded:   # the default reduce-scatter is the peer exchange
            assert (tr.exchange is not None) == (name != "zero1_nccl"), name
        norms = [tr.update(batches(step))["grad_norm"] for step in range(3)]
        torch.cuda.synchronize()
        out[name] = (tr.policy.w16.clone(), tr.policy.master.clone(), tr.policy)
        out[name + "_norms"] = norms
        tr.close()
    # the global gradient norm (peer: block sums of squares reduced in rank
    # order over NVLink; NCCL's all-reduce; the exact path's full gradient)
    # agrees on every rank and across the paths
    allnorms = [None] * world
    dist.all_gather_object(allnorms, out["zero1_norms"])
    assert all(nm == allnorms[0] for nm in allnorms), allnorms
    for a_, b_ in zip(out["zero1_norms"], out["full_norms"]):
        assert abs(a_ - b_) <= 1e-5 * abs(b_), (a_, b_)
    for a_, b_ in zip(out["zero1_norms"], out["zero1_nccl_norms"]):
        assert abs(a_ - b_) <= 1e-6 * abs(b_), (a_, b_)
    w_z, m_z, pol_z = out["zero1"]
    w_f, m_f, _ = out["full"]
    # peer exchange (node-order f64 sum) vs NCCL reduce-scatter (f32 ring
    # sum): the same update up to the sum's rounding
    w_n, m_n, _ = out["zero1_nccl"]
    # the optimizer tail storing its bf16 rows into the peers (default) and
    # the copy-engine pushes deliver the same bytes
    w_c, m_c, _ = out["zero1_ce_gather"]
    assert torch.equal(w_c.view(torch.int16), w_z.view(torch.int16))
    assert torch.equal(m_c, m_z)
    w_u, m_u, _ = out["zero1_runs"]
    du = (m_z - m_u).abs()
    assert float((du > 1e-6).float().mean()) < 1e-3, float((du > 1e-6).float().mean())
    dn = (m_z - m_n).abs()
    assert float((dn > 1e-6).float().mean()) < 1e-3, float((dn > 1e-6).float().mean())
    assert float((w_z.view(torch.int16) == w_n.view(torch.int16)).float().mean()) > 0.99
    # this rank's master block of the sharded learner vs the same rows of the
    # full one; the bf16 working copies everywhere
    Vs = pol_z.Vs
    rows = slice(rank * Vs * H, min(V, (rank + 1) * Vs) * H)
    mf = m_f[rows]
    mz = m_z[: mf.numel()]
    diff = (mz - mf).abs()
    # f32 vs f64 sums of the frames: equal up to rounding, except where Adam's
    # first steps flip with a near-zero gradient (|delta| <= 2 lr per step)
    assert float((diff > 1e-6).float().mean()) < 1e-3, float((diff > 1e-6).float().mean())
    assert float(diff.max()) <= 4 * cfg.lr + 1e-6
    same = (w_z.view(torch.int16) == w_f.view(torch.int16)).float().mean()
    assert float(same) > 0.99, float(same)
    assert bool((pol_z.w16pad[V * H:] == 0).all())          # padded rows stay zero
    dist.barrier()


def _exchange_scalars(rank, world):
    """The exchange's scalar reductions: f64 sums in rank order and u32
    maxima, identical on every rank, over several epochs."""
    from paper_2605_13276_b200.exchange import PeerGradExchange
    from paper_2605_13276_b200.pools import Pool, PoolKind
    dev = torch.device("cuda", torch.cuda.current_device())
    pool = Pool(PoolKind.MODEL_COMPUTE, (world + 1) * 4096 * 4 + (1 << 20), device=dev)
    ex = PeerGradExchange(torch.zeros(world, 4096, device=dev), pool)
    s = torch.cuda.current_stream()
    for step in range(1, 4):
        ex.epoch += 1
        v = torch.tensor([rank + 0.1 * step, 1e-300 * (rank + 1)], dtype=torch.float64,
                         device=dev)
        f = torch.tensor([7 * step if rank == world - 1 else 0, rank, 0], dtype=torch.int32,
                         device=dev)
        ex.reduce_sum_f64(v, s)
        ex.reduce_max_u32(f, s)
        torch.cuda.synchronize()
        want0 = 0.0
        for r in range(world):
            want0 += r + 0.1 * step
        assert v[0].item() == want0, (v[0].item(), want0)
        want1 = 0.0   # left to right (Python's sum() compensates since 3.12)
        for r in range(world):
            want1 += 1e-300 * (r + 1)
        assert v[1].item() == want1, (v.tolist(), want1, step)
        assert f.tolist() == [7 * step, world - 1, 0], f.tolist()
        # (in the learner the next step's writes are ordered after this
        # read by the exchange's own flags; here a barrier stands in)
        dist.barrier()
    ex.check()
    dist.barrier()
    ex.close()
    dist.barrier()


def _exchange_setup_failure_falls_back_to_nccl(rank, world):
    """A setup failure on one rank (injected on the last one) makes every
    learner fall back to NCCL's collectives together, and the update runs."""
    from paper_2605_13276_b200.pools import Pool, PoolKind
    from paper_2605_13276_b200.runtime import GradReducer, SwimlaneConfig, TrainerWorker
    from paper_2605_13276_b200.grpo import GroupBatch
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=512, action_bins=256,
                         hidden=64, seed=5)
    dev = torch.device("cuda", torch.cuda.current_device())
    os.environ["DVLA_TEST_EXCHANGE_FAIL_RANK"] = str(world - 1)
    try:
        red = GradReducer(world)
        tr = TrainerWorker(cfg, rank, Pool(PoolKind.MODEL_COMPUTE, 64 << 20, device=dev), red,
                           torch.cuda.Stream(device=dev), dev)
    finally:
        os.environ.pop("DVLA_TEST_EXCHANGE_FAIL_RANK", None)
    assert tr.sharded and tr.exchange is None and red.scatter == "nccl"
    G, T, H, V = cfg.group_size, cfg.tokens, cfg.hidden, cfg.vocab
    g = torch.Generator(device=dev).manual_seed(rank)
    n = cfg.n_groups * G
    feats = torch.randn(n, 1, H, device=dev, generator=g).to(torch.bfloat16)
    toks = torch.randint(0, V, (n, 1, T), device=dev, generator=g, dtype=torch.int32)
    blp = (torch.randn(n, 1, device=dev, generator=g) - 40.0).float()
    rw = torch.rand(n, device=dev, generator=g)
    batches = [GroupBatch(group_id=rank * cfg.n_groups + k, horizon=T, chunk=T,
                          obs=feats[k * G:(k + 1) * G], actions=toks[k * G:(k + 1) * G],
                          behavior_log_prob=blp[k * G:(k + 1) * G],
                          rewards=rw[k * G:(k + 1) * G], behavior_version=0,
                          tokens=toks[k * G:(k + 1) * G]) for k in range(cfg.n_groups)]
    st = tr.update(batches)
    assert st["version"] == 1 and np.isfinite(st["grad_norm"])
    tr.close()
    dist.barrier()


def _exchange_timeout(rank, world):
    """The peer exchange's waits are bounded: when the other learners never
    push, rank 0's sum wait times out, sets the error word and the stream
    goes on (ReplicationTimeout on check(), no hung stream)."""
    from paper_2605_13276_b200._lib import ReplicationTimeout
    from paper_2605_13276_b200.exchange import PeerGradExchange
    from paper_2605_13276_b200.pools import Pool, PoolKind
    dev = torch.device("cuda", torch.cuda.current_device())
    cs = 4096
    pool = Pool(PoolKind.MODEL_COMPUTE, (world + 1) * cs * 4 * 2 + (1 << 20), device=dev)
    gin = torch.ones(world, cs, device=dev)
    ex = PeerGradExchange(gin, pool, timeout_s=0.5)
    s = torch.cuda.current_stream()
    if rank == 0:
        out = torch.empty(cs, device=dev)
        sq = torch.zeros(1, dtype=torch.float64, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        import paper_2605_13276_b200._lib as L
        ws = torch.empty(L.dvla_grad_norm_workspace_bytes(cs), dtype=torch.uint8, device=dev)
        ex.begin(s)
        for j in ex.order():
            ex.pushed(j, s)
        ex.finish(s, out, cs, 1.0, sq, bad, ws)
        torch.cuda.synchronize()
        try:
            ex.check()
            raise AssertionError("the exchange wait did not time out")
        except ReplicationTimeout:
            pass
    dist.barrier()
    ex.close()
    dist.barrier()


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    opts = dist.ProcessGroupNCCL.Options()
    opts.is_high_priority_stream = True
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2605_13276_b200.replicate import (ChainReplicator, McReplicator, bytes_equal,
                                                 multicast_supported)
    from paper_2605_13276_b200.runtime import GradReducer, SwimlaneConfig, run_swimlane

    # (1) chain replication, 2 versions, odd size
    S = 123_456_784
    rep = ChainReplicator(S, chunk_bytes=4 << 20, ctas_per_hop=16)
    for v in (0, 1, 2):
        src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(100 + v))
        rep.broadcast(src, v)
        torch.cuda.synchronize()
        dist.barrier()
        rep.check()
        if rank > 0:
            assert bytes_equal(src, rep.replica(v)) == (0, -1), (rank, v)
    rep.close()

    # (1a') replica regions placed by the receivers' MODEL_COMPUTE pools
    from paper_2605_13276_b200.pools import Pool, PoolKind
    pool = None if rank == 0 else Pool(PoolKind.MODEL_COMPUTE, 2 * S + (1 << 20), device="cuda")
    prep = ChainReplicator(S, chunk_bytes=4 << 20, ctas_per_hop=16, pool=pool)
    for v in (0, 1):
        src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(150 + v))
        prep.broadcast(src, v)
        torch.cuda.synchronize()
        dist.barrier()
        prep.check()
        if rank > 0:
            reg = prep.replica(v)
            assert bytes_equal(src, reg) == (0, -1), ("pool", rank, v)
            base = pool.data.data_ptr()
            assert base <= reg.data_ptr() < base + pool.capacity  # inside the pool's slab
    dist.barrier()
    prep.close()

    # (1b) switch-multicast (NVLS) replication, 3 versions through 2 buffers
    if multicast_supported():
        mrep = McReplicator(S, n_buffers=2)
        for v in (0, 1, 2):
            src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                                generator=torch.Generator(device="cuda").manual_seed(200 + v))
            dist.barrier()
            mrep.broadcast(src, v)
            torch.cuda.synchronize()
            dist.barrier()
            mrep.check()
            assert bytes_equal(src, mrep.replica(v)) == (0, -1), ("mc", rank, v)
        dist.barrier()
        mrep.close()
        if rank == 0:
            print("MULTICAST_OK", flush=True)
        # (1c) switch-reduced all-reduce: exact on integer-valued f32, 3 calls
        from paper_2605_13276_b200.replicate import McAllReduce
        n = 1_000_004
        ar = McAllReduce(n)
        idx = torch.arange(n, device="cuda", dtype=torch.float32)
        for it in range(3):
            ar.buf.copy_((idx % 97) * (rank + 1) + it)
            ar.allreduce(scale=1.0)
            torch.cuda.synchronize()
            ar.check()
            want = (idx % 97) * (world * (world + 1) / 2) + it * world
            assert torch.equal(ar.buf, want), ("allreduce", rank, it)
        ar.buf.fill_(float(rank))
        ar.allreduce(scale=1.0 / world)
        torch.cuda.synchronize()
        assert torch.allclose(ar.buf, torch.full_like(ar.buf, (world - 1) / 2), rtol=1e-6)
        dist.barrier()
        ar.close()
        if rank == 0:
            print("MC_ALLREDUCE_OK", flush=True)
        # (1e) a setup failure on one rank surfaces on every rank (no hang)
        from paper_2605_13276_b200._lib import NativeError
        if rank == world - 1:
            os.environ["DVLA_TEST_MC_FAIL_RANK"] = str(rank)
        try:
            McAllReduce(1024)
            raise AssertionError("injected multicast failure did not surface")
        except NativeError as e:
            assert "injected failure" in str(e), str(e)
        os.environ.pop("DVLA_TEST_MC_FAIL_RANK", None)
        dist.barrier()

    # (1c') the size-based engine choice delivers bit-exact too
    from paper_2605_13276_b200.replicate import make_replicator
    for nb in (64 << 20, 600 << 20):
        r2 = make_replicator(nb)
        src = torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(nb % 1000))
        dist.barrier()
        r2.broadcast(src, 0)
        torch.cuda.synchronize()
        dist.barrier()
        r2.check()
        if rank > 0:
            assert bytes_equal(src, r2.replica(0)) == (0, -1), ("auto", type(r2).__name__, rank)
        dist.barrier()
        r2.close()
        del src

    # (1d) several sources, one region (C3 layout at 4 GPUs; two parts from
    # rank 0 along the same pair at 2)
    from paper_2605_13276_b200.replicate import SplitReplicator
    chains = [[0, 2, 3], [1, 3, 2]] if world >= 4 else [[0, 1], [0, 1]]
    srep = SplitReplicator(S - S % 32, chains, n_buffers=2, ctas_per_hop=16)
    heads = {c[0] for c in chains}
    receivers = {r for c in chains for r in c[1:]}
    for v in (0, 1, 2):
        src = torch.randint(0, 256, (S - S % 32,), dtype=torch.uint8, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(300 + v))
        dist.barrier()
        srep.broadcast(src if rank in heads else None, v)
        torch.cuda.synchronize()
        dist.barrier()
        srep.check()
        if rank in receivers:
            assert bytes_equal(src, srep.replica(v)) == (0, -1), ("split", rank, v)
    dist.barrier()
    srep.close()

    # (1f) trajectory batches rollout rank -> learner rank:
    # 7 batches through a 3-slot ring (wraps twice), bit-identical
    from paper_2605_13276_b200.grpo import GroupBatch
    from paper_2605_13276_b200.planes import PeerChannel

    def make_batch(gid, device):
        g = torch.Generator(device=device).manual_seed(1000 + gid)
        return GroupBatch(
            group_id=gid, horizon=8, chunk=1, behavior_version=gid // 2,
            obs=torch.randn(8, 1, 24, device=device, generator=g),
            actions=torch.randn(8, 1, 7, device=device, generator=g),
            behavior_log_prob=torch.randn(8, 1, device=device, generator=g),
            rewards=torch.randint(0, 2, (8,), device=device, generator=g).float(),
            tokens=torch.randint(0, 256, (8, 1, 56), device=device, generator=g,
                                 dtype=torch.int32))

    pc = PeerChannel(producer=0, consumer=1, slot_bytes=64 << 10, slots=3)
    if rank == 0:
        for gid in range(7):
            pc.put(make_batch(gid, "cuda"))
        torch.cuda.synchronize()
    elif rank == 1:
        for gid in range(7):
            got = pc.take()
            want = make_batch(gid, "cuda")
            assert got.group_id == gid and got.behavior_version == gid // 2
            for f in ("obs", "actions", "behavior_log_prob", "rewards", "tokens"):
                assert torch.equal(getattr(got, f), getattr(want, f)), (f, gid)
        torch.cuda.synchronize()
    dist.barrier()
    pc.close()
    # a ring of more than 64 slots (the flag slabs grow with the slot count)
    pc70 = PeerChannel(producer=0, consumer=1, slot_bytes=64 << 10, slots=70)
    if rank == 0:
        for gid in range(75):
            pc70.put(make_batch(gid, "cuda"))
        torch.cuda.synchronize()
    elif rank == 1:
        for gid in range(75):
            got = pc70.take()
            assert got.group_id == gid and torch.equal(got.tokens, make_batch(gid, "cuda").tokens)
        torch.cuda.synchronize()
    dist.barrier()
    pc70.close()
    if rank == 0:
        print("PEER_CHANNEL_OK", flush=True)

    # (2) gradient mean over NCCL, exact mode vs host arithmetic
    g = torch.full((1000,), float(rank + 1), dtype=torch.float64, device="cuda") / 3.0
    out = GradReducer(world, exact=True).reduce(g.clone())
    want = sum(float(np.float32((r + 1) / 3.0)) for r in range(world)) / world
    assert torch.allclose(out, torch.full_like(out, want), rtol=1e-15), (out[0].item(), want)

    # (3) group-sharded token loss + NCCL-averaged head gradient
    _sharded_learner_step(rank, world)
    if rank == 0:
        print("SHARDED_LOSS_OK", flush=True)

    # (3b) the ZeRO-1 learner (reduce-scatter / all-gather) against the
    # whole-gradient path (GradReducer(exact=True): f64 all-reduce of the f32
    # frames, full master weights on every rank) on a vocabulary that does
    # not split evenly over the ranks (padded row blocks)
    _zero1_matches_full_gradient(rank, world)
    if rank == 0:
        print("ZERO1_OK", flush=True)
    _exchange_scalars(rank, world)
    _exchange_setup_failure_falls_back_to_nccl(rank, world)
    _exchange_timeout(rank, world)
    if rank == 0:
        print("EXCHANGE_TIMEOUT_OK", flush=True)

    # (4) swimlane, topology replication with NCCL grad mean: every rank
    # ends with bitwise-identical master weights and bf16 working copies
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                         hidden=64, epochs=3, seed=11)
    res = run_swimlane(cfg)
    assert res.counters["updates"] == 3
    pol = res.policy
    t = pol.w16.reshape(-1)
    allw = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(allw, t.contiguous())
    for r in range(1, world):
        assert torch.equal(allw[0].view(torch.int16), allw[r].view(torch.int16)), ("w16", r)
    # ZeRO-1: each rank steps its own row block of the master weights; the
    # all-gathered bf16 block is that block's round-to-nearest
    assert pol.N == world and pol.rank == rank
    assert torch.equal(pol.w16_own, pol.master.to(torch.bfloat16))
    assert res.counters["updates"] == 3 and pol.step == 3
    if rank == 0:
        print("SWIMLANE_WEIGHTS_EQUAL_OK", flush=True)
    dist.barrier()
    if rank == 0:
        print("MULTIGPU_OK", world, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
