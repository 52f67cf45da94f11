"""Per-rank body of tests/test_multigpu.py (run under torch.distributed.run).

Checks, on N >= 2 GPUs over NCCL/NVLink: (1) the cross-process TMA chain
broadcast is bit-exact on every receiver for two versions (double buffer),
and so is the switch-multicast (NVLS) broadcast where the box supports it;
(2) GradReducer's NCCL mean equals the reference semantics; (3) the
group-sharded token loss gives every rank its own shard's result; (4) the
swimlane runs one closed loop per GPU with NCCL gradient reduction."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    if rank == 0:
        print("PEER_CHANNEL_OK", flush=True)

    # (2) gradient mean over NCCL, exact mode vs host arithmetic
    g = torch.full((1000,), float(rank + 1), dtype=torch.float64, device="cuda") / 3.0
    out = GradReducer(world, exact=True).reduce(g.clone())
    want = sum(float(np.float32((r + 1) / 3.0)) for r in range(world)) / world
    assert torch.allclose(out, torch.full_like(out, want), rtol=1e-15), (out[0].item(), want)

    # (4) swimlane, topology replication with NCCL grad mean
    cfg = SwimlaneConfig(n_groups=2, group_size=4, tokens=8, vocab=1024, action_bins=256,
                         hidden=64, epochs=3, seed=11)
    res = run_swimlane(cfg)
    assert res.counters["updates"] == 3
    dist.barrier()
    if rank == 0:
        print("MULTIGPU_OK", world, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
