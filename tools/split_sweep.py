"""C3 layout: two learners each source half of the weights to the replicas
(run under torch.distributed.run on 4 GPUs: learners 0, 1; replicas 2, 3),
vs one learner chaining the whole region.  GB/s per receiver, bit-exact."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2605_13276_b200.replicate import ChainReplicator, SplitReplicator, bytes_equal
    S = int(float(os.environ.get("S", "6.6e9"))) // 32 * 32
    src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(9))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, iters=4):
        ts = []
        for it in range(iters + 1):
            dist.barrier()
            torch.cuda.synchronize()
            e0.record()
            fn(it)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if it:
                ts.append(t.item())
        return sorted(ts)[len(ts) // 2]

    def ok_all(ok):
        t = torch.tensor([0.0 if ok else 1.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() == 0.0

    chains = [[0, 2, 3], [1, 3, 2]]
    engines = os.environ.get("ENGINES", "sm,ce_head,ce").split(",")
    for engine in engines:
        rep = SplitReplicator(S, chains, n_buffers=1, ctas_per_hop=64, engine=engine)
        ms = timed(lambda it: rep.broadcast(src if rank in (0, 1) else None, it))
        rep.check()
        ok = ok_all(rank < 2 or bytes_equal(src, rep.replica(0))[0] == 0)
        rep.close()
        if rank == 0:
            print(f"split 2 learners -> 2 replicas, engine {engine}: {ms:.3f} ms, "
                  f"{S / ms / 1e6:.1f} GB/s per replica, bit_exact={ok}", flush=True)
        del rep
    # one learner, chain 0 -> 2 -> 3 (replicas only), the 1-source baseline
    sub = dist.new_group([0, 2, 3])
    if rank in (0, 2, 3):
        rep = ChainReplicator(S, ranks=[0, 2, 3], n_buffers=1, group=sub)
    dist.barrier()

    def one(it):
        if rank in (0, 2, 3):
            rep.broadcast(src, it)
    ms = timed(one)
    if rank in (0, 2, 3):
        rep.check()
        ok = rank == 0 or bytes_equal(src, rep.replica(0))[0] == 0
    else:
        ok = True
    ok = ok_all(ok)
    if rank == 0:
        print(f"single learner chain 0 -> 2 -> 3: {ms:.3f} ms, {S / ms / 1e6:.1f} GB/s per replica, "
              f"bit_exact={ok}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
