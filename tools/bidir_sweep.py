"""4 GPUs: one source, the region split in two halves flowing around the
chain in opposite directions (0->1->2->3 and 0->3->2->1), vs one chain.
GB/s per receiver, bit-exact (run under torch.distributed.run)."""
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
                        generator=torch.Generator(device="cuda").manual_seed(3))
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

    ring = list(range(world))
    chains = [ring, [0] + ring[:0:-1]]
    for ctas in (64, 96):
        rep = SplitReplicator(S, chains, n_buffers=1, ctas_per_hop=ctas)
        ms = timed(lambda it: rep.broadcast(src, it))
        rep.check()
        ok = rank == 0 or bytes_equal(src, rep.replica(0))[0] == 0
        rep.close()
        if rank == 0:
            print(f"bidirectional {chains}, {ctas} CTAs/hop: {S / ms / 1e6:.1f} GB/s per receiver "
                  f"(rank0 check {ok})", flush=True)
        del rep
    rep = ChainReplicator(S, n_buffers=1)
    ms = timed(lambda it: rep.broadcast(src, it))
    rep.check()
    rep.close()
    if rank == 0:
        print(f"single chain {ring}: {S / ms / 1e6:.1f} GB/s per receiver", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
