"""C5 replication size sweep (SURVEY §8 d): one source to N-1 receivers for
S in {0.1 .. 100} GB, TMA chain vs NVSwitch multicast vs copy-engine fan-out.
GB/s per receiver = S / t(last receiver complete), CUDA events, max over
ranks, bit-exact check on every receiver.  Run under torch.distributed.run."""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def timed(fn, iters=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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


def fingerprint(t):
    """Position-weighted 64-bit checksum of a byte region, in 1 GB pieces."""
    acc = 0
    v = t.view(torch.int64) if t.numel() % 8 == 0 else t[: t.numel() // 8 * 8].view(torch.int64)
    piece = 1 << 27
    for a in range(0, v.numel(), piece):
        w = v[a:a + piece]
        idx = torch.arange(a, a + w.numel(), device=w.device, dtype=torch.int64)
        acc = (acc + int((w * (idx * 2654435761 + 1)).sum().item())) & ((1 << 64) - 1)
    return acc


def same_as_root(t_or_none):
    """Every receiver's region fingerprint equals the root's source one."""
    fp = fingerprint(t_or_none)
    allfp = [None] * dist.get_world_size()
    dist.all_gather_object(allfp, fp)
    return all(x == allfp[0] for x in allfp)


def all_ok(ok):
    t = torch.tensor([0.0 if ok else 1.0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() == 0.0


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2605_13276_b200.replicate import ChainReplicator, McReplicator, multicast_supported
    sizes = [float(x) for x in os.environ.get("SIZES", "0.1,0.316,1,3.16,10,31.6,100").split(",")]
    mc_ok = multicast_supported()
    if rank == 0:
        print(f"# world {world}: GB/s per receiver (bit-exact: every receiver's position-weighted checksum equals the source's)", flush=True)
        print(f"# {'S (GB)':>8} {'chain':>8} {'multicast':>10} {'CE fan-out':>11}", flush=True)
    for sg in sizes:
        S = int(sg * 1e9) // 16 * 16
        src = None
        if rank == 0:
            src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                                generator=torch.Generator(device="cuda").manual_seed(int(sg * 1000)))
        rep = ChainReplicator(S, n_buffers=1, ctas_per_hop=128)
        ms = timed(lambda it: rep.broadcast(src, it))
        rep.check()
        ok = same_as_root(src if rank == 0 else rep.replica(0))
        chain = (S / ms / 1e6) if ok else float("nan")
        ce_ms = timed(lambda it: rep.ce_fanout(src, 0))
        ce = S / ce_ms / 1e6
        rep.close()
        del rep
        gc.collect()
        torch.cuda.synchronize()
        mc = float("nan")
        fits = torch.tensor([1.0 if torch.cuda.mem_get_info()[0] > S + (4 << 30) else 0.0],
                            device="cuda")
        dist.all_reduce(fits, op=dist.ReduceOp.MIN)
        if mc_ok and fits.item() == 1.0:
            mrep = McReplicator(S, n_buffers=1)
            mms = timed(lambda it: mrep.broadcast(src, it))
            mrep.check()
            ok = same_as_root(mrep.replica(0))
            mc = (S / mms / 1e6) if ok else float("nan")
            dist.barrier()
            mrep.close()
            del mrep
            gc.collect()
        del src
        torch.cuda.empty_cache()
        if rank == 0:
            print(f"  {sg:8.3f} {chain:8.1f} {mc:10.1f} {ce:11.1f}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
