"""Switch-multicast replication sweep (run under torch.distributed.run):
GB/s per receiver for CTA counts at S bytes, max over ranks, bit-exact check."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    from paper_2605_13276_b200.replicate import McReplicator, bytes_equal
    S = int(float(os.environ.get("MC_BYTES", "6.6e9"))) // 16 * 16
    src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                        generator=torch.Generator(device="cuda").manual_seed(7))
    rep = McReplicator(S, n_buffers=1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    v = 0
    for ctas in [int(x) for x in os.environ.get("MC_CTAS", "148,296,592,1184").split(",")]:
        rep.ctas = ctas
        ts = []
        for it in range(4):
            dist.barrier()
            torch.cuda.synchronize()
            e0.record()
            rep.broadcast(src, v)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ts.append(t.item())
            v += 1
        rep.check()
        ok = bytes_equal(src, rep.replica(v - 1))[0] == 0
        okt = torch.tensor([0.0 if ok else 1.0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MAX)
        ms = sorted(ts[1:])[1]
        if rank == 0:
            print(f"world {dist.get_world_size()} S {S/1e9:.2f} GB ctas {ctas:5d}: {ms:8.3f} ms "
                  f"{S / ms / 1e6:7.1f} GB/s per receiver  bit_exact={okt.item() == 0}", flush=True)
    dist.barrier()
    rep.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
