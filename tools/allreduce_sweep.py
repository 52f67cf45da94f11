"""NCCL all-reduce busbw for learner-gradient buckets (run under torchrun)."""
import os, sys
import torch
import torch.distributed as dist
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
w = dist.get_world_size()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("MODE") == "nvls":
    from paper_2605_13276_b200.replicate import McAllReduce
    for nbytes in (64 << 20, 256 << 20, 1 << 30):
        ar = McAllReduce(nbytes // 4, ctas=int(os.environ.get("CTAS", "0")))
        ar.buf.fill_(1.0)
        for _ in range(3):
            ar.allreduce()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        for _ in range(10):
            ar.allreduce()
        e1.record()
        torch.cuda.synchronize()
        ar.check()
        t = torch.tensor([e0.elapsed_time(e1) / 10], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if dist.get_rank() == 0:
            bus = nbytes * 2 * (w - 1) / w / (t.item() / 1e3) / 1e9
            print(f"nvls     {nbytes >> 20:5d} MB float32   {t.item():7.3f} ms busbw {bus:6.1f} GB/s",
                  flush=True)
        dist.barrier()
        ar.close()
    dist.destroy_process_group()
    sys.exit(0)
for nbytes in (64 << 20, 256 << 20, 1 << 30):
    for dt in (torch.float32, torch.bfloat16):
        g = torch.ones(nbytes // torch.tensor([], dtype=dt).element_size(), dtype=dt, device="cuda")
        for _ in range(3):
            dist.all_reduce(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        for _ in range(10):
            dist.all_reduce(g)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if dist.get_rank() == 0:
            bus = nbytes * 2 * (w - 1) / w / (t.item() / 1e3) / 1e9
            print(f"{os.environ.get('NCCL_ALGO', 'default'):8s} {nbytes >> 20:5d} MB {str(dt)[6:]:9s} "
                  f"{t.item():7.3f} ms busbw {bus:6.1f} GB/s", flush=True)
dist.destroy_process_group()
