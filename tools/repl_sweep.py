"""Sweep chain-replication launch parameters (run under torchrun)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2605_13276_b200.replicate import ChainReplicator, bytes_equal

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
S = int(float(os.environ.get("S", "6.6e9"))) // 16 * 16
src = torch.randint(0, 256, (S,), dtype=torch.uint8, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(1))
res = []
CTAS = [int(x) for x in os.environ.get("CTAS", "16,32,64,128").split(",")]
CHUNKS = ([int(x) << 10 for x in os.environ["CHUNKS_KB"].split(",")] if "CHUNKS_KB" in os.environ
          else [int(x) << 20 for x in os.environ.get("CHUNKS_MB", "2,8,32").split(",")])
for ctas in CTAS:
    for chunk in CHUNKS:
        rep = ChainReplicator(S, chunk_bytes=chunk, ctas_per_hop=ctas,
                              engine=os.environ.get("ENGINE", "sm"))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for it in range(4):
            dist.barrier(); torch.cuda.synchronize()
            e0.record(); rep.broadcast(src, it); e1.record(); torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX); ts.append(t.item())
        rep.check()
        ok = rank == 0 or bytes_equal(src, rep.replica(3))[0] == 0
        rep.close(); del rep
        ms = sorted(ts[1:])[1]
        res.append((ctas, chunk >> 10, round(S / ms / 1e6, 1), ok))
if rank == 0:
    for r in res: print("ctas %4d chunk %6d KB  %7.1f GB/s  exact=%s" % r)
dist.destroy_process_group()
