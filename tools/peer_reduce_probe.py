"""Latency of the peer exchange's scalar reduction (dvla_peer_reduce) vs
NCCL's all-reduce of one f64, back to back on the same stream:
torchrun --nproc-per-node N tools/peer_reduce_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_13276_b200.exchange import PeerGradExchange  # noqa: E402
from paper_2605_13276_b200.pools import Pool, PoolKind  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", local)
pool = Pool(PoolKind.MODEL_COMPUTE, 64 << 20, device=dev)
gin = torch.zeros(world, 4096, device=dev)
ex = PeerGradExchange(gin, pool)
s = torch.cuda.current_stream()
v = torch.full((1,), float(rank + 1), dtype=torch.float64, device=dev)
f = torch.zeros(3, dtype=torch.int32, device=dev)
out = {}
for name in ("peer_sum", "peer_max", "nccl_sum"):
    for it in range(60):
        if it == 10:
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
        if name == "nccl_sum":
            dist.all_reduce(v)
        else:
            ex.epoch += 1
            if name == "peer_sum":
                ex.reduce_sum_f64(v, s)
            else:
                ex.reduce_max_u32(f, s)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(s)
    torch.cuda.synchronize()
    out[name + "_us"] = round(e0.elapsed_time(e1) * 1e3 / 50, 2)
    v.fill_(float(rank + 1))
if rank == 0:
    print(json.dumps(out), flush=True)
ex.close()
dist.destroy_process_group()
