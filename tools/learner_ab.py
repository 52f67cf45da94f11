"""A/B of the ZeRO-1 reduce-scatter transports inside the timed learner step
(bench._bench_learner_step), alternated REPS times under torchrun:
python -m torch.distributed.run --nproc-per-node N tools/learner_ab.py [REPS] [scatter:chunks,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", local)


def barrier():
    dist.barrier()
    torch.cuda.synchronize()


def mor(x):
    t = torch.tensor([float(x)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


variants = [("peer", "4"), ("peer", "1"), ("nccl", "4")]
if len(sys.argv) > 2:
    variants = [tuple(v.split(":")) for v in sys.argv[2].split(",")]
for rep in range(reps):
    for v in variants:
        sc, gc = v[0], v[1]
        os.environ["DVLA_GATHER_CHUNKS"] = gc
        if len(v) > 3 and v[3]:
            os.environ["DVLA_GRAD_PLAN"] = v[3]
        else:
            os.environ.pop("DVLA_GRAD_PLAN", None)
        if len(v) > 4:
            os.environ["DVLA_GATHER_MODE"] = v[4]
        else:
            os.environ.pop("DVLA_GATHER_MODE", None)
        if len(v) > 2 and v[2]:
            os.environ["DVLA_GRAD_SUB"] = v[2]
        else:
            os.environ.pop("DVLA_GRAD_SUB", None)
        out = bench._bench_learner_step(world, rank, dev, barrier, mor, scatter=sc)
        if rank == 0:
            print(json.dumps({"rep": rep, "scatter": sc + ":" + ":".join(v[2:]),
                              "gather_chunks": gc,
                              "grad_sub": out.get("grad_gemms_per_block"),
                              "value": round(out["value"]),
                              "ms_wall": round(out["ms_per_step_wall"], 3),
                              "ms_dev": round(out["ms_per_step_device"], 3),
                              "phases": out["phases_ms_rank0"],
                              "host": out.get("host_ms_rank0")}), flush=True)
dist.destroy_process_group()
