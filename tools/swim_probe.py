"""Learner step + swimlane at the bench's C4 shape (python or torchrun):
prints one JSON line per rank 0.  Usage:
  python tools/swim_probe.py [--epochs 8] [--no-swim]
  torchrun --nproc-per-node N tools/swim_probe.py"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=8)
    ap.add_argument("--no-swim", action="store_true")
    ap.add_argument("--no-learner", action="store_true")
    ap.add_argument("--disagg", action="store_true")
    a = ap.parse_args()
    world, rank, local = bench._dist()
    torch.cuda.set_device(local)
    if world > 1:
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    dev = torch.device("cuda", local)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def mx(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {"world": world}
    if not a.no_learner:
        out["learner_step"] = bench._bench_learner_step(world, rank, dev, barrier, mx)
    if not a.no_swim:
        barrier()
        out["swimlane"] = bench._bench_swimlane(world, rank, dev, mx, epochs=a.epochs)
    if a.disagg and world > 1:
        barrier()
        for eng, lim in (("ce_head", 0), ("ce_head", 1), ("ce_head", 2)):
            barrier()
            out[f"disaggregated_{eng}_limit{lim}"] = bench._bench_disaggregated(
                world, rank, dev, keep_timeline=True, engine=eng, staleness_limit=lim)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
