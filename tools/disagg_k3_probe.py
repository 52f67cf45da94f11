"""The disaggregated loop at the C4 shape with one learner fed by every other
rank (k rollout ranks per learner, as 2 learners / 6 rollout ranks give at
8 GPUs): torchrun --nproc-per-node 4 tools/disagg_k3_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2605_13276_b200.disagg import run_disaggregated  # noqa: E402
from paper_2605_13276_b200.runtime import SwimlaneConfig  # noqa: E402

world, rank, local = bench._dist()
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = SwimlaneConfig(n_groups=bench.N_GROUPS, group_size=bench.G, chunks=bench.C,
                     tokens=bench.T, vocab=bench.V, hidden=bench.SWIM_H, epochs=6, seed=29)
res = run_disaggregated(cfg, learners=[0], verify=True,
                        body_bytes=max(0, bench.C3_WEIGHT_BYTES - bench.V * bench.SWIM_H * 2),
                        timeout_s=300.0)
if rank == 0:
    print(json.dumps({"role": res.role, "updates": res.updates, "quarantined": res.quarantined,
                      "traj_per_s": res.trajectories_per_s, "mismatched": res.mismatched,
                      "recv_ms_median_max": res.recv_ms_median_max}), flush=True)
dist.destroy_process_group()
