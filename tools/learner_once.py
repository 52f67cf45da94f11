"""One C4-shaped learner update (for ncu captures of the optimizer tail):
python tools/learner_once.py [--warm N]"""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_13276_b200.pools import Pool, PoolKind  # noqa: E402
from paper_2605_13276_b200.runtime import (GradReducer, SamplerWorker, SwimlaneConfig,  # noqa: E402
                                           TrainerWorker)

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = SwimlaneConfig(n_groups=bench.N_GROUPS, group_size=bench.G, chunks=bench.C, tokens=bench.T,
                     vocab=bench.V, hidden=bench.SWIM_H, seed=23)
n = cfg.vocab * cfg.hidden
R = cfg.n_groups * cfg.group_size * cfg.chunks * cfg.tokens
mp = Pool(PoolKind.MODEL_COMPUTE, n * 26 + (64 << 20), device=dev)
ep = Pool(PoolKind.ENV_AUX, R * (cfg.vocab * 2 + cfg.hidden * 2 + 64) + (256 << 20), device=dev)
tr = TrainerWorker(cfg, 0, mp, GradReducer(1, None), torch.cuda.Stream(device=dev), dev)
sm = SamplerWorker(cfg, 0, 1, [ep], torch.cuda.Stream(device=dev), dev)
msgs, _ = sm.run_epoch(0, tr.snapshot())
for _ in range(a.warm + 1):
    st = tr.update(msgs)
torch.cuda.synchronize()
print("learner update ok", st["version"], st["loss"])
