"""Max |lp_chunk - oracle| of the fused bf16 path at the C2 vocabulary."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import grpo_oracle as O
from paper_2605_13276_b200 import grpo
rng = np.random.default_rng(3)
n_groups, G, C, T, V = 2, 8, 1, 56, 32064
x = torch.from_numpy(rng.normal(0, 2, (n_groups, G, C, T, V)).astype(np.float32)).to(torch.bfloat16)
xs = x.float().numpy()
tokens = rng.integers(31744, 32000, (n_groups, G, C, T)).astype(np.int32)
blp = np.full((n_groups, G, C), -600, np.float32)
rw = rng.integers(0, 2, (n_groups, G)).astype(np.float32)
_, _, st = grpo.grpo_token_grad(x.cuda(), torch.from_numpy(tokens).cuda(), torch.from_numpy(blp).cuda(),
                                torch.from_numpy(rw).cuda(), np.arange(n_groups),
                                grpo.GrpoConfig(group_size=G), write_dlogits=False)
_, _, ost = O.grpo_token_grad(xs, tokens, blp, rw, np.arange(n_groups), want_dlogits=False)
d = np.abs(st["lp_chunk"].cpu().numpy() - ost["lp_chunk"])
print(f"lp_chunk max abs err {d.max():.3e}  mean {d.mean():.3e}  (|lp| ~ {np.abs(ost['lp_chunk']).mean():.0f})")
