"""Time the rollout sampling kernel (categorical sample + behaviour
log-prob, one pass over the logits) at the C2 shape; GB/s vs HBM peak."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib
from paper_2605_13276_b200.rollout import sample_action_tokens
R, V, T = 64 * 8 * 56, 32064, 56
g = torch.Generator(device="cuda").manual_seed(0)
lg = (torch.randn(R, V, device="cuda", generator=g) * 2).to(torch.bfloat16)
for _ in range(3):
    sample_action_tokens(lg, T, seed=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for i in range(n):
    sample_action_tokens(lg, T, seed=1, offset=i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
gb = R * V * 2 / 1e9
import hashlib
out = sample_action_tokens(lg, T, seed=1)
h = hashlib.sha256()
for t in (out if isinstance(out, (tuple, list)) else [out]):
    if torch.is_tensor(t):
        h.update(t.cpu().numpy().tobytes())
print(os.environ.get("DVLA_B200_LIB", "default").split("/")[-1], h.hexdigest()[:16])
print(f"sample C2 bf16: {ms:.3f} ms/step  {gb / ms * 1e3:.0f} GB/s  (rows {R}, V {V})")
