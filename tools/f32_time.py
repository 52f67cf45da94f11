"""Time the token loss on f32 C2 logits (the parity dtype)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib, grpo
dev = torch.device("cuda", 0)
N_GROUPS, G, C, T, V = 64, 8, 1, 56, 32064
R = N_GROUPS * G * C * T
g = torch.Generator(device=dev).manual_seed(0)
logits = torch.randn(R, V, device=dev, generator=g) * 2
tokens = torch.randint(31744, 32000, (R,), device=dev, generator=g, dtype=torch.int32)
rw = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=g).float()
tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, grpo.GrpoConfig(group_size=G), dtype=torch.float32)
tl.launch(logits, tokens, torch.zeros(N_GROUPS * G, device=dev), rw, None)
blp = (tl.lp_chunk + 0.01).float()
dl = torch.empty_like(logits)
import time
t_end = time.perf_counter() + float(os.environ.get("WARM_S", "1.0"))   # reach the sustained state
while time.perf_counter() < t_end:
    tl.launch(logits, tokens, blp, rw, dl)
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n_it = int(os.environ.get("ITERS", "100"))
e0.record()
for _ in range(n_it):
    tl.launch(logits, tokens, blp, rw, dl)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n_it
algo = 2 * R * V * 4
print(f"f32 C2 step {ms:.3f} ms  {algo / ms / 1e6:.0f} GB/s algorithmic ({algo/1e9:.2f} GB)")
