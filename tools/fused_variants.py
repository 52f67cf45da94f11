"""Time the fused kernel in three regimes to locate the limiter:
forward-only (A ops only), full with all-zero coefficients (B writes zeros,
no exponentials), and the normal full step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib, grpo
dev = torch.device("cuda", 0)
N_GROUPS, G, C, T, V = 64, 8, 1, 56, 32064
R = N_GROUPS * G * C * T
g = torch.Generator(device=dev).manual_seed(0)
logits = (torch.randn(R, V, device=dev, generator=g) * 2).to(torch.bfloat16)
tokens = torch.randint(31744, 32000, (R,), device=dev, generator=g, dtype=torch.int32)
rw = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=g).float()
tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, grpo.GrpoConfig(group_size=G))
tl.launch(logits, tokens, torch.zeros(N_GROUPS * G, device=dev), rw, None)
blp = (tl.lp_chunk + 0.01).float()
dl = torch.empty_like(logits)

def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    _lib.dvla_profile_enable(1)
    for _ in range(n): fn()
    torch.cuda.synchronize()
    ms, k = _lib.profile_collect()
    _lib.dvla_profile_enable(0)
    return ms / k

Nb = R * V * 2
f = timeit(lambda: tl.launch(logits, tokens, blp, rw, None))
print(f"forward-only  {f:.3f} ms  {Nb/f/1e6:.0f} GB/s read")
ones = torch.ones_like(rw)
z = timeit(lambda: tl.launch(logits, tokens, blp, ones, dl))
print(f"full, c == 0  {z:.3f} ms  {2*Nb/z/1e6:.0f} GB/s")
n = timeit(lambda: tl.launch(logits, tokens, blp, rw, dl))
print(f"full, normal  {n:.3f} ms  {2*Nb/n/1e6:.0f} GB/s")
cp = timeit(lambda: _lib.dvla_memcpy_async(dl.data_ptr(), logits.data_ptr(), Nb, torch.cuda.current_stream().cuda_stream))
print(f"memcpy D2D    {cp:.3f} ms  {2*Nb/cp/1e6:.0f} GB/s")
