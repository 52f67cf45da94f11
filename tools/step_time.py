"""Whole-step time of the fused C2 bf16 loss (adv + fused + epilogue), no
profiling events inside the loop (they would sit between PDL-linked
kernels): 200 back-to-back launches between two CUDA events, 3 repeats.
Select a library variant with DVLA_B200_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import grpo
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
for _ in range(20):
    tl.launch(logits, tokens, blp, rw, dl)
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        tl.launch(logits, tokens, blp, rw, dl)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 200)
st = tl.stats(rw)
print(os.environ.get("DVLA_B200_LIB", "default").split("/")[-1],
      " ".join(f"{x:.4f}" for x in res), "ms/step", f"loss {st['loss']:.12g}")
