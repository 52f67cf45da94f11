"""Time the fused C2 bf16 step of the library selected by DVLA_B200_LIB and
print a checksum of (loss, lp, dlogits) so variants can be compared bitwise."""
import os, sys, hashlib
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
tl.launch(logits, tokens, blp, rw, dl)
torch.cuda.synchronize()
h = hashlib.sha256(dl.view(torch.int16).cpu().numpy().tobytes())
h.update(tl.lp_chunk.cpu().numpy().tobytes())
res = []
for rep in range(3):
    _lib.dvla_profile_enable(1)
    for _ in range(30):
        tl.launch(logits, tokens, blp, rw, dl)
    torch.cuda.synchronize()
    ms, k = _lib.profile_collect()
    _lib.dvla_profile_enable(0)
    res.append(ms / k)
print(os.environ.get("DVLA_B200_LIB", "default").split("/")[-1], " ".join(f"{x:.4f}" for x in res),
      "ms", h.hexdigest()[:16])
