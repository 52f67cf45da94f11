"""Forward-only C2 loss evaluation (lp, loss; no dlogits): time per call and
HBM fraction of the one-read roofline (R V 2 bytes), bf16 and f32."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import _lib, grpo
dev = torch.device("cuda", 0)
N_GROUPS, G, C, T, V = 64, 8, 1, 56, 32064
R = N_GROUPS * G * C * T
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
for dt in (torch.bfloat16, torch.float32):
    g = torch.Generator(device=dev).manual_seed(0)
    logits = (torch.randn(R, V, device=dev, generator=g) * 2).to(dt)
    tokens = torch.randint(31744, 32000, (R,), device=dev, generator=g, dtype=torch.int32)
    rw = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=g).float()
    tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, grpo.GrpoConfig(group_size=G), dtype=dt)
    blp = torch.zeros(N_GROUPS * G, device=dev)
    for _ in range(10):
        tl.launch(logits, tokens, blp, rw, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        tl.launch(logits, tokens, blp, rw, None)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 100
    _lib.dvla_profile_enable(1)
    for _ in range(100):
        tl.launch(logits, tokens, blp, rw, None)
    torch.cuda.synchronize()
    kms, kn = _lib.profile_collect()
    _lib.dvla_profile_enable(0)
    k = kms / max(kn, 1)
    b = logits.numel() * logits.element_size()
    print(f"{dt}: step {ms:.4f} ms, kernel {k:.4f} ms, {b / k / 1e6:.0f} GB/s = "
          f"{b / k / 1e6 / peak:.3f} of HBM peak")
